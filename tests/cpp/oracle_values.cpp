// Prints truncated_signature_kernel(20), truncated_kernel_levelwise(20),
// goursat_fd_solve(64) and picard_global(16, 200) for two CSV series
// (host-only oracles of the validate suites; no GPU needed).
#include <cstdio>

#include "sigker/csv.hpp"
#include "sigker/oracles.hpp"

int main(int argc, char** argv) {
  if (argc != 3) return 2;
  const auto x = sigker::load_csv(argv[1]);
  const auto y = sigker::load_csv(argv[2]);
  std::printf("%.17g %.17g %.17g %.17g\n", sigker::oracle::truncated_signature_kernel(x, y, 20),
              sigker::oracle::truncated_kernel_levelwise(x, y, 20), sigker::oracle::goursat_fd_solve(x, y, 64),
              sigker::oracle::picard_global(x, y, 16, 200).value);
  return 0;
}
