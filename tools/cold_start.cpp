// Cold-start breakdown of the first C-ABI call (acceptance.cpp:69-84 caps
// criterion 1, one single-tile propagate, at 0.1 s including everything).
// Build: g++ -O2 -I include tools/cold_start.cpp -L paper_2502_20392_b200 -lsigker_b200 \
//        -Wl,-rpath,$PWD/paper_2502_20392_b200 -o tools/cold_start
#include <chrono>
#include <cstdio>

#include "sigker_b200.h"

int main() {
  using clk = std::chrono::steady_clock;
  auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const double x[2] = {0.0, 1.0};
  double v = 0.0;
  sk_status st{};
  const auto t0 = clk::now();
  const int n = sk_device_count();
  const auto t1 = clk::now();
  int rc = sk_propagate(x, 2, x, 2, 1, 24, SK_STRICT_CORNER, &v, nullptr, nullptr, nullptr, &st);
  const auto t2 = clk::now();
  rc |= sk_propagate(x, 2, x, 2, 1, 24, SK_STRICT_CORNER, &v, nullptr, nullptr, nullptr, &st);
  const auto t3 = clk::now();
  rc |= sk_propagate(x, 2, x, 2, 1, 8, SK_STRICT_CORNER, &v, nullptr, nullptr, nullptr, &st);
  const auto t4 = clk::now();
  std::printf("devices %d: device_count %.1f ms, first propagate (N=24, literal) %.1f ms, second %.2f ms, "
              "first N=8 %.2f ms; K = %.17g rc %d\n",
              n, ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), v, rc);
  return 0;
}
