// `sigker` command-line tool on the B200 engine: the reference CLI's
// subcommands, options, outputs and exit codes (tools/main.cpp:86-424) --
//   kernel x.csv y.csv [--order N | --tol T] [--grid out.csv] [--json]
//   gram inputs... [--out gram.csv] [--order N | --tol T] [--bound]
//   validate --suite closed-form|oracle-triangle|bound|invariance|all [--inject-fault]
//   bench [--lengths ...] [--dims ...] [--repeats R] [--order N] [--out f.csv]
//   gen [--kind brownian|fbm|near-periodic] [--len L] [--dim D] [--seed S] [--out f.csv]
// Exit codes: 0 ok, 2 usage/input error, 3 numeric error (or failed Gram
// entries), 4 validation failure.  --config FILE reads a flat JSON object
// whose keys are option names; flags on the command line override it.
// --threads is accepted and ignored (the GPU schedule replaces the pool).
#include <algorithm>
#include <cctype>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "sigker/csv.hpp"
#include "sigker/datagen.hpp"
#include "sigker/errors.hpp"
#include "sigker/gram.hpp"
#include "sigker/oracles.hpp"
#include "sigker/truncation.hpp"
#include "sigker/validate.hpp"
#include "sigker/wavefront.hpp"

namespace fs = std::filesystem;

namespace {

constexpr int kOk = 0, kUsage = 2, kNumeric = 3, kValidation = 4;

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};

std::string g17(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

// ------------------------------------------------------------ tiny JSON
struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double n = 0;
  std::string s;
  std::vector<Json> a;
  std::map<std::string, Json> o;
};

struct JsonReader {
  const std::string& t;
  size_t i = 0;
  explicit JsonReader(const std::string& text) : t(text) {}
  void ws() {
    while (i < t.size() && std::isspace(static_cast<unsigned char>(t[i]))) ++i;
  }
  [[noreturn]] void fail(const std::string& what) { throw Usage("JSON: " + what + " at offset " + std::to_string(i)); }
  std::string str() {
    std::string out;
    ++i;  // opening quote
    while (i < t.size() && t[i] != '"') {
      if (t[i] == '\\' && i + 1 < t.size()) {
        const char e = t[++i];
        out += e == 'n' ? '\n' : e == 't' ? '\t' : e;
      } else {
        out += t[i];
      }
      ++i;
    }
    if (i >= t.size()) fail("unterminated string");
    ++i;
    return out;
  }
  Json value() {
    ws();
    if (i >= t.size()) fail("unexpected end");
    Json v;
    const char c = t[i];
    if (c == '{') {
      v.kind = Json::Obj;
      ++i;
      ws();
      if (i < t.size() && t[i] == '}') return ++i, v;
      for (;;) {
        ws();
        if (i >= t.size() || t[i] != '"') fail("expected a key");
        const std::string k = str();
        ws();
        if (i >= t.size() || t[i] != ':') fail("expected ':'");
        ++i;
        v.o[k] = value();
        ws();
        if (i < t.size() && t[i] == ',') {
          ++i;
          continue;
        }
        if (i < t.size() && t[i] == '}') return ++i, v;
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = Json::Arr;
      ++i;
      ws();
      if (i < t.size() && t[i] == ']') return ++i, v;
      for (;;) {
        v.a.push_back(value());
        ws();
        if (i < t.size() && t[i] == ',') {
          ++i;
          continue;
        }
        if (i < t.size() && t[i] == ']') return ++i, v;
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = Json::Str;
      v.s = str();
      return v;
    }
    if (t.compare(i, 4, "true") == 0) return i += 4, v.kind = Json::Bool, v.b = true, v;
    if (t.compare(i, 5, "false") == 0) return i += 5, v.kind = Json::Bool, v;
    if (t.compare(i, 4, "null") == 0) return i += 4, v;
    char* end = nullptr;
    v.n = std::strtod(t.c_str() + i, &end);
    if (end == t.c_str() + i) fail("bad value");
    i = static_cast<size_t>(end - t.c_str());
    v.kind = Json::Num;
    return v;
  }
};

std::string quote(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    if (c == '\n') {
      o += "\\n";
      continue;
    }
    o += c;
  }
  return o + "\"";
}

// ordered JSON object writer
struct JsonOut {
  std::vector<std::pair<std::string, std::string>> kv;
  void num(const std::string& k, double v) { kv.emplace_back(k, std::isfinite(v) ? g17(v) : "null"); }
  void integer(const std::string& k, long long v) { kv.emplace_back(k, std::to_string(v)); }
  void boolean(const std::string& k, bool v) { kv.emplace_back(k, v ? "true" : "false"); }
  void str(const std::string& k, const std::string& v) { kv.emplace_back(k, quote(v)); }
  void raw(const std::string& k, const std::string& v) { kv.emplace_back(k, v); }
  std::string dump(int indent = -1) const {
    std::string o = "{";
    for (size_t k = 0; k < kv.size(); ++k) {
      if (k) o += ",";
      if (indent >= 0) o += "\n" + std::string(indent, ' ');
      o += quote(kv[k].first) + ":" + (indent >= 0 ? " " : "") + kv[k].second;
    }
    if (indent >= 0 && !kv.empty()) o += "\n";
    return o + "}";
  }
};

// ------------------------------------------------------------ arguments
struct Args {
  std::vector<std::string> pos;
  std::map<std::string, std::vector<std::string>> opt;  // --name -> values
  Json cfg;

  bool has(const std::string& k) const { return opt.count(k) > 0 || (cfg.kind == Json::Obj && cfg.o.count(k) > 0); }
  bool cli(const std::string& k) const { return opt.count(k) > 0; }
  std::string get(const std::string& k, const std::string& dflt) const {
    if (auto it = opt.find(k); it != opt.end()) return it->second.back();
    if (cfg.kind == Json::Obj)
      if (auto it = cfg.o.find(k); it != cfg.o.end()) {
        if (it->second.kind == Json::Str) return it->second.s;
        if (it->second.kind == Json::Num) return g17(it->second.n);
        if (it->second.kind == Json::Bool) return it->second.b ? "1" : "0";
        throw Usage("config key '" + k + "' has an unsupported type");
      }
    return dflt;
  }
  double num(const std::string& k, double dflt) const {
    const std::string v = get(k, "");
    if (v.empty()) return dflt;
    char* end = nullptr;
    const double d = std::strtod(v.c_str(), &end);
    if (end != v.c_str() + v.size()) throw Usage("--" + k + ": not a number: " + v);
    return d;
  }
  long long integer(const std::string& k, long long dflt) const {
    const double d = num(k, static_cast<double>(dflt));
    if (d != std::floor(d)) throw Usage("--" + k + ": not an integer");
    return static_cast<long long>(d);
  }
  std::vector<long long> ints(const std::string& k, std::vector<long long> dflt) const {
    auto it = opt.find(k);
    if (it == opt.end()) {
      if (cfg.kind == Json::Obj)
        if (auto c = cfg.o.find(k); c != cfg.o.end() && c->second.kind == Json::Arr) {
          std::vector<long long> out;
          for (const Json& e : c->second.a) out.push_back(static_cast<long long>(e.n));
          return out;
        }
      return dflt;
    }
    std::vector<long long> out;
    for (const std::string& v : it->second) {
      std::stringstream ss(v);
      std::string part;
      while (std::getline(ss, part, ',')) out.push_back(std::stoll(part));
    }
    return out;
  }
};

Args parse_args(int argc, char** argv, int first, const std::vector<std::string>& flags,
                const std::vector<std::string>& multi) {
  Args a;
  for (int k = first; k < argc; ++k) {
    std::string s = argv[k];
    if (s.rfind("--", 0) == 0) {
      std::string name = s.substr(2), value;
      const size_t eq = name.find('=');
      if (eq != std::string::npos) {
        value = name.substr(eq + 1);
        name = name.substr(0, eq);
      } else if (std::find(flags.begin(), flags.end(), name) != flags.end()) {
        value = "1";
      } else {
        if (k + 1 >= argc) throw Usage("--" + name + " needs a value");
        value = argv[++k];
        // multi-valued options take every following non-option token
        if (std::find(multi.begin(), multi.end(), name) != multi.end())
          while (k + 1 < argc && std::string(argv[k + 1]).rfind("--", 0) != 0) value += std::string(",") + argv[++k];
      }
      a.opt[name].push_back(value);
    } else {
      a.pos.push_back(s);
    }
  }
  if (a.cli("config")) {
    std::ifstream in(a.get("config", ""));
    if (!in) throw Usage("cannot open config file " + a.get("config", ""));
    std::stringstream ss;
    ss << in.rdbuf();
    JsonReader r(ss.str());
    a.cfg = r.value();
    if (a.cfg.kind != Json::Obj) throw Usage("config file " + a.get("config", "") + " must hold a JSON object");
  }
  return a;
}

sigker::TruncationPolicy policy_of(const Args& a) {
  const bool o = a.has("order"), t = a.has("tol");
  if (o && t) throw Usage("--order and --tol are mutually exclusive");
  if (t) return sigker::TruncationPolicy::adaptive(a.num("tol", 1e-12));
  if (o) return sigker::TruncationPolicy::fixed(static_cast<int>(a.integer("order", 7)));
  return sigker::TruncationPolicy{};  // fixed, order 7
}

fs::path meta_path(const fs::path& out) {
  fs::path m = out;
  if (m.extension() == ".json")
    m += ".meta.json";
  else
    m.replace_extension(".json");
  return m;
}

// ------------------------------------------------------------ subcommands
int kernel_cmd(const Args& a) {
  if (a.pos.size() != 2) throw Usage("kernel: expected two CSV inputs x y");
  const auto policy = policy_of(a);
  sigker::TimeSeries x = sigker::load_csv(a.pos[0]);
  sigker::TimeSeries y = sigker::load_csv(a.pos[1]);
  if (x.dim() != y.dim())
    throw std::invalid_argument("kernel: input dimensions differ (" + std::to_string(x.dim()) + " vs " +
                                std::to_string(y.dim()) + ")");
  const size_t len = std::max<size_t>({x.length(), y.length(), 2});
  x = sigker::pad_to_length(x, len);
  y = sigker::pad_to_length(y, len);
  const std::string grid = a.get("grid", "");
  const auto t0 = std::chrono::steady_clock::now();
  sigker::KernelResult r;
  if (grid.empty()) {
    r = sigker::propagate_with_policy(x, y, policy);
  } else {
    int n = policy.order;
    bool conv = true;
    if (policy.mode == sigker::TruncationPolicy::Mode::kAdaptive) {
      const auto est = sigker::estimate_order(sigker::IncrementTable(x, y).max_abs_rho(), len, policy.tol);
      n = est.order;
      conv = est.converged;
    }
    r = sigker::propagate_grid(x, y, n);
    r.order_converged = conv;
    sigker::save_matrix_csv(r.grid, r.grid_rows, r.grid_cols, grid);
  }
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (!r.order_converged) std::cerr << "warning: adaptive search saturated at order 64 without meeting the tolerance\n";
  std::cout << "K=" << g17(r.value) << "\n";
  if (a.has("json") && a.get("json", "0") != "0") {
    JsonOut j;
    j.integer("schema", 1);
    j.num("value", r.value);
    j.integer("order", r.order);
    j.boolean("order_converged", r.order_converged);
    j.integer("tiles", static_cast<long long>(r.tiles_processed));
    j.integer("peak_live_series", static_cast<long long>(r.peak_live_series));
    j.integer("threads", a.integer("threads", 1));
    j.num("wall_seconds", secs);
    std::cout << j.dump() << "\n";
  }
  return kOk;
}

std::vector<fs::path> csv_inputs(const std::vector<std::string>& ins) {
  std::vector<fs::path> files;
  for (const std::string& s : ins) {
    const fs::path p(s);
    if (fs::is_directory(p)) {
      std::vector<fs::path> dir;
      for (const auto& e : fs::directory_iterator(p))
        if (e.is_regular_file() && e.path().extension() == ".csv") dir.push_back(e.path());
      std::sort(dir.begin(), dir.end());
      files.insert(files.end(), dir.begin(), dir.end());
    } else {
      files.push_back(p);
    }
  }
  if (files.empty()) throw Usage("gram: no input CSV files");
  return files;
}

int gram_cmd(const Args& a) {
  sigker::GramOptions opts;
  opts.policy = policy_of(a);
  opts.compute_bound = a.has("bound") && a.get("bound", "0") != "0";
  const std::string out = a.get("out", "gram.csv");
  const auto files = csv_inputs(a.pos);
  std::vector<sigker::TimeSeries> family;
  for (const auto& f : files) family.push_back(sigker::load_csv(f));
  const sigker::GramResult r = sigker::gram_matrix(family, opts);
  sigker::save_matrix_csv(r.values, r.size, r.size, out);
  JsonOut j;
  j.integer("schema", 1);
  j.integer("size", static_cast<long long>(r.size));
  j.str("policy", r.adaptive ? "adaptive" : "fixed");
  j.integer("order_min", r.min_order);
  j.integer("order_max", r.max_order);
  j.boolean("orders_converged", r.orders_converged);
  j.num("wall_seconds", r.wall_seconds);
  j.integer("peak_live_series", static_cast<long long>(r.peak_live_series));
  std::string names = "[";
  for (size_t k = 0; k < files.size(); ++k) names += (k ? ", " : "") + quote(files[k].string());
  j.raw("inputs", names + "]");
  if (opts.compute_bound) {
    j.num("bound", r.bound);
    j.num("max_abs_increment_product", r.max_abs_increment_product);
  }
  std::string fl = "[";
  for (size_t k = 0; k < r.failures.size(); ++k) {
    JsonOut e;
    e.integer("row", static_cast<long long>(r.failures[k].row));
    e.integer("col", static_cast<long long>(r.failures[k].col));
    e.str("message", r.failures[k].message);
    fl += (k ? ", " : "") + e.dump();
  }
  j.raw("failures", fl + "]");
  std::ofstream(meta_path(out)) << j.dump(2) << "\n";
  std::cout << "gram " << r.size << "x" << r.size << " -> " << out << "\n";
  for (const auto& f : r.failures) std::cerr << "entry (" << f.row << ", " << f.col << ") failed: " << f.message << "\n";
  return r.failures.empty() ? kOk : kNumeric;
}

int validate_cmd(const Args& a) {
  const std::string suite = a.get("suite", "");
  if (suite.empty()) throw Usage("validate: --suite is required");
  sigker::validate::SuiteOptions o;
  o.seed = static_cast<std::uint64_t>(a.integer("seed", 12345));
  o.cases = static_cast<size_t>(a.integer("cases", 0));
  o.tolerance = a.num("tolerance", 0.0);
  o.inject_fault = a.has("inject-fault") && a.get("inject-fault", "0") != "0";
  const std::vector<std::string> names =
      suite == "all" ? sigker::validate::suite_names() : std::vector<std::string>{suite};
  bool ok = true;
  for (const std::string& n : names) {
    const auto rep = sigker::validate::run_suite(n, o);
    std::printf("%-16s cases=%-4zu failures=%-3zu max_error=%.3e %s\n", rep.name.c_str(), rep.cases, rep.failures,
                rep.max_error, rep.passed() ? "PASS" : "FAIL");
    for (const auto& m : rep.messages) std::printf("  %s\n", m.c_str());
    ok = ok && rep.passed();
  }
  return ok ? kOk : kValidation;
}

int bench_cmd(const Args& a) {
  const auto lengths = a.ints("lengths", {129, 257, 513});
  const auto dims = a.ints("dims", {2});
  const long long repeats = a.integer("repeats", 10);
  const int order = static_cast<int>(a.integer("order", 7));
  const auto seed = static_cast<std::uint64_t>(a.integer("seed", 42));
  const long long oracle_max = a.integer("oracle-max-len", 64);
  const int depth = static_cast<int>(a.integer("oracle-depth", 20));
  const std::string out = a.get("out", "");
  std::ofstream file;
  std::ostream* os = &std::cout;
  if (!out.empty()) {
    file.open(out);
    if (!file) throw Usage("cannot write " + out);
    os = &file;
  }
  *os << "length,dim,order,mean_seconds,stdev_seconds,peak_live_series,mape\n";
  for (long long len : lengths)
    for (long long dim : dims) {
      const auto x = sigker::datagen::brownian(static_cast<size_t>(len), static_cast<size_t>(dim), seed);
      const auto y = sigker::datagen::brownian(static_cast<size_t>(len), static_cast<size_t>(dim), seed + 1);
      std::vector<double> t;
      sigker::KernelResult r;
      for (long long k = 0; k < repeats; ++k) {
        const auto t0 = std::chrono::steady_clock::now();
        r = sigker::propagate(x, y, order);
        t.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
      }
      double mean = 0, var = 0;
      for (double v : t) mean += v;
      mean /= static_cast<double>(t.size());
      for (double v : t) var += (v - mean) * (v - mean);
      const double sd = t.size() > 1 ? std::sqrt(var / static_cast<double>(t.size() - 1)) : 0.0;
      std::string mape;
      if (len <= oracle_max) {
        const double ref = sigker::oracle::truncated_kernel_levelwise(x, y, depth);
        if (ref != 0.0) mape = g17(std::abs(r.value - ref) / std::abs(ref));
      }
      *os << len << ',' << dim << ',' << order << ',' << g17(mean) << ',' << g17(sd) << ',' << r.peak_live_series << ','
          << mape << "\n";
    }
  return kOk;
}

int gen_cmd(const Args& a) {
  const std::string kind = a.get("kind", "brownian");
  const auto len = static_cast<size_t>(a.integer("len", 33));
  const auto dim = static_cast<size_t>(a.integer("dim", 2));
  const auto seed = static_cast<std::uint64_t>(a.integer("seed", 1));
  sigker::TimeSeries ts = [&] {
    if (kind == "brownian") return sigker::datagen::brownian(len, dim, seed);
    if (kind == "fbm") return sigker::datagen::fbm(len, dim, a.num("hurst", 0.5), seed);
    if (kind == "near-periodic")
      return sigker::datagen::near_periodic(len, dim, a.num("period", 0.25), a.num("amplitude", 1.0),
                                            a.num("noise", 0.0), seed);
    throw Usage("unknown generator kind: " + kind);
  }();
  const std::string out = a.get("out", "");
  if (out.empty()) {
    sigker::write_csv(ts, std::cout);
  } else {
    sigker::save_csv(ts, out);
    std::cout << kind << " length=" << len << " dim=" << dim << " -> " << out << "\n";
  }
  return kOk;
}

const char* kUsageText =
    "usage: sigker <kernel|gram|validate|bench|gen> [options]\n"
    "  kernel x.csv y.csv [--order N | --tol T] [--grid out.csv] [--json] [--config f.json]\n"
    "  gram inputs... [--out gram.csv] [--order N | --tol T] [--bound] [--config f.json]\n"
    "  validate --suite closed-form|oracle-triangle|bound|invariance|all [--seed S] [--cases C]\n"
    "           [--tolerance T] [--inject-fault]\n"
    "  bench [--lengths L...] [--dims D...] [--repeats R] [--order N] [--seed S]\n"
    "        [--oracle-max-len L] [--oracle-depth M] [--out f.csv]\n"
    "  gen [--kind brownian|fbm|near-periodic] [--len L] [--dim D] [--seed S] [--hurst H]\n"
    "      [--period P] [--amplitude A] [--noise S] [--out f.csv]\n";

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
    std::cout << kUsageText;
    return argc < 2 ? kUsage : kOk;
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "kernel") return kernel_cmd(parse_args(argc, argv, 2, {"json"}, {}));
    if (cmd == "gram") return gram_cmd(parse_args(argc, argv, 2, {"bound"}, {}));
    if (cmd == "validate") return validate_cmd(parse_args(argc, argv, 2, {"inject-fault"}, {}));
    if (cmd == "bench") return bench_cmd(parse_args(argc, argv, 2, {}, {"lengths", "dims"}));
    if (cmd == "gen") return gen_cmd(parse_args(argc, argv, 2, {}, {}));
    std::cerr << "error: unknown subcommand " << cmd << "\n" << kUsageText;
    return kUsage;
  } catch (const Usage& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kUsage;
  } catch (const sigker::NumericOverflowError& e) {
    std::cerr << "numeric error: " << e.what() << "\n";
    return kNumeric;
  } catch (const sigker::NumericError& e) {
    std::cerr << "numeric error: " << e.what() << "\n";
    return kNumeric;
  } catch (const sigker::ParseError& e) {
    std::cerr << "input error: " << e.what() << "\n";
    return kUsage;
  } catch (const std::invalid_argument& e) {
    std::cerr << "input error: " << e.what() << "\n";
    return kUsage;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kUsage;
  }
}
