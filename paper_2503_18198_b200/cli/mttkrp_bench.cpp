// mttkrp-bench (GPU backend): the reference's benchmark CLI (tools/mttkrp_bench.cpp) on the
// B200 path.  Same subcommands (gen / run / inspect), options, defaults, exit codes (0 ok,
// 1 error, 2 verify failed), console lines and JSON report schema (report.cpp:7-44:
// timing.modes[].{scheme,wall_ms,min_ms,median_ms,busy_workers,elements_per_worker},
// balance[], memory, verify.{tolerance,max_rel_err_per_mode,max_rel_err,passed}), so the
// reference's CLI tests (tests/test_cli.cpp) run unchanged against this binary.
//
// Differences, all GPU-specific:
//   --backend gpu     the only backend (the reference's CPU executor is not shipped);
//   --kappa default   SPMTTKRP_WORKERS, else the device's SM count (the reference: the host's
//                     logical cores, mttkrp_bench.cpp:54-57);
//   --tensor X.mkbt   a binary tensor cache is read directly; --cache parses a .tns once and
//                     keeps <file>.mkbt next to it;
//   run --verify      compares against the deterministic device executor, which is bitwise
//                     equal to the reference's oracle_mttkrp (tests/test_gpu_mttkrp.py);
//   run --fast        the B200 fast executor (MK_EXEC_FAST, within 1e-4 of the oracle) instead
//                     of the reference's executor contract (MK_EXEC_REFERENCE: Scheme 1 modes
//                     bitwise equal to --deterministic).
// No third-party dependency: argument parsing and JSON output are written out here.
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "mttkrp_b200/frostt.hpp"
#include "mttkrp_b200/mttkrp.hpp"

namespace mttkrp = mttkrp_b200;

namespace {

constexpr int exit_ok = 0;
constexpr int exit_error = 1;
constexpr int exit_verify_failed = 2;
constexpr int exit_usage = 106;  // CLI11's ValidationError code (argument errors)

// ----------------------------------------------------------------------------- JSON
class Json {
 public:
  using Array = std::vector<Json>;
  using Object = std::vector<std::pair<std::string, Json>>;
  Json() : v_(nullptr) {}
  Json(std::nullptr_t) : v_(nullptr) {}
  Json(bool b) : v_(b) {}
  Json(int x) : v_(static_cast<long long>(x)) {}
  Json(long x) : v_(static_cast<long long>(x)) {}
  Json(long long x) : v_(x) {}
  Json(unsigned x) : v_(static_cast<unsigned long long>(x)) {}
  Json(unsigned long x) : v_(static_cast<unsigned long long>(x)) {}
  Json(unsigned long long x) : v_(x) {}
  Json(double x) : v_(x) {}
  Json(const char* s) : v_(std::string(s)) {}
  Json(std::string s) : v_(std::move(s)) {}
  Json(std::string_view s) : v_(std::string(s)) {}
  template <typename T>
  Json(const std::vector<T>& xs) : v_(Array{}) {
    for (const auto& x : xs) std::get<Array>(v_).emplace_back(x);
  }
  static Json object() {
    Json j;
    j.v_ = Object{};
    return j;
  }
  static Json array() {
    Json j;
    j.v_ = Array{};
    return j;
  }
  Json& operator[](const std::string& k) {
    if (std::holds_alternative<std::nullptr_t>(v_)) v_ = Object{};
    auto& o = std::get<Object>(v_);
    for (auto& kv : o)
      if (kv.first == k) return kv.second;
    o.emplace_back(k, Json());
    return o.back().second;
  }
  void push_back(Json j) { std::get<Array>(v_).push_back(std::move(j)); }
  std::string dump(int indent = 2) const {
    std::string s;
    write(s, indent, 0);
    return s;
  }

 private:
  static void esc(std::string& s, const std::string& x) {
    s.push_back('"');
    for (unsigned char c : x) {
      switch (c) {
        case '"': s += "\\\""; break;
        case '\\': s += "\\\\"; break;
        case '\n': s += "\\n"; break;
        case '\t': s += "\\t"; break;
        case '\r': s += "\\r"; break;
        default:
          if (c < 0x20) {
            char b[8];
            std::snprintf(b, sizeof b, "\\u%04x", c);
            s += b;
          } else {
            s.push_back(static_cast<char>(c));
          }
      }
    }
    s.push_back('"');
  }
  void write(std::string& s, int ind, int depth) const {
    const std::string pad(static_cast<size_t>(ind * (depth + 1)), ' ');
    const std::string pad0(static_cast<size_t>(ind * depth), ' ');
    if (std::holds_alternative<std::nullptr_t>(v_)) {
      s += "null";
    } else if (auto* b = std::get_if<bool>(&v_)) {
      s += *b ? "true" : "false";
    } else if (auto* i = std::get_if<long long>(&v_)) {
      s += std::to_string(*i);
    } else if (auto* u = std::get_if<unsigned long long>(&v_)) {
      s += std::to_string(*u);
    } else if (auto* d = std::get_if<double>(&v_)) {
      if (!std::isfinite(*d)) {
        s += "null";
      } else {
        char b[32];
        std::snprintf(b, sizeof b, "%.17g", *d);
        s += b;
        if (!std::strpbrk(b, ".eE")) s += ".0";
      }
    } else if (auto* str = std::get_if<std::string>(&v_)) {
      esc(s, *str);
    } else if (auto* a = std::get_if<Array>(&v_)) {
      if (a->empty()) {
        s += "[]";
        return;
      }
      s += "[\n";
      for (size_t k = 0; k < a->size(); ++k) {
        s += pad;
        (*a)[k].write(s, ind, depth + 1);
        s += k + 1 < a->size() ? ",\n" : "\n";
      }
      s += pad0 + "]";
    } else if (auto* o = std::get_if<Object>(&v_)) {
      if (o->empty()) {
        s += "{}";
        return;
      }
      s += "{\n";
      for (size_t k = 0; k < o->size(); ++k) {
        s += pad;
        esc(s, (*o)[k].first);
        s += ": ";
        (*o)[k].second.write(s, ind, depth + 1);
        s += k + 1 < o->size() ? ",\n" : "\n";
      }
      s += pad0 + "}";
    }
  }
  std::variant<std::nullptr_t, bool, long long, unsigned long long, double, std::string, Array,
               Object>
      v_;
};

Json to_json(const mttkrp::BalanceMetrics& bm) {  // report.cpp:7-15
  Json j = Json::object();
  j["mode"] = bm.mode;
  j["scheme"] = mttkrp::to_string(bm.scheme);
  j["kappa"] = bm.kappa;
  j["loads"] = bm.loads;
  j["owned_index_counts"] = bm.owned_index_counts;
  j["max_over_mean"] = bm.max_over_mean;
  j["empty_partitions"] = bm.empty_partitions;
  return j;
}

Json to_json(const mttkrp::MemoryEstimate& m) {  // report.cpp:17-23
  Json j = Json::object();
  j["bits_per_element"] = m.bits_per_element;
  j["total_copy_bits"] = m.total_copy_bits;
  j["total_copy_bytes"] = m.total_copy_bytes;
  j["factor_matrix_bytes"] = m.factor_matrix_bytes;
  j["storage_bytes_actual"] = m.storage_bytes_actual;
  return j;
}

Json to_json(const mttkrp::ModeTiming& mt) {  // report.cpp:25-32
  Json j = Json::object();
  j["mode"] = mt.mode;
  j["scheme"] = mttkrp::to_string(mt.scheme);
  j["wall_ms"] = mt.wall_ms;
  j["min_ms"] = mt.min_ms;
  j["median_ms"] = mt.median_ms;
  j["busy_workers"] = mt.busy_workers;
  j["elements_per_worker"] = mt.elements_per_worker;
  return j;
}

Json to_json(const mttkrp::TimingReport& r) {  // report.cpp:34-44
  Json modes = Json::array();
  for (const auto& mt : r.modes) modes.push_back(to_json(mt));
  Json j = Json::object();
  j["iters"] = r.iters;
  j["modes"] = std::move(modes);
  j["total_ms"] = r.total_ms;
  j["total_min_ms"] = r.total_min_ms;
  j["total_median_ms"] = r.total_median_ms;
  j["outputs_bit_identical"] = r.outputs_bit_identical;
  return j;
}

// ----------------------------------------------------------------------------- options
struct Options {
  std::string tensor_path;
  std::size_t rank = 32;
  std::size_t kappa = 0;  // 0 = SPMTTKRP_WORKERS or the device's SM count
  std::size_t batch_p = 32;
  std::string policy = "adaptive";
  std::string strategy = "cyclic";
  std::string precision = "f32";
  std::string backend = "gpu";
  std::size_t iters = 1;
  std::uint64_t seed = 1;
  bool verify = false;
  bool deterministic = false;
  bool fast = false;
  bool cache = false;
  std::string json_path;
  std::vector<mttkrp::index_t> dims;
  std::size_t nnz = 0;
  bool nnz_set = false;
  std::string dist = "uniform";
  std::size_t skew_mode = 0;
  std::size_t skew_distinct = 2;
  std::string out_path;
};

struct UsageError {
  std::string msg;
};

std::size_t detect_kappa() {
  int sms = 0;
  if (mk_device_sm_count(0, &sms) != MK_OK || sms < 1)
    throw mttkrp::error(std::string("gpu backend: no CUDA device (") + mk_last_error() + ")");
  return static_cast<std::size_t>(sms);
}

mttkrp::SchemePolicy parse_policy(const std::string& s) {
  if (s == "adaptive") return mttkrp::SchemePolicy::adaptive;
  if (s == "s1") return mttkrp::SchemePolicy::scheme1_only;
  if (s == "s2") return mttkrp::SchemePolicy::scheme2_only;
  throw mttkrp::error("unknown policy '" + s + "'");
}

mttkrp::Strategy parse_strategy(const std::string& s) {
  if (s == "cyclic") return mttkrp::Strategy::cyclic;
  if (s == "lpt") return mttkrp::Strategy::least_loaded;
  throw mttkrp::error("unknown strategy '" + s + "'");
}

void write_json_file(const std::string& path, const Json& j) {
  std::ofstream out(path);
  if (!out) throw mttkrp::error("cannot write JSON report to '" + path + "'");
  out << j.dump(2) << '\n';
}

void maybe_write_json(const Options& opt, const Json& j) {
  if (!opt.json_path.empty()) write_json_file(opt.json_path, j);
}

bool is_cache_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  char m[4] = {};
  in.read(m, 4);
  return in.gcount() == 4 && std::memcmp(m, "MKBT", 4) == 0;
}

template <typename T>
mttkrp::SparseTensorCOO<T> load_tensor(const Options& opt, Json& report) {
  mttkrp::FrosttParseResult<T> parsed{mttkrp::SparseTensorCOO<T>(mttkrp::Shape({1})), 0};
  if (is_cache_file(opt.tensor_path))
    parsed = {mttkrp::load_tensor_cache<T>(opt.tensor_path), 0};
  else if (opt.cache)
    parsed = mttkrp::load_tensor<T>(opt.tensor_path);
  else
    parsed = mttkrp::read_frostt_file<T>(opt.tensor_path);
  if (parsed.duplicates_merged > 0)
    std::cerr << "warning: merged " << parsed.duplicates_merged
              << " duplicate index tuples (values summed)\n";
  if (parsed.tensor.mode_count() < 3)
    std::cerr << "warning: tensor has fewer than 3 modes; this layout targets "
                 "3-mode and higher tensors\n";
  report["tensor"] = opt.tensor_path;
  report["shape"] = parsed.tensor.shape().dims;
  report["nnz"] = parsed.tensor.nnz();
  report["duplicates_merged"] = parsed.duplicates_merged;
  return std::move(parsed.tensor);
}

template <typename T>
int cmd_run(const Options& opt) {
  Json report = Json::object();
  report["command"] = "run";
  auto tensor = load_tensor<T>(opt, report);

  const std::size_t kappa = opt.kappa ? opt.kappa : detect_kappa();
  const auto policy = parse_policy(opt.policy);
  const auto strategy = parse_strategy(opt.strategy);
  mttkrp::ExecConfig config{kappa, opt.batch_p, opt.deterministic};
  config.fast = opt.fast;
  config.validate();

  report["backend"] = opt.backend;
  report["rank"] = opt.rank;
  report["kappa"] = kappa;
  report["batch_p"] = opt.batch_p;
  report["policy"] = opt.policy;
  report["strategy"] = opt.strategy;
  report["precision"] = opt.precision;
  report["iters"] = opt.iters;
  report["seed"] = opt.seed;
  report["deterministic"] = opt.deterministic;
  report["exec"] = opt.deterministic ? "deterministic" : (opt.fast ? "fast" : "reference");

  auto plans = mttkrp::build_mode_plans(tensor, kappa, strategy, policy);
  auto factors = mttkrp::random_factors<T>(tensor.shape(), opt.rank, opt.seed);
  auto timed = mttkrp::run_timed(tensor, plans, factors, config, opt.iters);

  report["timing"] = to_json(timed.report);
  Json balance = Json::array();
  for (std::size_t d = 0; d < plans.size(); ++d)
    balance.push_back(to_json(mttkrp::balance_metrics(plans[d], mttkrp::plan_degrees(tensor, plans[d]))));
  report["balance"] = std::move(balance);
  report["memory"] = to_json(mttkrp::estimate_memory(tensor, opt.rank));

  std::printf("tensor %s: %zu modes, nnz=%zu\n", opt.tensor_path.c_str(), tensor.mode_count(),
              tensor.nnz());
  for (const auto& mt : timed.report.modes)
    std::printf("  mode %zu  %-7s  busy %zu/%zu  min %.3f ms  median %.3f ms\n", mt.mode,
                std::string(mttkrp::to_string(mt.scheme)).c_str(), mt.busy_workers, kappa,
                mt.min_ms, mt.median_ms);
  std::printf("total: min %.3f ms  median %.3f ms over %zu iter(s)\n", timed.report.total_min_ms,
              timed.report.total_median_ms, opt.iters);

  bool verify_passed = true;
  if (opt.verify) {
    const double tol = mttkrp::verify_tolerance<T>();
    Json verify = Json::object();
    verify["enabled"] = true;
    verify["tolerance"] = tol;
    verify["reference"] = "deterministic device executor (bitwise = oracle_mttkrp)";
    Json per_mode = Json::array();
    double worst = 0.0;
    std::size_t worst_mode = 0;
    mttkrp::VerifyResult worst_detail;
    const mttkrp::ExecConfig det{kappa, opt.batch_p, true};
    for (std::size_t d = 0; d < plans.size(); ++d) {
      auto reference = mttkrp::mttkrp_mode(tensor, plans[d], factors, det);
      auto res = mttkrp::verify_against(timed.outputs[d], reference);
      per_mode.push_back(res.max_rel_err);
      if (res.max_rel_err > worst) {
        worst = res.max_rel_err;
        worst_mode = d;
        worst_detail = res;
      }
    }
    verify_passed = worst <= tol;
    verify["max_rel_err_per_mode"] = std::move(per_mode);
    verify["max_rel_err"] = worst;
    verify["passed"] = verify_passed;
    report["verify"] = std::move(verify);
    if (verify_passed)
      std::printf("verify: OK, max relative error %.3e (tolerance %.0e)\n", worst, tol);
    else
      std::fprintf(stderr,
                   "verify: FAILED, max relative error %.3e > %.0e at mode %zu row %u col %zu\n",
                   worst, tol, worst_mode, worst_detail.worst_row, worst_detail.worst_col);
  }
  maybe_write_json(opt, report);
  return verify_passed ? exit_ok : exit_verify_failed;
}

template <typename T>
int cmd_gen(const Options& opt) {
  mttkrp::SyntheticSpec spec;
  spec.dims = opt.dims;
  spec.nnz = opt.nnz;
  spec.dist = opt.dist == "skewed" ? mttkrp::SyntheticDist::mode_skewed
                                   : mttkrp::SyntheticDist::uniform;
  spec.skew_mode = opt.skew_mode;
  spec.skew_distinct = opt.skew_distinct;
  spec.seed = opt.seed;
  auto tensor = mttkrp::generate_synthetic<T>(spec);
  const bool binary = opt.out_path.size() >= 5 &&
                      opt.out_path.compare(opt.out_path.size() - 5, 5, ".mkbt") == 0;
  if (binary) mttkrp::save_tensor_cache(tensor, opt.out_path);
  else mttkrp::write_frostt_file(tensor, opt.out_path);

  std::printf("wrote %zu elements", tensor.nnz());
  std::printf(" shape");
  for (auto e : tensor.shape().dims) std::printf(" %u", e);
  std::printf(" -> %s\n", opt.out_path.c_str());

  Json report = Json::object();
  report["command"] = "gen";
  report["out"] = opt.out_path;
  report["shape"] = tensor.shape().dims;
  report["nnz"] = tensor.nnz();
  report["dist"] = opt.dist;
  report["seed"] = opt.seed;
  maybe_write_json(opt, report);
  return exit_ok;
}

template <typename T>
int cmd_inspect(const Options& opt) {
  Json report = Json::object();
  report["command"] = "inspect";
  auto tensor = load_tensor<T>(opt, report);
  const std::size_t kappa = opt.kappa ? opt.kappa : detect_kappa();
  const auto strategy = parse_strategy(opt.strategy);
  report["kappa"] = kappa;
  report["rank"] = opt.rank;
  report["precision"] = opt.precision;

  std::printf("tensor %s\n", opt.tensor_path.c_str());
  std::printf("  modes: %zu  shape:", tensor.mode_count());
  for (auto e : tensor.shape().dims) std::printf(" %u", e);
  std::printf("  nnz: %zu\n", tensor.nnz());

  auto plans = mttkrp::build_mode_plans(tensor, kappa, strategy, mttkrp::SchemePolicy::adaptive);
  Json modes = Json::array();
  for (std::size_t d = 0; d < plans.size(); ++d) {
    auto profile = mttkrp::plan_degrees(tensor, plans[d]);
    auto bm = mttkrp::balance_metrics(plans[d], profile);
    std::printf("  mode %zu: extent %u, distinct %zu -> %s, max/mean %.3f, empty %zu\n", d,
                tensor.extent(d), profile.distinct(),
                std::string(mttkrp::to_string(plans[d].scheme)).c_str(), bm.max_over_mean,
                bm.empty_partitions);
    Json m = to_json(bm);
    m["extent"] = tensor.extent(d);
    m["distinct_indices"] = profile.distinct();
    modes.push_back(std::move(m));
  }
  report["modes"] = std::move(modes);
  const unsigned beta = opt.precision == "f64" ? 64 : 32;
  auto mem = mttkrp::estimate_memory(tensor, opt.rank, beta);
  std::printf("  memory: %llu bits/element, %llu bytes for %zu copies, %llu bytes factors\n",
              static_cast<unsigned long long>(mem.bits_per_element),
              static_cast<unsigned long long>(mem.total_copy_bytes), tensor.mode_count(),
              static_cast<unsigned long long>(mem.factor_matrix_bytes));
  report["memory"] = to_json(mem);
  maybe_write_json(opt, report);
  return exit_ok;
}

// ----------------------------------------------------------------------------- argv
std::uint64_t parse_uint(const std::string& name, const std::string& v, bool positive) {
  std::uint64_t x = 0;
  auto [p, ec] = std::from_chars(v.data(), v.data() + v.size(), x);
  if (ec != std::errc{} || p != v.data() + v.size())
    throw UsageError{name + ": Value " + v + " could not be converted"};
  if (positive && x == 0) throw UsageError{name + ": Value " + v + " not a positive number"};
  return x;
}

void member(const std::string& name, const std::string& v, std::initializer_list<const char*> ok) {
  for (const char* o : ok)
    if (v == o) return;
  throw UsageError{name + ": " + v + " not in {...}"};
}

void usage() {
  std::puts(
      "Sparse MTTKRP benchmark harness with mode-specific tensor layouts (B200 backend)\n"
      "Usage: mttkrp-bench <run|gen|inspect> [options]\n"
      "  run     --tensor F [--rank R] [--kappa K] [--batch P] [--policy adaptive|s1|s2]\n"
      "          [--strategy cyclic|lpt] [--iters N] [--verify] [--deterministic] [--fast]\n"
      "          [--precision f32|f64] [--seed S] [--json PATH] [--cache] [--backend gpu]\n"
      "  gen     --dims A,B,C --nnz M --out F(.tns|.mkbt) [--dist uniform|skewed]\n"
      "          [--skew-mode D] [--skew-distinct K] [--seed S] [--precision f32|f64] [--json PATH]\n"
      "  inspect --tensor F [--rank R] [--kappa K] [--strategy cyclic|lpt] [--precision ..]\n"
      "          [--seed S] [--json PATH] [--cache] [--backend gpu]");
}

enum class Cmd { run, gen, inspect };

Cmd parse_args(int argc, char** argv, Options& opt) {
  if (argc < 2) throw UsageError{"A subcommand is required"};
  const std::string sub = argv[1];
  Cmd cmd;
  if (sub == "run") cmd = Cmd::run;
  else if (sub == "gen") cmd = Cmd::gen;
  else if (sub == "inspect") cmd = Cmd::inspect;
  else throw UsageError{"The following argument was not expected: " + sub};
  bool tensor_set = false, dims_set = false, out_set = false, kappa_set = false;
  for (int i = 2; i < argc; ++i) {
    std::string a = argv[i], v;
    const auto eq = a.find('=');
    if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
      v = a.substr(eq + 1);
      a = a.substr(0, eq);
    }
    auto flag = [&](const char* name) { return a == name; };
    const bool is_flag = flag("--verify") || flag("--deterministic") || flag("--cache") || flag("--fast") ||
                         flag("--help") || flag("-h");
    if (!is_flag && eq == std::string::npos) {
      if (i + 1 >= argc) throw UsageError{a + " requires an argument"};
      v = argv[++i];
    }
    const bool common = cmd != Cmd::gen;
    if (flag("--help") || flag("-h")) {
      usage();
      std::exit(exit_ok);
    } else if (common && flag("--tensor")) {
      opt.tensor_path = v;
      tensor_set = true;
      if (!std::filesystem::exists(v)) throw UsageError{"--tensor: File does not exist: " + v};
    } else if (common && flag("--rank")) {
      opt.rank = parse_uint("--rank", v, true);
    } else if (common && flag("--kappa")) {
      opt.kappa = parse_uint("--kappa", v, true);
      kappa_set = true;
    } else if (flag("--precision")) {
      member("--precision", v, {"f32", "f64"});
      opt.precision = v;
    } else if (flag("--seed")) {
      opt.seed = parse_uint("--seed", v, false);
    } else if (flag("--json")) {
      opt.json_path = v;
    } else if (common && flag("--backend")) {
      member("--backend", v, {"gpu"});
      opt.backend = v;
    } else if (common && flag("--cache")) {
      opt.cache = true;
    } else if (cmd == Cmd::run && flag("--batch")) {
      opt.batch_p = parse_uint("--batch", v, true);
    } else if (cmd == Cmd::run && flag("--policy")) {
      member("--policy", v, {"adaptive", "s1", "s2"});
      opt.policy = v;
    } else if (common && flag("--strategy")) {
      member("--strategy", v, {"cyclic", "lpt"});
      opt.strategy = v;
    } else if (cmd == Cmd::run && flag("--iters")) {
      opt.iters = parse_uint("--iters", v, true);
    } else if (cmd == Cmd::run && flag("--verify")) {
      opt.verify = true;
    } else if (cmd == Cmd::run && flag("--deterministic")) {
      opt.deterministic = true;
    } else if (cmd == Cmd::run && flag("--fast")) {
      opt.fast = true;
    } else if (cmd == Cmd::gen && flag("--dims")) {
      opt.dims.clear();
      std::stringstream ss(v);
      std::string tok;
      while (std::getline(ss, tok, ','))
        opt.dims.push_back(static_cast<mttkrp::index_t>(parse_uint("--dims", tok, false)));
      dims_set = true;
    } else if (cmd == Cmd::gen && flag("--nnz")) {
      opt.nnz = parse_uint("--nnz", v, false);
      opt.nnz_set = true;
    } else if (cmd == Cmd::gen && flag("--dist")) {
      member("--dist", v, {"uniform", "skewed"});
      opt.dist = v;
    } else if (cmd == Cmd::gen && flag("--skew-mode")) {
      opt.skew_mode = parse_uint("--skew-mode", v, false);
    } else if (cmd == Cmd::gen && flag("--skew-distinct")) {
      opt.skew_distinct = parse_uint("--skew-distinct", v, true);
    } else if (cmd == Cmd::gen && flag("--out")) {
      opt.out_path = v;
      out_set = true;
    } else {
      throw UsageError{"The following argument was not expected: " + a};
    }
  }
  if (cmd != Cmd::gen && !tensor_set) throw UsageError{"--tensor is required"};
  if (cmd == Cmd::gen && (!dims_set || !opt.nnz_set || !out_set))
    throw UsageError{"--dims, --nnz and --out are required"};
  if (cmd != Cmd::gen && !kappa_set)  // CLI11 envname (mttkrp_bench.cpp:284)
    if (const char* w = std::getenv("SPMTTKRP_WORKERS"))
      opt.kappa = parse_uint("SPMTTKRP_WORKERS", w, true);
  return cmd;
}

template <int (*Fn32)(const Options&), int (*Fn64)(const Options&)>
int dispatch(const Options& opt) {
  if (opt.precision == "f64") return Fn64(opt);
  return Fn32(opt);
}

}  // namespace

int main(int argc, char** argv) {
  Options opt;
  Cmd cmd;
  try {
    cmd = parse_args(argc, argv, opt);
  } catch (const UsageError& e) {
    std::fprintf(stderr, "%s\nRun with --help for more information.\n", e.msg.c_str());
    return exit_usage;
  }
  try {
    switch (cmd) {
      case Cmd::run: return dispatch<cmd_run<float>, cmd_run<double>>(opt);
      case Cmd::gen: return dispatch<cmd_gen<float>, cmd_gen<double>>(opt);
      case Cmd::inspect: return dispatch<cmd_inspect<float>, cmd_inspect<double>>(opt);
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    if (!opt.json_path.empty()) {
      try {
        Json j = Json::object();
        j["error"] = e.what();
        write_json_file(opt.json_path, j);
      } catch (...) {
      }
    }
    return exit_error;
  }
  return exit_error;
}
