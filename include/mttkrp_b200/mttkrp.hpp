// mttkrp_b200/mttkrp.hpp — C++ drop-in for the reference's `mttkrp` core API
// (/root/reference/proj/core/include/mttkrp), running the hot path on a B200 through the
// C ABI of include/mttkrp_b200.h.
//
// Migration: replace `#include "mttkrp/kernel.hpp"` (and layout/factor/tensor/synthetic)
// with `#include "mttkrp_b200/mttkrp.hpp"` and `namespace mttkrp = mttkrp_b200;`.  Names,
// argument meaning, return types and exception messages follow the reference:
//
//   SparseTensorCOO<float>            tensor.hpp:34-111 (host storage, same validation)
//   FactorMatrix<float>, random_factors   factor.hpp:16-84
//   generate_synthetic, SyntheticSpec synthetic.hpp:20-158 (bit-identical, host C++)
//   ModePlan, build_mode_plans, partition_scheme1/2, mode_degrees, select_scheme
//                                     layout.hpp:17-149 — built on the GPU, bit-exact
//   ExecConfig, mttkrp_mode, mttkrp_all_modes, run_timed, element_update
//                                     kernel.hpp:23-287 — spMTTKRP on the GPU
//   cpd_als                           (absent in the reference)
//
// T = float runs the fast fp32 kernels; T = double (the reference's fp64 instantiation,
// SURVEY §8 f-4) runs the fp64 device path (mk_*_f64; deterministic = oracle_mttkrp<double>
// bitwise).  A ModePlan keeps a handle to the device session that owns the uploaded tensor
// and its mode copies; plans of one build_mode_plans call share it, and every call gets its
// own session.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <initializer_list>
#include <memory>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <type_traits>
#include <utility>
#include <vector>

#include "mttkrp_b200.h"

namespace mttkrp_b200 {

using index_t = std::uint32_t;

class error : public std::runtime_error {
 public:
  explicit error(const std::string& what) : std::runtime_error(what) {}
};

namespace detail {
inline void check(int rc) {
  if (rc != MK_OK) throw error(mk_last_error());
}
}  // namespace detail

struct Shape {
  std::vector<index_t> dims;
  Shape() = default;
  explicit Shape(std::vector<index_t> d) : dims(std::move(d)) { validate(); }
  std::size_t mode_count() const { return dims.size(); }
  index_t extent(std::size_t d) const { return dims[d]; }
  std::uint64_t capacity() const {  // types.hpp:38-46, saturating
    std::uint64_t cap = 1;
    for (index_t e : dims) {
      if (e != 0 && cap > UINT64_MAX / e) return UINT64_MAX;
      cap *= e;
    }
    return cap;
  }
  void validate() const {
    if (dims.empty()) throw error("shape: a tensor needs at least one mode");
    for (index_t e : dims)
      if (e == 0) throw error("shape: zero extent");
  }
  bool operator==(const Shape&) const = default;
};

template <typename T>
class SparseTensorCOO {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>,
                "the device path computes in fp32 or fp64");

 public:
  using value_type = T;
  explicit SparseTensorCOO(Shape shape) : shape_(std::move(shape)) {}
  static SparseTensorCOO from_parts(Shape shape, std::vector<index_t> coords,
                                    std::vector<T> values) {
    SparseTensorCOO t(std::move(shape));
    const std::size_t n = t.mode_count();
    if (values.empty() ? !coords.empty() : coords.size() != values.size() * n)
      throw error("tensor: coordinate/value storage size mismatch");
    t.coords_ = std::move(coords);
    t.values_ = std::move(values);
    for (std::size_t i = 0; i < t.nnz(); ++i) t.check_element(t.coords(i), t.values_[i]);
    return t;
  }
  const Shape& shape() const { return shape_; }
  std::size_t mode_count() const { return shape_.mode_count(); }
  index_t extent(std::size_t d) const { return shape_.extent(d); }
  std::size_t nnz() const { return values_.size(); }
  void add(std::span<const index_t> c, T v) {
    check_element(c, v);
    coords_.insert(coords_.end(), c.begin(), c.end());
    values_.push_back(v);
  }
  void add(std::initializer_list<index_t> c, T v) {
    add(std::span<const index_t>(c.begin(), c.size()), v);
  }
  std::span<const index_t> coords(std::size_t i) const {
    return {coords_.data() + i * mode_count(), mode_count()};
  }
  index_t index(std::size_t i, std::size_t mode) const { return coords_[i * mode_count() + mode]; }
  T value(std::size_t i) const { return values_[i]; }
  std::span<const T> values() const { return values_; }
  const index_t* coord_data() const { return coords_.data(); }
  std::vector<index_t> mode_column(std::size_t d) const {
    if (d >= mode_count()) throw error("tensor: mode out of range");
    std::vector<index_t> col(nnz());
    for (std::size_t i = 0; i < col.size(); ++i) col[i] = index(i, d);
    return col;
  }
  bool operator==(const SparseTensorCOO& o) const {
    return shape_ == o.shape_ && coords_ == o.coords_ && values_ == o.values_;
  }

 private:
  void check_element(std::span<const index_t> c, T v) const {
    if (c.size() != mode_count()) throw error("tensor: element has wrong number of coordinates");
    for (std::size_t h = 0; h < c.size(); ++h)
      if (c[h] >= shape_.dims[h])
        throw error("tensor: coordinate " + std::to_string(c[h]) + " out of range for mode " +
                    std::to_string(h));
    if (!std::isfinite(static_cast<double>(v))) throw error("tensor: non-finite element value");
  }
  Shape shape_;
  std::vector<index_t> coords_;
  std::vector<T> values_;
};

// tensor.hpp:115-131: order-insensitive equality of two tensors as <indices, value> sets
template <typename T>
bool same_element_set(const SparseTensorCOO<T>& a, const SparseTensorCOO<T>& b) {
  if (!(a.shape() == b.shape()) || a.nnz() != b.nnz()) return false;
  auto sorted = [](const SparseTensorCOO<T>& t) {
    std::vector<std::pair<std::vector<index_t>, T>> v;
    v.reserve(t.nnz());
    for (std::size_t i = 0; i < t.nnz(); ++i) {
      auto c = t.coords(i);
      v.emplace_back(std::vector<index_t>(c.begin(), c.end()), t.value(i));
    }
    std::sort(v.begin(), v.end());
    return v;
  };
  return sorted(a) == sorted(b);
}

template <typename T>
struct FactorMatrix {
  std::size_t mode = 0;
  index_t rows = 0;
  std::size_t rank = 0;
  std::vector<T> data;
  static FactorMatrix zeros(std::size_t mode, index_t rows, std::size_t rank) {
    FactorMatrix m;
    m.mode = mode;
    m.rows = rows;
    m.rank = rank;
    m.data.assign(static_cast<std::size_t>(rows) * rank, T{0});
    return m;
  }
  std::span<T> row(index_t i) { return {data.data() + static_cast<std::size_t>(i) * rank, rank}; }
  std::span<const T> row(index_t i) const {
    return {data.data() + static_cast<std::size_t>(i) * rank, rank};
  }
  T& at(index_t i, std::size_t r) { return data[static_cast<std::size_t>(i) * rank + r]; }
  T at(index_t i, std::size_t r) const { return data[static_cast<std::size_t>(i) * rank + r]; }
  bool operator==(const FactorMatrix&) const = default;
};

// verify.hpp:15-45: |got - want| / max(1, |want|), worst entry
struct VerifyResult {
  double max_rel_err = 0.0;
  index_t worst_row = 0;
  std::size_t worst_col = 0;
};

template <typename T>
VerifyResult verify_against(const FactorMatrix<T>& got, const FactorMatrix<T>& want) {
  if (got.rows != want.rows || got.rank != want.rank) throw error("verify: matrix shapes differ");
  VerifyResult res;
  for (index_t i = 0; i < got.rows; ++i)
    for (std::size_t r = 0; r < got.rank; ++r) {
      const double g = static_cast<double>(got.at(i, r)), w = static_cast<double>(want.at(i, r));
      const double err = std::abs(g - w) / std::max(1.0, std::abs(w));
      if (err > res.max_rel_err) {
        res.max_rel_err = err;
        res.worst_row = i;
        res.worst_col = r;
      }
    }
  return res;
}

template <typename T>
constexpr double verify_tolerance() {
  return sizeof(T) == 4 ? 1e-5 : 1e-12;
}

template <typename T>
bool bitwise_equal(const FactorMatrix<T>& a, const FactorMatrix<T>& b) {
  return a.mode == b.mode && a.rows == b.rows && a.rank == b.rank &&
         a.data.size() == b.data.size() &&
         (a.data.empty() || std::memcmp(a.data.data(), b.data.data(), a.data.size() * sizeof(T)) == 0);
}
template <typename T>
bool bitwise_equal(const std::vector<FactorMatrix<T>>& a, const std::vector<FactorMatrix<T>>& b) {
  if (a.size() != b.size()) return false;
  for (std::size_t i = 0; i < a.size(); ++i)
    if (!bitwise_equal(a[i], b[i])) return false;
  return true;
}

template <typename T>
std::vector<FactorMatrix<T>> random_factors(const Shape& shape, std::size_t rank,
                                            std::uint64_t seed) {
  if (rank < 1) throw error("factor: rank must be at least 1");
  std::vector<FactorMatrix<T>> out;
  std::vector<T*> ptrs;
  for (std::size_t d = 0; d < shape.mode_count(); ++d)
    out.push_back(FactorMatrix<T>::zeros(d, shape.extent(d), rank));
  for (auto& m : out) ptrs.push_back(m.data.data());
  if constexpr (std::is_same_v<T, double>)
    detail::check(mk_random_factors_f64(static_cast<uint32_t>(shape.mode_count()),
                                        shape.dims.data(), rank, seed, ptrs.data()));
  else
    detail::check(mk_random_factors(static_cast<uint32_t>(shape.mode_count()), shape.dims.data(),
                                    rank, seed, ptrs.data()));
  return out;
}

// rng.hpp:12-39: the reference's public random primitives (test support uses them).
namespace rng {
using engine = std::mt19937_64;
inline std::uint64_t splitmix64(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
inline engine seeded(std::uint64_t seed, std::uint64_t stream = 0) {
  return engine(splitmix64(seed ^ splitmix64(stream)));
}
inline std::uint64_t bounded(engine& g, std::uint64_t n) {  // rejects the low (2^64 mod n)
  const std::uint64_t low = (0 - n) % n;
  std::uint64_t x = g();
  while (x < low) x = g();
  return x % n;
}
template <typename T>
inline T unit_open_closed(engine& g) {
  return static_cast<T>(1.0 - static_cast<double>(g() >> 11) * 0x1.0p-53);
}
}  // namespace rng

enum class SyntheticDist { uniform, mode_skewed };
struct SyntheticSpec {
  std::vector<index_t> dims;
  std::size_t nnz = 0;
  SyntheticDist dist = SyntheticDist::uniform;
  std::size_t skew_mode = 0;
  std::size_t skew_distinct = 2;
  std::uint64_t seed = 0;
};

template <typename T = float>
SparseTensorCOO<T> generate_synthetic(const SyntheticSpec& spec) {
  Shape shape(spec.dims);
  std::vector<index_t> coords(spec.nnz * shape.mode_count());
  std::vector<T> values(spec.nnz);
  auto gen = [&](auto fn) {
    detail::check(fn(static_cast<uint32_t>(shape.mode_count()), spec.dims.data(), spec.nnz,
                     spec.dist == SyntheticDist::uniform ? 0 : 1, spec.skew_mode,
                     spec.skew_distinct, spec.seed, coords.data(), values.data()));
  };
  if constexpr (std::is_same_v<T, double>)
    gen(mk_generate_synthetic_f64);
  else
    gen(mk_generate_synthetic);
  return SparseTensorCOO<T>::from_parts(std::move(shape), std::move(coords), std::move(values));
}

enum class Scheme { scheme1, scheme2 };
enum class Strategy { cyclic, least_loaded };
enum class SchemePolicy { adaptive, scheme1_only, scheme2_only };

inline Scheme select_scheme(std::uint64_t index_count, std::size_t kappa) {  // layout.cpp:25-28
  if (kappa < 1) throw error("layout: kappa must be at least 1");
  return index_count >= kappa ? Scheme::scheme1 : Scheme::scheme2;
}

namespace detail {
// Device session: one mk_context holding one uploaded tensor and its N mode copies.
struct Session {
  mk_context* ctx = nullptr;
  const void* tensor = nullptr;
  std::size_t nnz = 0;
  std::size_t rank = 0;
  explicit Session(int device = 0) { check(mk_create(device, &ctx)); }
  ~Session() {
    if (ctx) mk_destroy(ctx);
  }
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;
};
}  // namespace detail

struct ModePlan {
  std::size_t mode = 0;
  Scheme scheme = Scheme::scheme1;
  std::size_t kappa = 1;
  std::vector<std::uint64_t> order;
  std::vector<std::uint64_t> partition_offsets;
  std::vector<std::vector<index_t>> owned_indices;
  std::shared_ptr<detail::Session> device;  // the GPU copy this plan describes
  std::size_t nnz() const { return order.size(); }
  std::uint64_t partition_size(std::size_t z) const {
    return partition_offsets[z + 1] - partition_offsets[z];
  }
};

struct DegreeProfile {
  std::size_t mode = 0;
  std::vector<std::uint64_t> degrees;
  std::uint64_t total = 0;
  std::size_t distinct() const {
    std::size_t c = 0;
    for (auto d : degrees) c += d > 0;
    return c;
  }
};

namespace detail {
template <typename T>
std::shared_ptr<Session> upload(const SparseTensorCOO<T>& t) {
  auto s = std::make_shared<Session>();
  if constexpr (std::is_same_v<T, double>)
    check(mk_tensor_upload_f64(s->ctx, static_cast<uint32_t>(t.mode_count()),
                               t.shape().dims.data(), t.nnz(), t.coord_data(), t.values().data()));
  else
    check(mk_tensor_upload(s->ctx, static_cast<uint32_t>(t.mode_count()), t.shape().dims.data(),
                           t.nnz(), t.coord_data(), t.values().data()));
  s->tensor = &t;
  s->nnz = t.nnz();
  return s;
}

inline ModePlan export_plan(const std::shared_ptr<Session>& s, std::size_t mode) {
  mk_plan_info info{};
  check(mk_get_plan_info(s->ctx, static_cast<uint32_t>(mode), &info));
  ModePlan p;
  p.mode = mode;
  p.scheme = info.scheme == MK_SCHEME1 ? Scheme::scheme1 : Scheme::scheme2;
  p.kappa = info.kappa;
  p.order.resize(info.nnz);
  p.partition_offsets.resize(info.kappa + 1);
  std::vector<uint32_t> owned(info.owned_total);
  std::vector<uint64_t> owned_off(info.kappa + 1);
  check(mk_plan_export(s->ctx, static_cast<uint32_t>(mode), p.order.data(),
                       p.partition_offsets.data(), owned.data(), owned_off.data()));
  if (p.scheme == Scheme::scheme1) {
    p.owned_indices.resize(info.kappa);
    for (std::size_t z = 0; z < info.kappa; ++z)
      p.owned_indices[z].assign(owned.begin() + owned_off[z], owned.begin() + owned_off[z + 1]);
  }
  p.device = s;
  return p;
}

inline int policy_code(SchemePolicy p) {
  return p == SchemePolicy::scheme1_only ? MK_SCHEME1_ONLY
                                         : (p == SchemePolicy::scheme2_only ? MK_SCHEME2_ONLY
                                                                            : MK_ADAPTIVE);
}
}  // namespace detail

// layout.hpp:131-149 — the N mode-specific copies, built and kept on the device.
template <typename T>
std::vector<ModePlan> build_mode_plans(const SparseTensorCOO<T>& t, std::size_t kappa,
                                       Strategy strategy = Strategy::cyclic,
                                       SchemePolicy policy = SchemePolicy::adaptive) {
  if (kappa < 1) throw error("layout: kappa must be at least 1");
  auto s = detail::upload(t);
  detail::check(mk_build_plans(s->ctx, kappa,
                               strategy == Strategy::cyclic ? MK_CYCLIC : MK_LEAST_LOADED,
                               detail::policy_code(policy)));
  std::vector<ModePlan> plans;
  for (std::size_t d = 0; d < t.mode_count(); ++d) plans.push_back(detail::export_plan(s, d));
  return plans;
}

template <typename T>
ModePlan partition_scheme1(const SparseTensorCOO<T>& t, std::size_t d, std::size_t kappa,
                           Strategy strategy = Strategy::cyclic) {
  if (d >= t.mode_count()) throw error("layout: mode out of range");
  return build_mode_plans(t, kappa, strategy, SchemePolicy::scheme1_only).at(d);
}

template <typename T>
ModePlan partition_scheme2(const SparseTensorCOO<T>& t, std::size_t d, std::size_t kappa) {
  if (d >= t.mode_count()) throw error("layout: mode out of range");
  return build_mode_plans(t, kappa, Strategy::cyclic, SchemePolicy::scheme2_only).at(d);
}

template <typename T>
DegreeProfile mode_degrees(const SparseTensorCOO<T>& t, std::size_t d) {
  if (d >= t.mode_count()) throw error("layout: mode out of range");
  auto s = detail::upload(t);
  detail::check(mk_build_plans(s->ctx, 1, MK_CYCLIC, MK_SCHEME2_ONLY));
  DegreeProfile p;
  p.mode = d;
  p.degrees.resize(t.extent(d));
  detail::check(mk_mode_degrees(s->ctx, static_cast<uint32_t>(d), p.degrees.data()));
  p.total = t.nnz();
  return p;
}

inline std::string_view to_string(Scheme s) {  // layout.cpp:9-11
  return s == Scheme::scheme1 ? "scheme1" : "scheme2";
}
inline std::string_view to_string(Strategy s) {  // layout.cpp:13-15
  return s == Strategy::cyclic ? "cyclic" : "least_loaded";
}
inline std::string_view to_string(SchemePolicy p) {  // layout.cpp:17-23
  return p == SchemePolicy::scheme1_only ? "s1-only"
                                         : (p == SchemePolicy::scheme2_only ? "s2-only" : "adaptive");
}

// types.hpp:50-55: ceil(log2(extent)) with a 1-bit floor
inline std::uint64_t index_bits(index_t extent) {
  if (extent <= 2) return 1;
  std::uint64_t v = static_cast<std::uint64_t>(extent) - 1, b = 0;
  while (v) {
    ++b;
    v >>= 1;
  }
  return b;
}

// layout.hpp:66-86 — host-side report structs (no device work involved)
struct MemoryEstimate {
  std::uint64_t bits_per_element = 0;
  std::uint64_t total_copy_bits = 0;
  std::uint64_t total_copy_bytes = 0;
  std::uint64_t factor_matrix_bytes = 0;
  std::uint64_t storage_bytes_actual = 0;
};

struct BalanceMetrics {
  std::size_t mode = 0;
  Scheme scheme = Scheme::scheme1;
  std::size_t kappa = 1;
  std::vector<std::uint64_t> loads;
  std::vector<std::uint64_t> owned_index_counts;
  double max_over_mean = 1.0;
  std::size_t empty_partitions = 0;
};

// layout.cpp:30-48
inline MemoryEstimate estimate_memory_for(const Shape& shape, std::size_t nnz, std::size_t rank,
                                          unsigned beta_float_bits) {
  if (rank < 1) throw error("layout: rank must be at least 1");
  if (beta_float_bits != 32 && beta_float_bits != 64)
    throw error("layout: value width must be 32 or 64 bits");
  MemoryEstimate m;
  for (index_t e : shape.dims) m.bits_per_element += index_bits(e);
  m.bits_per_element += beta_float_bits;
  const std::uint64_t n = shape.mode_count();
  m.total_copy_bits = n * static_cast<std::uint64_t>(nnz) * m.bits_per_element;
  m.total_copy_bytes = (m.total_copy_bits + 7) / 8;
  for (index_t e : shape.dims)
    m.factor_matrix_bytes += static_cast<std::uint64_t>(e) * rank * (beta_float_bits / 8);
  m.storage_bytes_actual =
      n * static_cast<std::uint64_t>(nnz) * (n * sizeof(index_t) + beta_float_bits / 8);
  return m;
}

template <typename T>
MemoryEstimate estimate_memory(const SparseTensorCOO<T>& t, std::size_t rank,
                               unsigned beta_float_bits = sizeof(T) * 8) {  // layout.hpp:151-155
  return estimate_memory_for(t.shape(), t.nnz(), rank, beta_float_bits);
}

// layout.cpp:50-72
inline BalanceMetrics balance_metrics(const ModePlan& plan, const DegreeProfile& profile) {
  if (plan.mode != profile.mode)
    throw error("layout: plan and degree profile describe different modes");
  if (plan.nnz() != profile.total)
    throw error("layout: plan and degree profile describe different tensors");
  BalanceMetrics bm;
  bm.mode = plan.mode;
  bm.scheme = plan.scheme;
  bm.kappa = plan.kappa;
  for (std::size_t z = 0; z < plan.kappa; ++z) {
    const std::uint64_t load = plan.partition_size(z);
    bm.loads.push_back(load);
    bm.empty_partitions += load == 0;
  }
  for (const auto& owned : plan.owned_indices) bm.owned_index_counts.push_back(owned.size());
  const std::uint64_t max_load =
      bm.loads.empty() ? 0 : *std::max_element(bm.loads.begin(), bm.loads.end());
  const double mean = static_cast<double>(plan.nnz()) / static_cast<double>(plan.kappa);
  bm.max_over_mean = plan.nnz() == 0 ? 1.0 : static_cast<double>(max_load) / mean;
  return bm;
}

// mode_degrees read from a plan's own device copy (no second upload of the tensor)
template <typename T>
DegreeProfile plan_degrees(const SparseTensorCOO<T>& t, const ModePlan& plan) {
  DegreeProfile p;
  p.mode = plan.mode;
  p.degrees.resize(t.extent(plan.mode));
  detail::check(mk_mode_degrees(plan.device->ctx, static_cast<uint32_t>(plan.mode), p.degrees.data()));
  p.total = plan.nnz();
  return p;
}

struct ExecConfig {
  std::size_t kappa = 1;
  std::size_t batch_p = 32;
  bool deterministic = false;
  bool partitioned = false;  // MK_EXEC_PARTITIONED: the reference's partition-per-worker split
  // Extension (no reference counterpart).  false: the reference's parallel-executor contract,
  // MK_EXEC_REFERENCE (Scheme 1 modes bitwise equal to deterministic);
  // true: the B200 fast path, MK_EXEC_FAST (level-ordered kernels, within 1e-4 of the oracle).
  bool fast = false;
  int exec_code() const {
    if (deterministic) return MK_EXEC_DETERMINISTIC;
    if (partitioned) return MK_EXEC_PARTITIONED;
    return fast ? MK_EXEC_FAST : MK_EXEC_REFERENCE;
  }
  // the fp64 device path has no partitioned executor
  int exec_code64() const {
    return partitioned && !deterministic ? (fast ? MK_EXEC_FAST : MK_EXEC_REFERENCE) : exec_code();
  }
  void validate() const {
    if (kappa < 1) throw error("kernel: kappa must be at least 1");
    if (batch_p < 1) throw error("kernel: batch size P must be at least 1");
  }
};

namespace detail {
template <typename T>
void validate_factors(const SparseTensorCOO<T>& t, const std::vector<FactorMatrix<T>>& f) {
  if (f.size() != t.mode_count()) throw error("kernel: expected one factor matrix per mode");
  const std::size_t rank = f.empty() ? 0 : f[0].rank;
  if (rank < 1) throw error("kernel: rank must be at least 1");
  for (std::size_t w = 0; w < f.size(); ++w) {
    if (f[w].mode != w)
      throw error("kernel: factor matrix " + std::to_string(w) + " labeled mode " +
                  std::to_string(f[w].mode));
    if (f[w].rows != t.extent(w))
      throw error("kernel: factor matrix " + std::to_string(w) + " has " +
                  std::to_string(f[w].rows) + " rows, tensor extent is " +
                  std::to_string(t.extent(w)));
    if (f[w].rank != rank) throw error("kernel: factor matrices disagree on rank");
  }
}

template <typename T>
void validate_plan(const SparseTensorCOO<T>& t, const ModePlan& plan, const ExecConfig& config) {
  if (plan.mode >= t.mode_count()) throw error("kernel: plan mode out of range");
  if (plan.nnz() != t.nnz() || !plan.device || plan.device->tensor != &t ||
      plan.device->nnz != t.nnz())
    throw error("kernel: plan does not cover this tensor");
  if (plan.partition_offsets.size() != plan.kappa + 1 || plan.partition_offsets.front() != 0 ||
      plan.partition_offsets.back() != t.nnz())
    throw error("kernel: malformed partition offsets");
  if (plan.kappa != config.kappa)
    throw error("kernel: plan built for kappa " + std::to_string(plan.kappa) +
                ", config requests " + std::to_string(config.kappa));
}

template <typename T>
void upload_factors(Session& s, const std::vector<FactorMatrix<T>>& f) {
  std::vector<const T*> p;
  for (auto& m : f) p.push_back(m.data.data());
  if constexpr (std::is_same_v<T, double>)
    check(mk_factors_upload_f64(s.ctx, static_cast<uint32_t>(f[0].rank), p.data()));
  else
    check(mk_factors_upload(s.ctx, static_cast<uint32_t>(f[0].rank), p.data()));
  s.rank = f[0].rank;
}

template <typename T>
int mode_call(mk_context* ctx, uint32_t mode, int exec, T* out) {
  if constexpr (std::is_same_v<T, double>)
    return mk_mttkrp_mode_f64(ctx, mode, exec, out);
  else
    return mk_mttkrp_mode(ctx, mode, exec, out);
}
}  // namespace detail

// kernel.hpp:133-155 (host arithmetic; API parity)
template <typename T>
void element_update(std::span<const index_t> coords, T value,
                    const std::vector<FactorMatrix<T>>& factors, std::size_t output_mode,
                    std::span<T> acc) {
  const std::size_t rank = acc.size();
  for (const auto& f : factors)
    if (f.rank != rank) throw error("kernel: factor matrices disagree on rank");
  for (std::size_t r = 0; r < rank; ++r) acc[r] = value;
  for (std::size_t w = 0; w < factors.size(); ++w) {
    if (w == output_mode) continue;
    auto vec = factors[w].row(coords[w]);
    for (std::size_t r = 0; r < rank; ++r) acc[r] *= vec[r];
  }
}

template <typename T>
std::vector<T> element_update(const SparseTensorCOO<T>& t, std::size_t element,
                              const std::vector<FactorMatrix<T>>& factors,
                              std::size_t output_mode) {  // kernel.hpp:145-153
  std::vector<T> acc(factors.empty() ? 0 : factors[0].rank);
  element_update<T>(t.coords(element), t.value(element), factors, output_mode, acc);
  return acc;
}

// Extension (no reference counterpart): how the fast path picks its plan for the tensor the
// plans were built from.  timed (default): candidates timed on the first fast call of each
// mode; model: the cost model's plan, no timing, the same on every run and box.
enum class PlanMode { timed = MK_PLAN_TIMED, model = MK_PLAN_MODEL };
inline void set_plan_mode(const std::vector<ModePlan>& plans, PlanMode mode) {
  if (plans.empty()) throw error("kernel: expected one plan per mode");
  detail::check(mk_set_plan_mode(plans[0].device->ctx, static_cast<int>(mode)));
}

// kernel.hpp:161-169 on the device.
template <typename T>
FactorMatrix<T> mttkrp_mode(const SparseTensorCOO<T>& t, const ModePlan& plan,
                            const std::vector<FactorMatrix<T>>& factors, const ExecConfig& config) {
  config.validate();
  detail::validate_factors(t, factors);
  detail::validate_plan(t, plan, config);
  detail::upload_factors(*plan.device, factors);
  auto out = FactorMatrix<T>::zeros(plan.mode, t.extent(plan.mode), factors[0].rank);
  detail::check(detail::mode_call<T>(
      plan.device->ctx, static_cast<uint32_t>(plan.mode),
      std::is_same_v<T, double> ? config.exec_code64() : config.exec_code(),
      out.data.data()));
  return out;
}

// kernel.hpp:177-197 on the device.
template <typename T>
std::vector<FactorMatrix<T>> mttkrp_all_modes(const SparseTensorCOO<T>& t,
                                              const std::vector<ModePlan>& plans,
                                              const std::vector<FactorMatrix<T>>& factors,
                                              const ExecConfig& config, bool chain_outputs) {
  if (plans.size() != t.mode_count()) throw error("kernel: expected one plan per mode");
  for (std::size_t d = 0; d < plans.size(); ++d)
    if (plans[d].mode != d) throw error("kernel: plans out of mode order");
  config.validate();
  detail::validate_factors(t, factors);
  for (const auto& p : plans) detail::validate_plan(t, p, config);
  detail::upload_factors(*plans[0].device, factors);
  std::vector<FactorMatrix<T>> outs;
  std::vector<T*> ptr;
  for (std::size_t d = 0; d < plans.size(); ++d)
    outs.push_back(FactorMatrix<T>::zeros(d, t.extent(d), factors[0].rank));
  for (auto& o : outs) ptr.push_back(o.data.data());
  const int exec = std::is_same_v<T, double> ? config.exec_code64() : config.exec_code();
  if constexpr (std::is_same_v<T, double>)
    detail::check(mk_mttkrp_all_modes_f64(plans[0].device->ctx, chain_outputs ? 1 : 0, exec,
                                          ptr.data()));
  else
    detail::check(mk_mttkrp_all_modes(plans[0].device->ctx, chain_outputs ? 1 : 0, exec,
                                      ptr.data()));
  return outs;
}

struct ModeTiming {
  std::size_t mode = 0;
  Scheme scheme = Scheme::scheme1;
  std::vector<double> wall_ms;
  double min_ms = 0;
  double median_ms = 0;
  std::size_t busy_workers = 0;
  std::vector<std::uint64_t> elements_per_worker;
};

struct TimingReport {
  std::size_t iters = 0;
  std::vector<ModeTiming> modes;
  std::vector<double> total_ms;
  double total_min_ms = 0;
  double total_median_ms = 0;
  bool outputs_bit_identical = true;
};

template <typename T>
struct TimedRun {
  TimingReport report;
  std::vector<FactorMatrix<T>> outputs;
};

namespace detail {
inline double median_of(std::vector<double> v) {
  if (v.empty()) return 0;
  std::sort(v.begin(), v.end());
  const std::size_t mid = v.size() / 2;
  return v.size() % 2 ? v[mid] : 0.5 * (v[mid - 1] + v[mid]);
}
}  // namespace detail

// kernel.hpp:239-287: per-mode device time from CUDA events, L2 flushed between iterations.
template <typename T>
TimedRun<T> run_timed(const SparseTensorCOO<T>& t, const std::vector<ModePlan>& plans,
                      const std::vector<FactorMatrix<T>>& factors, const ExecConfig& config,
                      std::size_t iters) {
  if (iters < 1) throw error("kernel: iters must be at least 1");
  config.validate();
  detail::validate_factors(t, factors);
  for (const auto& p : plans) detail::validate_plan(t, p, config);
  detail::upload_factors(*plans[0].device, factors);
  const std::size_t n = plans.size();
  std::vector<double> mode_ms(iters * n), total(iters);
  int same = 1;
  if constexpr (std::is_same_v<T, double>) {
    // fp64: host-timed per-mode calls as in the reference (steady_clock around each mode,
    // kernel.hpp:258-265), outputs compared bitwise across iterations
    TimedRun<T> run;
    run.report.iters = iters;
    std::vector<ModeTiming> modes(n);
    for (std::size_t it = 0; it < iters; ++it) {
      std::vector<FactorMatrix<T>> outs;
      double tot = 0;
      for (std::size_t d = 0; d < n; ++d) {
        auto o = FactorMatrix<T>::zeros(d, t.extent(d), factors[0].rank);
        const auto t0 = std::chrono::steady_clock::now();
        detail::check(mk_mttkrp_mode_f64(plans[0].device->ctx, static_cast<uint32_t>(d),
                                         config.exec_code64(),
                                         o.data.data()));
        const double ms = std::chrono::duration<double, std::milli>(
                              std::chrono::steady_clock::now() - t0).count();
        modes[d].wall_ms.push_back(ms);
        tot += ms;
        outs.push_back(std::move(o));
      }
      run.report.total_ms.push_back(tot);
      if (it == 0)
        run.outputs = std::move(outs);
      else if (!bitwise_equal(outs, run.outputs))
        run.report.outputs_bit_identical = false;
    }
    for (std::size_t d = 0; d < n; ++d) {
      ModeTiming& mt = modes[d];
      mt.mode = d;
      mt.scheme = plans[d].scheme;
      mt.min_ms = *std::min_element(mt.wall_ms.begin(), mt.wall_ms.end());
      mt.median_ms = detail::median_of(mt.wall_ms);
      for (std::size_t z = 0; z < plans[d].kappa; ++z) {
        mt.elements_per_worker.push_back(plans[d].partition_size(z));
        mt.busy_workers += plans[d].partition_size(z) > 0;
      }
    }
    run.report.modes = std::move(modes);
    run.report.total_min_ms = *std::min_element(run.report.total_ms.begin(), run.report.total_ms.end());
    run.report.total_median_ms = detail::median_of(run.report.total_ms);
    return run;
  } else {
  detail::check(mk_run_timed(plans[0].device->ctx, iters,
                             config.exec_code(), 1,
                             mode_ms.data(), total.data(), &same));
  TimedRun<T> run;
  run.report.iters = iters;
  run.report.outputs_bit_identical = same != 0;
  run.report.total_ms = total;
  for (std::size_t d = 0; d < n; ++d) {
    ModeTiming mt;
    mt.mode = d;
    mt.scheme = plans[d].scheme;
    for (std::size_t it = 0; it < iters; ++it) mt.wall_ms.push_back(mode_ms[it * n + d]);
    mt.min_ms = *std::min_element(mt.wall_ms.begin(), mt.wall_ms.end());
    mt.median_ms = detail::median_of(mt.wall_ms);
    for (std::size_t z = 0; z < plans[d].kappa; ++z) {
      mt.elements_per_worker.push_back(plans[d].partition_size(z));
      mt.busy_workers += plans[d].partition_size(z) > 0;
    }
    run.report.modes.push_back(std::move(mt));
  }
  run.report.total_min_ms = *std::min_element(total.begin(), total.end());
  run.report.total_median_ms = detail::median_of(total);
  for (std::size_t d = 0; d < n; ++d) {
    auto o = FactorMatrix<T>::zeros(d, t.extent(d), factors[0].rank);
    detail::check(mk_output_download(plans[0].device->ctx, static_cast<uint32_t>(d), o.data.data()));
    run.outputs.push_back(std::move(o));
  }
  return run;
  }
}

// CPD-ALS driver (no reference counterpart).  Returns the final fit; factors are updated
// in place (normalised columns) and lambda receives the column weights.
template <typename T>
double cpd_als(const SparseTensorCOO<T>& t, const std::vector<ModePlan>& plans,
               std::vector<FactorMatrix<T>>& factors, std::size_t max_iters, double tol,
               std::vector<T>* lambda = nullptr, std::size_t* iters_done = nullptr) {
  static_assert(std::is_same_v<T, float>, "cpd_als runs in fp32 on the device");
  detail::validate_factors(t, factors);
  auto& s = *plans.at(0).device;
  detail::upload_factors(s, factors);
  double fit = 0;
  uint64_t done = 0;
  std::vector<float> lam(factors[0].rank);
  detail::check(mk_cpd_als(s.ctx, max_iters, tol, &fit, &done, lam.data()));
  for (std::size_t d = 0; d < factors.size(); ++d)
    detail::check(mk_factor_download(s.ctx, static_cast<uint32_t>(d), factors[d].data.data()));
  if (lambda) *lambda = lam;
  if (iters_done) *iters_done = done;
  return fit;
}

}  // namespace mttkrp_b200
