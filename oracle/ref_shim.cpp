// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference library (arxiv 2503.18198 CPU model) so
// that Python tests and bench.py's reference arm can drive the reference's own code
// path: generate_synthetic (synthetic.hpp:58-158), random_factors (factor.hpp:71-84),
// build_mode_plans (layout.hpp:131-149 + layout.cpp:108-183), mttkrp_mode /
// mttkrp_all_modes (kernel.hpp:161-197), run_timed (kernel.hpp:239-287) and
// oracle_mttkrp (oracle.hpp:20-43).
//
// Built by oracle/Makefile directly from the reference sources where they lie under
// /root/reference (no source is copied) into oracle/_ref/libmttkrp_ref.so.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "mttkrp/factor.hpp"
#include "mttkrp/frostt.hpp"
#include "mttkrp/kernel.hpp"
#include "mttkrp/layout.hpp"
#include "mttkrp/oracle.hpp"
#include "mttkrp/synthetic.hpp"
#include "mttkrp/tensor.hpp"

using namespace mttkrp;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

template <typename T = float>
SparseTensorCOO<T> make_tensor(uint32_t n, const uint32_t* dims, uint64_t nnz,
                               const uint32_t* coords, const float* values) {
  std::vector<index_t> d(dims, dims + n);
  std::vector<index_t> c(coords, coords + nnz * n);
  std::vector<T> v(values, values + nnz);  // float -> T widening is exact
  return SparseTensorCOO<T>::from_parts(Shape(d), std::move(c), std::move(v));
}

template <typename T = float>
std::vector<FactorMatrix<T>> make_factors(uint32_t n, const uint32_t* dims, uint64_t rank,
                                          const float* concat) {
  std::vector<FactorMatrix<T>> f;
  std::size_t off = 0;
  for (uint32_t d = 0; d < n; ++d) {
    auto m = FactorMatrix<T>::zeros(d, dims[d], rank);
    for (std::size_t i = 0; i < m.data.size(); ++i) m.data[i] = concat[off + i];
    off += m.data.size();
    f.push_back(std::move(m));
  }
  return f;
}

// ModePlan objects from exported arrays (the layout of ref_build_plans_all).
std::vector<ModePlan> plans_from_arrays(uint32_t n, const uint32_t* dims, uint64_t nnz,
                                        uint64_t kappa, const int* schemes,
                                        const uint64_t* orders, const uint64_t* offsets,
                                        const uint32_t* owned_flat,
                                        const uint64_t* owned_offsets) {
  std::vector<ModePlan> plans(n);
  uint64_t owned_base = 0;
  for (uint32_t d = 0; d < n; ++d) {
    ModePlan& p = plans[d];
    p.mode = d;
    p.scheme = schemes[d] == 1 ? Scheme::scheme1 : Scheme::scheme2;
    p.kappa = kappa;
    p.order.assign(orders + d * nnz, orders + (d + 1) * nnz);
    p.partition_offsets.assign(offsets + d * (kappa + 1), offsets + (d + 1) * (kappa + 1));
    if (p.scheme == Scheme::scheme1) {
      p.owned_indices.resize(kappa);
      const uint64_t* oo = owned_offsets + d * (kappa + 1);
      for (uint64_t z = 0; z < kappa; ++z)
        p.owned_indices[z].assign(owned_flat + owned_base + oo[z], owned_flat + owned_base + oo[z + 1]);
    }
    owned_base += dims[d];
  }
  return plans;
}

Strategy strat(int s) { return s == 0 ? Strategy::cyclic : Strategy::least_loaded; }
SchemePolicy pol(int p) {
  return p == 1 ? SchemePolicy::scheme1_only
                : (p == 2 ? SchemePolicy::scheme2_only : SchemePolicy::adaptive);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_generate_synthetic(uint32_t n, const uint32_t* dims, uint64_t nnz, int dist,
                           uint64_t skew_mode, uint64_t skew_distinct, uint64_t seed,
                           uint32_t* coords_out, float* values_out) {
  return guarded([&] {
    SyntheticSpec spec;
    spec.dims.assign(dims, dims + n);
    spec.nnz = nnz;
    spec.dist = dist == 0 ? SyntheticDist::uniform : SyntheticDist::mode_skewed;
    spec.skew_mode = skew_mode;
    spec.skew_distinct = skew_distinct;
    spec.seed = seed;
    auto t = generate_synthetic<float>(spec);
    for (std::size_t i = 0; i < t.nnz(); ++i) {
      auto c = t.coords(i);
      std::memcpy(coords_out + i * n, c.data(), n * sizeof(uint32_t));
      values_out[i] = t.value(i);
    }
  });
}

int ref_random_factors(uint32_t n, const uint32_t* dims, uint64_t rank, uint64_t seed,
                       float* out) {
  return guarded([&] {
    std::vector<index_t> d(dims, dims + n);
    auto f = random_factors<float>(Shape(d), rank, seed);
    std::size_t off = 0;
    for (auto& m : f) {
      std::memcpy(out + off, m.data.data(), m.data.size() * sizeof(float));
      off += m.data.size();
    }
  });
}

// Builds all plans; plan of `mode` is exported. owned_flat must hold >= extent entries.
int ref_build_plan(uint32_t n, const uint32_t* dims, uint64_t nnz, const uint32_t* coords,
                   const float* values, uint32_t mode, uint64_t kappa, int strategy, int policy,
                   int* scheme, uint64_t* order, uint64_t* offsets, uint32_t* owned_flat,
                   uint64_t* owned_offsets) {
  return guarded([&] {
    auto t = make_tensor(n, dims, nnz, coords, values);
    auto plans = build_mode_plans(t, kappa, strat(strategy), pol(policy));
    const ModePlan& p = plans.at(mode);
    *scheme = p.scheme == Scheme::scheme1 ? 1 : 2;
    std::memcpy(order, p.order.data(), p.order.size() * sizeof(uint64_t));
    std::memcpy(offsets, p.partition_offsets.data(), p.partition_offsets.size() * sizeof(uint64_t));
    uint64_t pos = 0;
    owned_offsets[0] = 0;
    for (std::size_t z = 0; z < kappa; ++z) {
      if (p.scheme == Scheme::scheme1) {
        for (index_t v : p.owned_indices[z]) owned_flat[pos++] = v;
      }
      owned_offsets[z + 1] = pos;
    }
  });
}

int ref_oracle_mttkrp(uint32_t n, const uint32_t* dims, uint64_t nnz, const uint32_t* coords,
                      const float* values, uint64_t rank, const float* factors, uint32_t mode,
                      float* out) {
  return guarded([&] {
    auto t = make_tensor(n, dims, nnz, coords, values);
    auto f = make_factors(n, dims, rank, factors);
    auto o = oracle_mttkrp(t, f, mode);
    std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
  });
}

// oracle_mttkrp<double> (oracle.hpp:20-43, the reference's own fp64 instantiation) on the
// fp32 inputs widened exactly to double: the fp64 truth the fast path is gated against.
int ref_oracle_mttkrp_f64(uint32_t n, const uint32_t* dims, uint64_t nnz, const uint32_t* coords,
                          const float* values, uint64_t rank, const float* factors, uint32_t mode,
                          double* out) {
  return guarded([&] {
    auto t = make_tensor<double>(n, dims, nnz, coords, values);
    auto f = make_factors<double>(n, dims, rank, factors);
    auto o = oracle_mttkrp(t, f, mode);
    std::memcpy(out, o.data.data(), o.data.size() * sizeof(double));
  });
}

// build_mode_plans once, every mode exported: orders[n * nnz], offsets[n * (kappa+1)],
// owned_flat[sum dims] (mode d's owned indices start at sum_{w<d} dims[w]),
// owned_offsets[n * (kappa+1)] (relative to the mode's base), schemes[n].
int ref_build_plans_all(uint32_t n, const uint32_t* dims, uint64_t nnz, const uint32_t* coords,
                        const float* values, uint64_t kappa, int strategy, int policy,
                        int* schemes, uint64_t* orders, uint64_t* offsets, uint32_t* owned_flat,
                        uint64_t* owned_offsets, double* plan_ms) {
  return guarded([&] {
    auto t = make_tensor(n, dims, nnz, coords, values);
    auto t0 = std::chrono::steady_clock::now();
    auto plans = build_mode_plans(t, kappa, strat(strategy), pol(policy));
    *plan_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    uint64_t owned_base = 0;
    for (uint32_t d = 0; d < n; ++d) {
      const ModePlan& p = plans[d];
      schemes[d] = p.scheme == Scheme::scheme1 ? 1 : 2;
      std::memcpy(orders + d * nnz, p.order.data(), nnz * sizeof(uint64_t));
      std::memcpy(offsets + d * (kappa + 1), p.partition_offsets.data(), (kappa + 1) * sizeof(uint64_t));
      uint64_t* oo = owned_offsets + d * (kappa + 1);
      uint64_t pos = 0;
      oo[0] = 0;
      for (uint64_t z = 0; z < kappa; ++z) {
        if (p.scheme == Scheme::scheme1)
          for (index_t v : p.owned_indices[z]) owned_flat[owned_base + pos++] = v;
        oo[z + 1] = pos;
      }
      owned_base += dims[d];
    }
  });
}

// run_timed (kernel.hpp:239-287) on plans given as arrays (bit-identical plans built by the
// oracle's fast planner, pinned against the reference's build_mode_plans in tests): the
// reference's timed executor without its ~90 s single-threaded plan sort at 77M nnz.
int ref_run_timed_plans(uint32_t n, const uint32_t* dims, uint64_t nnz, const uint32_t* coords,
                        const float* values, uint64_t rank, const float* factors, uint64_t kappa,
                        const int* schemes, const uint64_t* orders, const uint64_t* offsets,
                        const uint32_t* owned_flat, const uint64_t* owned_offsets,
                        uint64_t batch_p, uint64_t iters, double* total_ms_per_iter,
                        double* mode_min_ms, int* bit_identical) {
  return guarded([&] {
    auto t = make_tensor(n, dims, nnz, coords, values);
    auto f = make_factors(n, dims, rank, factors);
    auto plans = plans_from_arrays(n, dims, nnz, kappa, schemes, orders, offsets, owned_flat,
                                   owned_offsets);
    ExecConfig cfg{kappa, batch_p, false};
    auto run = run_timed(t, plans, f, cfg, iters);
    for (std::size_t i = 0; i < run.report.total_ms.size(); ++i)
      total_ms_per_iter[i] = run.report.total_ms[i];
    for (std::size_t d = 0; d < run.report.modes.size(); ++d)
      mode_min_ms[d] = run.report.modes[d].min_ms;
    *bit_identical = run.report.outputs_bit_identical ? 1 : 0;
  });
}

// mttkrp_all_modes through the reference executor; outputs concatenated per mode.
int ref_mttkrp_all_modes(uint32_t n, const uint32_t* dims, uint64_t nnz, const uint32_t* coords,
                         const float* values, uint64_t rank, const float* factors,
                         uint64_t kappa, int strategy, int policy, int deterministic, int chain,
                         float* outs) {
  return guarded([&] {
    auto t = make_tensor(n, dims, nnz, coords, values);
    auto f = make_factors(n, dims, rank, factors);
    auto plans = build_mode_plans(t, kappa, strat(strategy), pol(policy));
    ExecConfig cfg{kappa, 32, deterministic != 0};
    auto o = mttkrp_all_modes(t, plans, f, cfg, chain != 0);
    std::size_t off = 0;
    for (auto& m : o) {
      std::memcpy(outs + off, m.data.data(), m.data.size() * sizeof(float));
      off += m.data.size();
    }
  });
}

// The reference's measured unit: run_timed (kernel.hpp:239-287) after build_mode_plans.
// plan_ms receives the host wall time of build_mode_plans.
int ref_run_timed(uint32_t n, const uint32_t* dims, uint64_t nnz, const uint32_t* coords,
                  const float* values, uint64_t rank, const float* factors, uint64_t kappa,
                  int strategy, int policy, uint64_t batch_p, uint64_t iters,
                  double* total_ms_per_iter, double* mode_min_ms, double* plan_ms) {
  return guarded([&] {
    auto t = make_tensor(n, dims, nnz, coords, values);
    auto f = make_factors(n, dims, rank, factors);
    auto t0 = std::chrono::steady_clock::now();
    auto plans = build_mode_plans(t, kappa, strat(strategy), pol(policy));
    auto t1 = std::chrono::steady_clock::now();
    *plan_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    ExecConfig cfg{kappa, batch_p, false};
    auto run = run_timed(t, plans, f, cfg, iters);
    for (std::size_t i = 0; i < run.report.total_ms.size(); ++i)
      total_ms_per_iter[i] = run.report.total_ms[i];
    for (std::size_t d = 0; d < run.report.modes.size(); ++d)
      mode_min_ms[d] = run.report.modes[d].min_ms;
  });
}

// The reference's FROSTT parser (frostt.hpp:74-160) on a text buffer.  Outputs go to caller
// buffers sized for `cap` elements of up to `max_modes` modes; returns the element count.
int ref_frostt_parse(const char* text, uint64_t len, int prec, int merge,
                     const uint32_t* dims_override, uint32_t n_override, uint64_t cap,
                     uint32_t max_modes, uint32_t* n_out, uint32_t* dims_out, uint64_t* nnz_out,
                     uint64_t* dups_out, uint32_t* coords_out, void* values_out) {
  return guarded([&] {
    FrosttOptions opt;
    opt.merge_duplicates = merge != 0;
    if (n_override) opt.dims_override.assign(dims_override, dims_override + n_override);
    auto emit = [&](const auto& res) {
      const auto& t = res.tensor;
      if (t.nnz() > cap || t.mode_count() > max_modes) throw error("shim: buffer too small");
      *n_out = static_cast<uint32_t>(t.mode_count());
      for (std::size_t h = 0; h < t.mode_count(); ++h) dims_out[h] = t.extent(h);
      *nnz_out = t.nnz();
      *dups_out = res.duplicates_merged;
      using V = typename std::decay_t<decltype(t)>::value_type;
      for (std::size_t i = 0; i < t.nnz(); ++i) {
        auto c = t.coords(i);
        std::memcpy(coords_out + i * t.mode_count(), c.data(), t.mode_count() * sizeof(uint32_t));
        static_cast<V*>(values_out)[i] = t.value(i);
      }
    };
    const std::string_view sv(text, len);
    if (prec == 64) emit(parse_frostt<double>(sv, opt));
    else emit(parse_frostt<float>(sv, opt));
  });
}

// The reference's writer (frostt.hpp:165-192); returns the byte length, copies up to cap.
int ref_frostt_write(uint32_t n, const uint32_t* dims, uint64_t nnz, const uint32_t* coords,
                     const void* values, int prec, char* out, uint64_t cap, uint64_t* len) {
  return guarded([&] {
    auto go = [&](auto tag) {
      using V = decltype(tag);
      std::vector<index_t> d(dims, dims + n);
      std::vector<index_t> c(coords, coords + nnz * n);
      std::vector<V> v(static_cast<const V*>(values), static_cast<const V*>(values) + nnz);
      auto t = SparseTensorCOO<V>::from_parts(Shape(d), std::move(c), std::move(v));
      const std::string s = write_frostt_string(t);
      *len = s.size();
      std::memcpy(out, s.data(), std::min<uint64_t>(cap, s.size()));
    };
    if (prec == 64) go(double{});
    else go(float{});
  });
}

}  // extern "C"
