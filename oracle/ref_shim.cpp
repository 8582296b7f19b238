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
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "mttkrp/factor.hpp"
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

SparseTensorCOO<float> make_tensor(uint32_t n, const uint32_t* dims, uint64_t nnz,
                                   const uint32_t* coords, const float* values) {
  std::vector<index_t> d(dims, dims + n);
  std::vector<index_t> c(coords, coords + nnz * n);
  std::vector<float> v(values, values + nnz);
  return SparseTensorCOO<float>::from_parts(Shape(d), std::move(c), std::move(v));
}

std::vector<FactorMatrix<float>> make_factors(uint32_t n, const uint32_t* dims, uint64_t rank,
                                              const float* concat) {
  std::vector<FactorMatrix<float>> f;
  std::size_t off = 0;
  for (uint32_t d = 0; d < n; ++d) {
    auto m = FactorMatrix<float>::zeros(d, dims[d], rank);
    std::memcpy(m.data.data(), concat + off, m.data.size() * sizeof(float));
    off += m.data.size();
    f.push_back(std::move(m));
  }
  return f;
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

}  // extern "C"
