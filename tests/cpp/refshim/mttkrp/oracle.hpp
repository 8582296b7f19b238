// TEST INFRASTRUCTURE: the reference's oracle API (oracle.hpp:16-111) over the drop-in's types,
// for compiling the reference's acceptance suite against the B200 library.  These are the
// checkers, restated here (sequential, host-only); nothing in the product calls them.
//   oracle_mttkrp          element order, term = val * Y_w ascending (oracle.hpp:20-43)
//   dense_unfolding_mttkrp dense unfolding times an explicit Khatri-Rao product (:49-98)
//   brute_force_optimal_partition  exhaustive min-makespan assignment (oracle.cpp:40-70)
#pragma once
#include <algorithm>
#include <cstdint>
#include <functional>
#include <span>
#include <vector>

#include "mttkrp_b200/mttkrp.hpp"

namespace mttkrp_b200 {

template <typename T>
FactorMatrix<T> oracle_mttkrp(const SparseTensorCOO<T>& t, const std::vector<FactorMatrix<T>>& f,
                              std::size_t d) {
  if (d >= t.mode_count()) throw error("oracle: mode out of range");
  const std::size_t R = f.at(d).rank;
  auto out = FactorMatrix<T>::zeros(d, t.extent(d), R);
  std::vector<T> term(R);
  for (std::size_t e = 0; e < t.nnz(); ++e) {
    std::fill(term.begin(), term.end(), t.value(e));
    for (std::size_t w = 0; w < t.mode_count(); ++w) {
      if (w == d) continue;
      const index_t c = t.index(e, w);
      for (std::size_t r = 0; r < R; ++r) term[r] *= f[w].at(c, r);
    }
    const index_t row = t.index(e, d);
    for (std::size_t r = 0; r < R; ++r) out.at(row, r) += term[r];
  }
  return out;
}

template <typename T>
FactorMatrix<T> dense_unfolding_mttkrp(const SparseTensorCOO<T>& t,
                                       const std::vector<FactorMatrix<T>>& f, std::size_t d,
                                       std::uint64_t capacity_limit = 4096) {
  if (d >= t.mode_count()) throw error("oracle: mode out of range");
  std::uint64_t cap = 1;
  for (index_t e : t.shape().dims) cap *= e;
  if (cap > capacity_limit) throw error("oracle: tensor too large for the dense cross-check");
  const std::size_t R = f.at(d).rank, N = t.mode_count();
  // column index of a coordinate tuple: the other modes, lowest mode fastest
  auto column = [&](std::span<const index_t> c) {
    std::uint64_t col = 0, stride = 1;
    for (std::size_t h = 0; h < N; ++h)
      if (h != d) col += c[h] * stride, stride *= t.extent(h);
    return col;
  };
  const std::uint64_t ncol = cap / t.extent(d);
  std::vector<T> X(static_cast<std::size_t>(t.extent(d)) * ncol, T{0});
  for (std::size_t e = 0; e < t.nnz(); ++e)
    X[t.index(e, d) * ncol + column(t.coords(e))] += t.value(e);
  // Khatri-Rao row of every column: decode the column back into coordinates
  auto out = FactorMatrix<T>::zeros(d, t.extent(d), R);
  std::vector<index_t> c(N, 0);
  for (std::uint64_t col = 0; col < ncol; ++col) {
    std::uint64_t rem = col;
    for (std::size_t h = 0; h < N; ++h)
      if (h != d) c[h] = static_cast<index_t>(rem % t.extent(h)), rem /= t.extent(h);
    for (index_t i = 0; i < t.extent(d); ++i) {
      const T x = X[i * ncol + col];
      if (x == T{0}) continue;
      for (std::size_t r = 0; r < R; ++r) {
        T k = T{1};
        for (std::size_t h = 0; h < N; ++h)
          if (h != d) k *= f[h].at(c[h], r);
        out.at(i, r) += x * k;
      }
    }
  }
  return out;
}

struct OptimalPartitionResult {
  std::uint64_t opt_max_load = 0;
  std::vector<std::uint32_t> witness;
};

inline OptimalPartitionResult brute_force_optimal_partition(std::span<const std::uint64_t> deg,
                                                            std::size_t kappa) {
  if (kappa < 1 || deg.size() > 14 || kappa > 4) throw error("oracle: instance too large");
  // heaviest first, branch and bound on the running makespan
  std::vector<std::size_t> idx(deg.size());
  for (std::size_t i = 0; i < idx.size(); ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](std::size_t a, std::size_t b) { return deg[a] > deg[b]; });
  OptimalPartitionResult best;
  best.opt_max_load = UINT64_MAX;
  std::vector<std::uint64_t> load(kappa, 0);
  std::vector<std::uint32_t> cur(deg.size(), 0);
  std::function<void(std::size_t, std::uint64_t)> go = [&](std::size_t k, std::uint64_t mk) {
    if (mk >= best.opt_max_load) return;
    if (k == idx.size()) {
      best.opt_max_load = mk;
      best.witness = cur;
      return;
    }
    for (std::size_t z = 0; z < kappa; ++z) {
      if (z > 0 && load[z] == load[z - 1]) continue;  // symmetric partitions
      load[z] += deg[idx[k]];
      cur[idx[k]] = static_cast<std::uint32_t>(z);
      go(k + 1, std::max(mk, load[z]));
      load[z] -= deg[idx[k]];
    }
  };
  go(0, 0);
  if (deg.empty()) best.opt_max_load = 0;
  return best;
}

}  // namespace mttkrp_b200
namespace mttkrp = mttkrp_b200;
