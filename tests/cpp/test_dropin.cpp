// The reference's own kernel/layout test cases (proj/tests/test_kernel.cpp,
// test_layout.cpp), re-stated against the C++ drop-in header so they read like the
// reference's tests: only the include and the namespace alias change.
#include <cmath>
#include <cstdio>
#include <functional>
#include <set>
#include <string>
#include <vector>

#include "mttkrp_b200/frostt.hpp"
#include "mttkrp_b200/mttkrp.hpp"

namespace mttkrp = mttkrp_b200;
using namespace mttkrp;

static int g_fail = 0, g_checks = 0;
#define CHECK(x)                                                            \
  do {                                                                      \
    ++g_checks;                                                             \
    if (!(x)) {                                                             \
      ++g_fail;                                                             \
      std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #x);      \
    }                                                                       \
  } while (0)
#define CHECK_THROWS(x)                                                     \
  do {                                                                      \
    ++g_checks;                                                             \
    bool thrown = false;                                                    \
    try {                                                                   \
      (void)(x);                                                            \
    } catch (const mttkrp::error&) {                                        \
      thrown = true;                                                        \
    }                                                                       \
    if (!thrown) {                                                          \
      ++g_fail;                                                             \
      std::printf("CHECK_THROWS failed %s:%d: %s\n", __FILE__, __LINE__, #x); \
    }                                                                       \
  } while (0)

template <typename T>
std::vector<FactorMatrix<T>> matrices_from(const std::vector<std::vector<std::vector<T>>>& vals) {
  std::vector<FactorMatrix<T>> out;
  for (std::size_t d = 0; d < vals.size(); ++d) {
    auto m = FactorMatrix<T>::zeros(d, static_cast<index_t>(vals[d].size()), vals[d][0].size());
    for (index_t i = 0; i < vals[d].size(); ++i)
      for (std::size_t r = 0; r < m.rank; ++r) m.at(i, r) = vals[d][i][r];
    out.push_back(std::move(m));
  }
  return out;
}

SparseTensorCOO<float> tensor_with_mode0_degrees(const std::vector<std::uint64_t>& degrees) {
  std::uint64_t max_deg = 1;
  for (auto d : degrees) max_deg = std::max(max_deg, d);
  SparseTensorCOO<float> t(
      Shape({static_cast<index_t>(degrees.size()), static_cast<index_t>(max_deg)}));
  for (index_t v = 0; v < degrees.size(); ++v)
    for (index_t k = 0; k < degrees[v]; ++k) t.add({v, k}, 1.0f);
  return t;
}

std::vector<std::uint64_t> sizes(const ModePlan& p) {
  std::vector<std::uint64_t> s;
  for (std::size_t z = 0; z < p.kappa; ++z) s.push_back(p.partition_size(z));
  return s;
}

void single_nonzero() {
  SparseTensorCOO<float> t(Shape({1, 2, 2}));
  t.add({0, 1, 1}, 3.0f);
  auto factors = matrices_from<float>({{{1, 1}}, {{7, 8}, {1, 2}}, {{6, 7}, {2, 1}}});
  ExecConfig config{2, 32, false};
  for (auto pol : {SchemePolicy::scheme1_only, SchemePolicy::scheme2_only}) {
    auto plans = build_mode_plans(t, 2, Strategy::cyclic, pol);
    auto out0 = mttkrp_mode(t, plans[0], factors, config);
    CHECK(out0.at(0, 0) == 6.0f && out0.at(0, 1) == 6.0f);
    auto out1 = mttkrp_mode(t, plans[1], factors, config);
    CHECK(out1.row(0)[0] == 0.0f && out1.at(1, 0) == 6.0f && out1.at(1, 1) == 3.0f);
    auto out2 = mttkrp_mode(t, plans[2], factors, config);
    CHECK(out2.at(1, 0) == 3.0f && out2.at(1, 1) == 6.0f);
  }
}

void partition_kats() {
  auto t = tensor_with_mode0_degrees({5, 4, 3, 2, 1});
  auto plan = partition_scheme1(t, 0, 2, Strategy::cyclic);
  CHECK(plan.scheme == Scheme::scheme1);
  CHECK((sizes(plan) == std::vector<std::uint64_t>{9, 6}));
  CHECK((plan.owned_indices[0] == std::vector<index_t>{0, 2, 4}));
  CHECK((plan.owned_indices[1] == std::vector<index_t>{1, 3}));
  auto lpt = partition_scheme1(t, 0, 2, Strategy::least_loaded);
  CHECK((lpt.owned_indices[0] == std::vector<index_t>{0, 3, 4}));
  CHECK((lpt.owned_indices[1] == std::vector<index_t>{1, 2}));
  CHECK((sizes(partition_scheme2(tensor_with_mode0_degrees({10}), 0, 3)) ==
         std::vector<std::uint64_t>{4, 3, 3}));
  CHECK((sizes(partition_scheme2(tensor_with_mode0_degrees({2}), 0, 5)) ==
         std::vector<std::uint64_t>{1, 1, 0, 0, 0}));
  auto p0 = mode_degrees(tensor_with_mode0_degrees({1, 3, 2}), 0);
  CHECK((p0.degrees == std::vector<std::uint64_t>{1, 3, 2}));
}

void adaptive_selection() {
  SyntheticSpec spec;
  spec.dims = {6186, 24, 77, 32};
  spec.nnz = 20000;
  spec.seed = 9;
  auto t = generate_synthetic<float>(spec);
  auto plans = build_mode_plans(t, 82);
  CHECK(plans[0].scheme == Scheme::scheme1 && plans[1].scheme == Scheme::scheme2 &&
        plans[2].scheme == Scheme::scheme2 && plans[3].scheme == Scheme::scheme2);
  CHECK_THROWS(build_mode_plans(t, 0));
  CHECK(select_scheme(82, 82) == Scheme::scheme1 && select_scheme(24, 82) == Scheme::scheme2);
}

void determinism_and_chain() {
  SyntheticSpec spec;
  spec.dims = {60, 2, 40};
  spec.nnz = 900;
  spec.dist = SyntheticDist::mode_skewed;
  spec.skew_mode = 1;
  spec.seed = 77;
  auto t = generate_synthetic<float>(spec);
  auto factors = random_factors<float>(t.shape(), 8, 7);
  auto plans = build_mode_plans(t, 8);
  auto base = mttkrp_all_modes(t, plans, factors, ExecConfig{8, 1, true}, false);
  for (std::size_t p : {7u, 32u})
    CHECK(bitwise_equal(base, mttkrp_all_modes(t, plans, factors, ExecConfig{8, p, true}, false)));
  auto chained = mttkrp_all_modes(t, plans, factors, ExecConfig{8, 32, true}, true);
  CHECK(bitwise_equal(base[0], chained[0]));
  auto swapped = factors;
  swapped[0] = chained[0];
  CHECK(bitwise_equal(mttkrp_mode(t, plans[1], swapped, ExecConfig{8, 32, true}), chained[1]));
  auto timed = run_timed(t, plans, factors, ExecConfig{8, 32, true}, 3);
  CHECK(timed.report.iters == 3 && timed.report.total_ms.size() == 3);
  CHECK(timed.report.modes[1].busy_workers == 8);
  CHECK(bitwise_equal(timed.outputs, base));
  CHECK(timed.report.outputs_bit_identical);  // deterministic exec: computed, kernel.hpp:271-276
}

void errors() {
  SparseTensorCOO<float> t(Shape({1, 2, 2}));
  t.add({0, 1, 1}, 3.0f);
  auto factors = matrices_from<float>({{{1, 1}}, {{7, 8}, {1, 2}}, {{6, 7}, {2, 1}}});
  auto plans = build_mode_plans(t, 2);
  ExecConfig config{2, 32, false};
  auto short_f = factors;
  short_f.pop_back();
  CHECK_THROWS(mttkrp_mode(t, plans[0], short_f, config));
  auto bad_rank = factors;
  bad_rank[1] = FactorMatrix<float>::zeros(1, 2, 3);
  CHECK_THROWS(mttkrp_mode(t, plans[0], bad_rank, config));
  CHECK_THROWS(mttkrp_mode(t, plans[0], factors, ExecConfig{0, 32, false}));
  CHECK_THROWS(mttkrp_mode(t, plans[0], factors, ExecConfig{2, 0, false}));
  SparseTensorCOO<float> bad(Shape({1, 2, 2}));
  bad.add({0, 0, 0}, 1.0f);
  bad.add({0, 1, 1}, 3.0e38f);
  auto ff = matrices_from<float>({{{1, 1}}, {{1, 1}, {3.0e38f, 1}}, {{1, 1}, {1, 1}}});
  auto bp = build_mode_plans(bad, 2);
  bool got = false;
  try {
    (void)mttkrp_mode(bad, bp[0], ff, ExecConfig{2, 32, false});
  } catch (const mttkrp::error& e) {
    got = std::string(e.what()).find("non-finite") != std::string::npos;
  }
  CHECK(got);
}

void element_updates() {  // test_kernel.cpp:39-55
  SparseTensorCOO<float> ones(Shape({2, 2, 2}));
  ones.add({0, 1, 0}, 1.0f);
  auto all_ones = matrices_from<float>({{{1, 1}, {1, 1}}, {{1, 1}, {1, 1}}, {{1, 1}, {1, 1}}});
  CHECK(element_update(ones, 0, all_ones, 2) == std::vector<float>({1, 1}));
  SparseTensorCOO<float> t(Shape({1, 2, 1}));
  t.add({0, 1, 0}, 3.0f);
  auto f = matrices_from<float>({{{1, 2}}, {{9, 9}, {2, 1}}, {{5, 5}}});
  CHECK(element_update(t, 0, f, 2) == std::vector<float>({6, 6}));
  auto disjoint = matrices_from<float>({{{1, 0}}, {{9, 9}, {0, 1}}, {{5, 5}}});
  SparseTensorCOO<float> t2(Shape({1, 2, 1}));
  t2.add({0, 1, 0}, 2.0f);
  CHECK(element_update(t2, 0, disjoint, 2) == std::vector<float>({0, 0}));
  auto bad = f;
  bad[1] = FactorMatrix<float>::zeros(1, 2, 3);
  CHECK_THROWS(element_update(t, 0, bad, 2));
}

void fp64_path() {  // T = double: deterministic == oracle_mttkrp<double> order (f-4)
  SyntheticSpec spec;
  spec.dims = {40, 30, 20};
  spec.nnz = 3000;
  spec.seed = 5;
  auto t = generate_synthetic<double>(spec);
  auto factors = random_factors<double>(t.shape(), 8, 3);
  auto plans = build_mode_plans(t, 8);
  auto det = mttkrp_all_modes(t, plans, factors, ExecConfig{8, 32, true}, false);
  auto fast = mttkrp_all_modes(t, plans, factors, ExecConfig{8, 32, false}, false);
  for (std::size_t d = 0; d < 3; ++d) {
    auto want = FactorMatrix<double>::zeros(d, t.extent(d), 8);
    for (std::size_t i = 0; i < t.nnz(); ++i) {
      auto c = t.coords(i);
      for (std::size_t r = 0; r < 8; ++r) {
        double term = t.value(i);
        for (std::size_t w = 0; w < 3; ++w)
          if (w != d) term *= factors[w].at(c[w], r);
        want.at(c[d], r) += term;
      }
    }
    CHECK(bitwise_equal(det[d], want));
    double worst = 0;
    for (std::size_t k = 0; k < want.data.size(); ++k)
      worst = std::max(worst, std::abs(fast[d].data[k] - want.data[k]) /
                                  std::max(1.0, std::abs(want.data[k])));
    CHECK(worst <= 1e-12);
  }
  auto timed = run_timed(t, plans, factors, ExecConfig{8, 32, true}, 2);
  CHECK(timed.report.outputs_bit_identical && bitwise_equal(timed.outputs, det));
  auto g = rng::seeded(7);
  auto g2 = rng::seeded(7);
  CHECK(rng::bounded(g, 10) == rng::bounded(g2, 10));
}

// test_frostt.cpp:8-100 through the drop-in frostt.hpp (host ingest, no device work)
void frostt_cases() {
  auto res = parse_frostt<float>("1 1 1 2.0\n2 2 2 3.0\n");
  CHECK(res.tensor.shape().dims == std::vector<index_t>({2, 2, 2}));
  CHECK(res.tensor.nnz() == 2 && res.tensor.value(1) == 3.0f && res.tensor.index(1, 2) == 1);
  auto merged = parse_frostt<float>("1 1 1 2.0\n1 1 1 3.0\n");
  CHECK(merged.tensor.nnz() == 1 && merged.tensor.value(0) == 5.0f && merged.duplicates_merged == 1);
  FrosttOptions strict;
  strict.merge_duplicates = false;
  CHECK_THROWS(parse_frostt<float>("1 1 1 2.0\n1 1 1 3.0\n", strict));
  auto sci = parse_frostt<double>("# header comment\n\n  \n1 2 1.5e2\n#tail\n2 1 -3e-1\n");
  CHECK(sci.tensor.value(0) == 150.0 && sci.tensor.value(1) == -0.3);
  for (const char* bad : {"", "# comments only\n\n", "1 1 1 1\n1 1 1\n", "1 x 1 1\n",
                          "1 1 1 abc\n", "0 1 1 1\n", "1\n", "1 1 1 inf\n",
                          "5000000000 1 1 1\n"})
    CHECK_THROWS(parse_frostt<float>(bad));
  try {
    (void)parse_frostt<float>("1 1 1 1\n1 1 1\n");
  } catch (const error& e) {
    CHECK(std::string(e.what()).find("line 2") != std::string::npos);
  }
  FrosttOptions ovr;
  ovr.dims_override = {4, 4, 4};
  CHECK(parse_frostt<float>("1 1 1 1\n", ovr).tensor.shape().dims == std::vector<index_t>({4, 4, 4}));
  SparseTensorCOO<double> u(Shape({2, 3}));
  u.add({1, 2}, 0.1);
  u.add({0, 0}, -1e30);
  CHECK(write_frostt_string(u) == "2 3 0.1\n1 1 -1e+30\n");
  auto g = generate_synthetic<float>(SyntheticSpec{{30, 20, 10}, 400, SyntheticDist::uniform, 0, 2, 3});
  FrosttOptions exact;
  exact.merge_duplicates = false;
  exact.dims_override = g.shape().dims;
  CHECK(parse_frostt<float>(write_frostt_string(g), exact).tensor == g);
  const char* path = "/tmp/mkb_dropin_cache.mkbt";
  save_tensor_cache(g, path);
  CHECK(load_tensor_cache<float>(path) == g);
  std::remove(path);
}

int main() {
  const std::vector<std::pair<const char*, std::function<void()>>> cases = {
      {"single nonzero", single_nonzero}, {"partition KATs", partition_kats},
      {"adaptive selection", adaptive_selection}, {"determinism & chain", determinism_and_chain},
      {"errors", errors}, {"element_update", element_updates}, {"fp64 path", fp64_path},
      {"frostt I/O", frostt_cases}};
  for (auto& [name, fn] : cases) {
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("exception in %s: %s\n", name, e.what());
    }
    std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", name);
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
