// Host-side tensor ingest for the device path: a bit-identical, faster re-implementation of
// the reference's synthetic generator (synthetic.hpp:58-158) and factor initialiser
// (factor.hpp:71-84), plus the DESIGN.md §5 power-law generator.
//
// Same engine (std::mt19937_64 seeded through splitmix64, rng.hpp:16-24), same draw
// sequence and same accept/reject decisions as the reference; only the duplicate filter
// differs: an open-addressing table of 64-bit packed tuples (when the index bits fit,
// else hashed tuples compared in place) instead of std::unordered_set<std::vector>.  Set
// semantics are all the draw sequence depends on, so the output is identical.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "mttkrp_b200.h"

namespace mkb {
std::string& last_error_ref();
}

namespace {

struct GenError {
  std::string msg;
};

uint64_t splitmix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

std::mt19937_64 engine_for(uint64_t seed, uint64_t stream) {
  return std::mt19937_64(splitmix(seed ^ splitmix(stream)));
}

struct Bounded {  // rng::bounded with the rejection threshold hoisted per modulus
  uint64_t n, threshold;
  explicit Bounded(uint64_t n_) : n(n_), threshold((0 - n_) % n_) {}
  uint64_t operator()(std::mt19937_64& g) const {
    for (;;) {
      const uint64_t r = g();
      if (r >= threshold) return r % n;
    }
  }
};

double unit_open_closed64(std::mt19937_64& g) {  // rng.hpp:37-39, T = double
  return 1.0 - static_cast<double>(g() >> 11) * 0x1.0p-53;
}
float unit_open_closed(std::mt19937_64& g) { return static_cast<float>(unit_open_closed64(g)); }

uint64_t sat_mul(uint64_t a, uint64_t b) {
  if (a && b > UINT64_MAX / a) return UINT64_MAX;
  return a * b;
}

// Distinct-tuple filter.  Packed mode stores the tuple as one 64-bit word (+1, 0 = empty);
// wide mode stores tuple indices into the caller's coordinate array.
class TupleSet {
 public:
  TupleSet(uint64_t expected, uint32_t n, const uint32_t* dims, const uint32_t* base)
      : n_(n), base_(base) {
    int total = 0;
    for (uint32_t h = 0; h < n; ++h) {
      shift_[h] = total;
      int b = 0;
      while (b < 32 && (uint64_t{1} << b) < dims[h]) ++b;
      total += std::max(b, 1);
    }
    packed_ = total <= 63;
    uint64_t cap = 64;
    while (cap < 2 * expected + 64) cap <<= 1;
    slot_.assign(cap, 0);
    mask_ = cap - 1;
  }
  // tuple t (n words) at index idx of base_; returns true when it was not seen before
  bool insert(const uint32_t* t, uint64_t idx) {
    uint64_t key = 0, h;
    if (packed_) {
      for (uint32_t i = 0; i < n_; ++i) key |= static_cast<uint64_t>(t[i]) << shift_[i];
      h = splitmix(key);
      ++key;
    } else {
      uint64_t x = 0xcbf29ce484222325ull;
      for (uint32_t i = 0; i < n_; ++i) x = (x ^ t[i]) * 0x100000001b3ull;
      h = splitmix(x);
      key = idx + 1;
    }
    for (h &= mask_;; h = (h + 1) & mask_) {
      const uint64_t v = slot_[h];
      if (!v) {
        slot_[h] = key;
        return true;
      }
      if (packed_) {
        if (v == key) return false;
      } else if (std::memcmp(base_ + (v - 1) * n_, t, n_ * sizeof(uint32_t)) == 0) {
        return false;
      }
    }
  }

 private:
  uint32_t n_;
  const uint32_t* base_;
  int shift_[64] = {};
  bool packed_ = true;
  std::vector<uint64_t> slot_;
  uint64_t mask_ = 0;
};

// synthetic.hpp:33-54
std::vector<uint64_t> sample_distinct(std::mt19937_64& g, uint64_t space, uint64_t count) {
  std::vector<uint64_t> out;
  out.reserve(count);
  const uint64_t enumerable = std::max<uint64_t>(uint64_t{1} << 22, 4 * count);
  if (space <= enumerable) {
    std::vector<uint64_t> ids(space);
    std::iota(ids.begin(), ids.end(), 0);
    for (uint64_t i = 0; i < count; ++i) {
      const uint64_t j = i + Bounded(space - i)(g);
      std::swap(ids[i], ids[j]);
      out.push_back(ids[i]);
    }
  } else {
    std::vector<uint32_t> words(2 * count);
    const uint32_t wide[2] = {0xffffffffu, 0xffffffffu};
    TupleSet seen(count, 2, wide, words.data());
    const Bounded b(space);
    while (out.size() < count) {
      const uint64_t v = b(g);
      uint32_t* t = words.data() + 2 * out.size();
      t[0] = static_cast<uint32_t>(v);
      t[1] = static_cast<uint32_t>(v >> 32);
      if (seen.insert(t, out.size())) out.push_back(v);
    }
  }
  return out;
}

// values: fp32 (values32) or fp64 (values64, SparseTensorCOO<double>); the draws are the same
void generate(uint32_t n, const uint32_t* dims, uint64_t nnz, int dist, uint64_t skew_mode,
              uint64_t skew_distinct, uint64_t seed, uint32_t* coords, float* values32,
              double* values64 = nullptr) {
  if (n == 0) throw GenError{"shape: a tensor needs at least one mode"};
  for (uint32_t h = 0; h < n; ++h)
    if (!dims[h]) throw GenError{"shape: zero extent"};
  const bool skewed = dist == 1;
  if (skewed && skew_mode >= n) throw GenError{"synthetic: skew mode out of range"};
  const uint64_t sm = skewed ? skew_mode : 0;
  const uint64_t skew_values =
      skewed ? std::min<uint64_t>(std::max<uint64_t>(skew_distinct, 1), dims[sm]) : 0;
  uint64_t other_cap = 1;
  for (uint32_t h = 0; h < n; ++h)
    if (!(skewed && h == sm)) other_cap = sat_mul(other_cap, dims[h]);
  uint64_t cap = 1;
  if (skewed) {
    cap = sat_mul(other_cap, skew_values);
  } else {
    for (uint32_t h = 0; h < n; ++h) cap = sat_mul(cap, dims[h]);
  }
  if (nnz > cap)
    throw GenError{"synthetic: nnz " + std::to_string(nnz) + " exceeds index capacity " +
                   std::to_string(cap)};

  std::mt19937_64 g = engine_for(seed, 0);
  std::vector<Bounded> bnd;
  for (uint32_t h = 0; h < n; ++h) bnd.emplace_back(dims[h]);
  auto decode = [&](uint64_t id, uint32_t* dst) {
    for (uint32_t h = 0; h < n; ++h) {
      if (skewed && h == sm) {
        dst[h] = 0;
        continue;
      }
      dst[h] = static_cast<uint32_t>(id % dims[h]);
      id /= dims[h];
    }
  };
  auto lim = [](uint64_t c) { return std::max<uint64_t>(uint64_t{1} << 22, 4 * c); };

  if (!skewed) {
    if (cap <= lim(nnz)) {
      auto ids = sample_distinct(g, cap, nnz);
      for (uint64_t i = 0; i < nnz; ++i) decode(ids[i], coords + i * n);
    } else {
      TupleSet seen(nnz, n, dims, coords);
      uint64_t have = 0;
      while (have < nnz) {
        uint32_t* t = coords + have * n;
        for (uint32_t h = 0; h < n; ++h) t[h] = static_cast<uint32_t>(bnd[h](g));
        if (seen.insert(t, have)) ++have;
      }
    }
  } else {
    auto chosen = sample_distinct(g, dims[sm], skew_values);
    std::sort(chosen.begin(), chosen.end());
    uint64_t base = 0;
    for (uint64_t j = 0; j < skew_values; ++j) {
      const uint64_t quota = nnz / skew_values + (j < nnz % skew_values ? 1 : 0);
      if (quota > other_cap)
        throw GenError{"synthetic: per-coordinate quota exceeds off-mode capacity"};
      uint32_t* blk = coords + base * n;
      if (other_cap <= lim(quota)) {
        auto ids = sample_distinct(g, other_cap, quota);
        for (uint64_t i = 0; i < quota; ++i) decode(ids[i], blk + i * n);
      } else {
        TupleSet seen(quota, n, dims, blk);
        uint64_t have = 0;
        while (have < quota) {
          uint32_t* t = blk + have * n;
          for (uint32_t h = 0; h < n; ++h)
            t[h] = h == sm ? 0u : static_cast<uint32_t>(bnd[h](g));
          if (seen.insert(t, have)) ++have;
        }
      }
      for (uint64_t i = 0; i < quota; ++i) blk[i * n + sm] = static_cast<uint32_t>(chosen[j]);
      base += quota;
    }
  }
  if (values64)
    for (uint64_t i = 0; i < nnz; ++i) values64[i] = unit_open_closed64(g);
  else
    for (uint64_t i = 0; i < nnz; ++i) values32[i] = unit_open_closed(g);
}

// per-mode Zipf(exponent) over a seeded permutation of [0, I_h).
void generate_powerlaw(uint32_t n, const uint32_t* dims, uint64_t nnz, double exponent,
                       uint64_t seed, uint32_t* coords, float* values) {
  if (n == 0) throw GenError{"shape: a tensor needs at least one mode"};
  uint64_t cap = 1;
  for (uint32_t h = 0; h < n; ++h) {
    if (!dims[h]) throw GenError{"shape: zero extent"};
    cap = sat_mul(cap, dims[h]);
  }
  if (nnz > cap)
    throw GenError{"synthetic: nnz " + std::to_string(nnz) + " exceeds index capacity " +
                   std::to_string(cap)};
  std::mt19937_64 g = engine_for(seed, 0);
  std::vector<std::vector<uint32_t>> perm(n);
  std::vector<std::vector<double>> cdf(n);
  for (uint32_t h = 0; h < n; ++h) {
    const uint32_t e = dims[h];
    perm[h].resize(e);
    std::iota(perm[h].begin(), perm[h].end(), 0u);
    for (uint32_t i = 0; i + 1 < e; ++i)
      std::swap(perm[h][i], perm[h][i + static_cast<uint32_t>(Bounded(e - i)(g))]);
    cdf[h].resize(e);
    double acc = 0.0;
    for (uint32_t k = 0; k < e; ++k) {
      acc += exponent == 1.0 ? 1.0 / static_cast<double>(k + 1)
                             : std::pow(static_cast<double>(k + 1), -exponent);
      cdf[h][k] = acc;
    }
    for (double& x : cdf[h]) x /= acc;
  }
  TupleSet seen(nnz, n, dims, coords);
  uint64_t have = 0, attempts = 0;
  const uint64_t limit = 64 * nnz + 1000000;
  while (have < nnz) {
    if (++attempts > limit)
      throw GenError{"synthetic: power-law sampler could not find enough distinct tuples"};
    uint32_t* t = coords + have * n;
    for (uint32_t h = 0; h < n; ++h) {
      const double u = static_cast<double>(g() >> 11) * 0x1.0p-53;
      const auto it = std::upper_bound(cdf[h].begin(), cdf[h].end(), u);
      const size_t k = std::min<size_t>(it - cdf[h].begin(), dims[h] - 1);
      t[h] = perm[h][k];
    }
    if (seen.insert(t, have)) ++have;
  }
  for (uint64_t i = 0; i < nnz; ++i) values[i] = unit_open_closed(g);
}

template <typename F>
int run(F&& f) {
  try {
    f();
    mkb::last_error_ref().clear();
    return MK_OK;
  } catch (const GenError& e) {
    mkb::last_error_ref() = e.msg;
    return MK_EINVAL;
  } catch (const std::bad_alloc&) {
    mkb::last_error_ref() = "host allocation failed";
    return MK_ENOMEM;
  }
}

}  // namespace

extern "C" {

int mk_generate_synthetic(uint32_t n, const uint32_t* dims, uint64_t nnz, int dist,
                          uint64_t skew_mode, uint64_t skew_distinct, uint64_t seed,
                          uint32_t* coords, float* values) {
  return run([&] { generate(n, dims, nnz, dist, skew_mode, skew_distinct, seed, coords, values); });
}

int mk_generate_powerlaw(uint32_t n, const uint32_t* dims, uint64_t nnz, double exponent,
                         uint64_t seed, uint32_t* coords, float* values) {
  return run([&] { generate_powerlaw(n, dims, nnz, exponent, seed, coords, values); });
}

int mk_generate_synthetic_f64(uint32_t n, const uint32_t* dims, uint64_t nnz, int dist,
                              uint64_t skew_mode, uint64_t skew_distinct, uint64_t seed,
                              uint32_t* coords, double* values) {
  return run([&] {
    generate(n, dims, nnz, dist, skew_mode, skew_distinct, seed, coords, nullptr, values);
  });
}

int mk_random_factors_f64(uint32_t n, const uint32_t* dims, uint64_t rank, uint64_t seed,
                          double* const* factors) {
  return run([&] {
    if (rank < 1) throw GenError{"factor: rank must be at least 1"};
    for (uint32_t d = 0; d < n; ++d) {
      std::mt19937_64 g = engine_for(seed, uint64_t{d} + 1);
      const uint64_t cnt = static_cast<uint64_t>(dims[d]) * rank;
      for (uint64_t i = 0; i < cnt; ++i) factors[d][i] = unit_open_closed64(g);
    }
  });
}

int mk_random_factors(uint32_t n, const uint32_t* dims, uint64_t rank, uint64_t seed,
                      float* const* factors) {
  return run([&] {
    if (rank < 1) throw GenError{"factor: rank must be at least 1"};
    for (uint32_t d = 0; d < n; ++d) {
      std::mt19937_64 g = engine_for(seed, uint64_t{d} + 1);
      const uint64_t cnt = static_cast<uint64_t>(dims[d]) * rank;
      for (uint64_t i = 0; i < cnt; ++i) factors[d][i] = unit_open_closed(g);
    }
  });
}

}  // extern "C"
