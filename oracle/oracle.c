/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle (plain C restatement of the reference path).
 * See oracle.h for the rules.  Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj/core).  Compiled with -ffp-contract=off so
 * every fp32 multiply/add rounds exactly like the reference build (g++ -O3, SSE2).
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];
const char* orc_last_error(void) { return g_err; }
#define FAIL(...)                                      \
  do {                                                 \
    snprintf(g_err, sizeof g_err, __VA_ARGS__);        \
    return 1;                                          \
  } while (0)

/* ---------------------------------------------------------------- rng.hpp:12-39 */
static uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* std::mt19937_64 as fixed by the C++ standard [rand.eng.mers]. */
static void mt_init(orc_engine* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->mti = 312;
}

uint64_t orc_next(orc_engine* g) {
  static const uint64_t A = 0xB5026F5AA96619E9ull, UM = 0xFFFFFFFF80000000ull,
                        LM = 0x7FFFFFFFull;
  if (g->mti >= 312) {
    int i;
    for (i = 0; i < 312 - 156; ++i) {
      uint64_t x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
      g->mt[i] = g->mt[i + 156] ^ (x >> 1) ^ ((x & 1ull) ? A : 0ull);
    }
    for (; i < 311; ++i) {
      uint64_t x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
      g->mt[i] = g->mt[i + 156 - 312] ^ (x >> 1) ^ ((x & 1ull) ? A : 0ull);
    }
    uint64_t x = (g->mt[311] & UM) | (g->mt[0] & LM);
    g->mt[311] = g->mt[155] ^ (x >> 1) ^ ((x & 1ull) ? A : 0ull);
    g->mti = 0;
  }
  uint64_t x = g->mt[g->mti++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= (x >> 43);
  return x;
}

/* rng.hpp:22-24 */
void orc_seeded(orc_engine* g, uint64_t seed, uint64_t stream) {
  mt_init(g, splitmix64(seed ^ splitmix64(stream)));
}

/* rng.hpp:27-33 */
uint64_t orc_bounded(orc_engine* g, uint64_t n) {
  const uint64_t threshold = (0 - n) % n;
  for (;;) {
    uint64_t r = orc_next(g);
    if (r >= threshold) return r % n;
  }
}

/* rng.hpp:36-39 */
static float unit_open_closed_f(orc_engine* g) {
  return (float)(1.0 - (double)(orc_next(g) >> 11) * 0x1.0p-53);
}

/* ------------------------------------------------------ tuple set (std::unordered_set
 * stand-in: only set semantics matter to the draw sequence, synthetic.hpp:113-120). */
typedef struct {
  uint64_t* slot; /* tuple index + 1, 0 = empty */
  uint64_t mask;
  const uint32_t* base; /* tuples stored contiguously, n words each */
  uint32_t n;
} tset;

static int tset_init(tset* s, uint64_t expected, uint32_t n) {
  uint64_t cap = 16;
  while (cap < 2 * expected + 16) cap <<= 1;
  s->slot = (uint64_t*)calloc(cap, sizeof(uint64_t));
  s->mask = cap - 1;
  s->n = n;
  return s->slot ? 0 : 1;
}
static uint64_t thash(const uint32_t* t, uint32_t n) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint32_t i = 0; i < n; ++i) h = (h ^ t[i]) * 0x100000001b3ull;
  return splitmix64(h);
}
/* Inserts tuple at index idx of base (already written there). Returns 1 if new. */
static int tset_insert(tset* s, uint64_t idx) {
  const uint32_t* t = s->base + idx * s->n;
  uint64_t h = thash(t, s->n) & s->mask;
  for (;;) {
    uint64_t v = s->slot[h];
    if (!v) {
      s->slot[h] = idx + 1;
      return 1;
    }
    if (memcmp(s->base + (v - 1) * s->n, t, s->n * sizeof(uint32_t)) == 0) return 0;
    h = (h + 1) & s->mask;
  }
}

/* synthetic.hpp:33-54 */
static uint64_t* sample_distinct(orc_engine* g, uint64_t space, uint64_t count) {
  uint64_t* out = (uint64_t*)malloc((count ? count : 1) * sizeof(uint64_t));
  uint64_t enumerable = (uint64_t)1 << 22;
  if (4 * count > enumerable) enumerable = 4 * count;
  if (space <= enumerable) {
    uint64_t* ids = (uint64_t*)malloc((space ? space : 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < space; ++i) ids[i] = i;
    for (uint64_t i = 0; i < count; ++i) {
      uint64_t j = i + orc_bounded(g, space - i);
      uint64_t tmp = ids[i];
      ids[i] = ids[j];
      ids[j] = tmp;
      out[i] = ids[i];
    }
    free(ids);
  } else {
    /* distinct scalar ids: reuse the tuple set over a 2-word view of each id */
    uint32_t* words = (uint32_t*)malloc((count ? count : 1) * 2 * sizeof(uint32_t));
    tset s;
    tset_init(&s, count, 2);
    s.base = words;
    uint64_t have = 0;
    while (have < count) {
      uint64_t v = orc_bounded(g, space);
      words[2 * have] = (uint32_t)v;
      words[2 * have + 1] = (uint32_t)(v >> 32);
      if (tset_insert(&s, have)) out[have++] = v;
    }
    free(s.slot);
    free(words);
  }
  return out;
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y);
}

static uint64_t sat_mul(uint64_t a, uint64_t b) {
  if (a && b > UINT64_MAX / a) return UINT64_MAX;
  return a * b;
}

/* synthetic.hpp:96-106 */
static void decode_into(uint64_t id, uint32_t n, const uint32_t* dims, int skewed,
                        uint64_t skip, uint32_t* dst) {
  for (uint32_t h = 0; h < n; ++h) {
    if (skewed && h == skip) {
      dst[h] = 0;
      continue;
    }
    dst[h] = (uint32_t)(id % dims[h]);
    id /= dims[h];
  }
}

/* synthetic.hpp:58-158 */
int orc_generate_synthetic(uint32_t n, const uint32_t* dims, uint64_t nnz, int dist,
                           uint64_t skew_mode, uint64_t skew_distinct, uint64_t seed,
                           uint32_t* coords, float* values) {
  if (n == 0) FAIL("shape: a tensor needs at least one mode");
  for (uint32_t h = 0; h < n; ++h)
    if (!dims[h]) FAIL("shape: zero extent");
  const int skewed = dist == 1;
  if (skewed && skew_mode >= n) FAIL("synthetic: skew mode out of range");
  const uint64_t sm = skewed ? skew_mode : 0;
  uint64_t skew_values = 0;
  if (skewed) {
    skew_values = skew_distinct < 1 ? 1 : skew_distinct;
    if (skew_values > dims[sm]) skew_values = dims[sm];
  }
  uint64_t other_cap = 1;
  for (uint32_t h = 0; h < n; ++h) {
    if (skewed && h == sm) continue;
    other_cap = sat_mul(other_cap, dims[h]);
  }
  uint64_t cap;
  if (skewed) {
    cap = sat_mul(other_cap, skew_values);
  } else {
    cap = 1;
    for (uint32_t h = 0; h < n; ++h) cap = sat_mul(cap, dims[h]);
  }
  if (nnz > cap)
    FAIL("synthetic: nnz %llu exceeds index capacity %llu", (unsigned long long)nnz,
         (unsigned long long)cap);

  orc_engine g;
  orc_seeded(&g, seed, 0);
  uint64_t lim = (uint64_t)1 << 22;

  if (!skewed) {
    if (cap <= (lim > 4 * nnz ? lim : 4 * nnz)) {
      uint64_t* ids = sample_distinct(&g, cap, nnz);
      for (uint64_t i = 0; i < nnz; ++i) decode_into(ids[i], n, dims, 0, n, coords + i * n);
      free(ids);
    } else {
      tset s;
      tset_init(&s, nnz, n);
      s.base = coords;
      uint64_t have = 0;
      while (have < nnz) {
        uint32_t* t = coords + have * n;
        for (uint32_t h = 0; h < n; ++h) t[h] = (uint32_t)orc_bounded(&g, dims[h]);
        if (tset_insert(&s, have)) ++have;
      }
      free(s.slot);
    }
  } else {
    uint64_t* chosen = sample_distinct(&g, dims[sm], skew_values);
    qsort(chosen, skew_values, sizeof(uint64_t), cmp_u64);
    uint64_t base = 0;
    for (uint64_t j = 0; j < skew_values; ++j) {
      const uint64_t quota = nnz / skew_values + (j < nnz % skew_values ? 1 : 0);
      if (quota > other_cap) {
        free(chosen);
        FAIL("synthetic: per-coordinate quota exceeds off-mode capacity");
      }
      if (other_cap <= (lim > 4 * quota ? lim : 4 * quota)) {
        uint64_t* ids = sample_distinct(&g, other_cap, quota);
        for (uint64_t i = 0; i < quota; ++i)
          decode_into(ids[i], n, dims, 1, sm, coords + (base + i) * n);
        free(ids);
      } else {
        tset s;
        tset_init(&s, quota, n);
        s.base = coords + base * n;
        uint64_t have = 0;
        while (have < quota) {
          uint32_t* t = coords + (base + have) * n;
          for (uint32_t h = 0; h < n; ++h)
            t[h] = h == sm ? 0u : (uint32_t)orc_bounded(&g, dims[h]);
          if (tset_insert(&s, have)) ++have;
        }
        free(s.slot);
      }
      for (uint64_t i = base; i < base + quota; ++i) coords[i * n + sm] = (uint32_t)chosen[j];
      base += quota;
    }
    free(chosen);
  }
  for (uint64_t i = 0; i < nnz; ++i) values[i] = unit_open_closed_f(&g);
  return 0;
}

/* DESIGN.md §5 power-law generator (our own spec; the reference can only express
 * uniform / mode_skewed).  Engine = rng::seeded(seed).  Per mode h: a Fisher-Yates
 * permutation of [0, I_h) drawn with bounded(); then Zipf(exponent) ranks via an
 * inverse-CDF lookup of u = (g() >> 11) * 2^-53; duplicate tuples rejected in draw order;
 * values unit_open_closed<float> after the coordinates. */
int orc_generate_powerlaw(uint32_t n, const uint32_t* dims, uint64_t nnz, double exponent,
                          uint64_t seed, uint32_t* coords, float* values) {
  if (n == 0) FAIL("shape: a tensor needs at least one mode");
  uint64_t cap = 1;
  for (uint32_t h = 0; h < n; ++h) {
    if (!dims[h]) FAIL("shape: zero extent");
    cap = sat_mul(cap, dims[h]);
  }
  if (nnz > cap) FAIL("synthetic: nnz %llu exceeds index capacity %llu",
                      (unsigned long long)nnz, (unsigned long long)cap);
  orc_engine g;
  orc_seeded(&g, seed, 0);
  uint32_t** perm = (uint32_t**)calloc(n, sizeof(uint32_t*));
  double** cdf = (double**)calloc(n, sizeof(double*));
  for (uint32_t h = 0; h < n; ++h) {
    uint32_t e = dims[h];
    perm[h] = (uint32_t*)malloc(e * sizeof(uint32_t));
    cdf[h] = (double*)malloc(e * sizeof(double));
    for (uint32_t i = 0; i < e; ++i) perm[h][i] = i;
    for (uint32_t i = 0; i + 1 < e; ++i) {
      uint32_t j = i + (uint32_t)orc_bounded(&g, e - i);
      uint32_t t = perm[h][i];
      perm[h][i] = perm[h][j];
      perm[h][j] = t;
    }
    double acc = 0.0;
    for (uint32_t k = 0; k < e; ++k) {
      double w = exponent == 1.0 ? 1.0 / (double)(k + 1) : pow((double)(k + 1), -exponent);
      acc += w;
      cdf[h][k] = acc;
    }
    for (uint32_t k = 0; k < e; ++k) cdf[h][k] /= acc;
  }
  tset s;
  tset_init(&s, nnz, n);
  s.base = coords;
  uint64_t have = 0, attempts = 0, limit = 64 * nnz + 1000000;
  int rc = 0;
  while (have < nnz) {
    if (++attempts > limit) {
      snprintf(g_err, sizeof g_err,
               "synthetic: power-law sampler could not find enough distinct tuples");
      rc = 1;
      break;
    }
    uint32_t* t = coords + have * n;
    for (uint32_t h = 0; h < n; ++h) {
      double u = (double)(orc_next(&g) >> 11) * 0x1.0p-53;
      uint32_t lo = 0, hi = dims[h] - 1; /* first k with cdf[k] > u */
      while (lo < hi) {
        uint32_t mid = lo + (hi - lo) / 2;
        if (cdf[h][mid] > u) hi = mid; else lo = mid + 1;
      }
      t[h] = perm[h][lo];
    }
    if (tset_insert(&s, have)) ++have;
  }
  free(s.slot);
  for (uint32_t h = 0; h < n; ++h) {
    free(perm[h]);
    free(cdf[h]);
  }
  free(perm);
  free(cdf);
  if (rc) return rc;
  for (uint64_t i = 0; i < nnz; ++i) values[i] = unit_open_closed_f(&g);
  return 0;
}

/* factor.hpp:71-84: stream d+1 per mode, row-major fill. */
int orc_random_factors(uint32_t n, const uint32_t* dims, uint64_t rank, uint64_t seed,
                       float* out) {
  if (rank < 1) FAIL("factor: rank must be at least 1");
  uint64_t off = 0;
  for (uint32_t d = 0; d < n; ++d) {
    orc_engine g;
    orc_seeded(&g, seed, (uint64_t)d + 1);
    uint64_t cnt = (uint64_t)dims[d] * rank;
    for (uint64_t i = 0; i < cnt; ++i) out[off + i] = unit_open_closed_f(&g);
    off += cnt;
  }
  return 0;
}

/* ------------------------------------------------------------------ layout */
typedef struct {
  uint64_t deg;
  uint32_t idx;
} vdeg;
/* layout.cpp:90-99: degree descending, ties by ascending coordinate. */
static int cmp_vdeg(const void* a, const void* b) {
  const vdeg* x = (const vdeg*)a;
  const vdeg* y = (const vdeg*)b;
  if (x->deg != y->deg) return x->deg > y->deg ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* Stable counting sort of element positions by key[c] (ties keep position order),
 * which equals std::sort with the total-order comparators of layout.cpp:145-151 and
 * layout.cpp:170-173 because the position is the final tie-break there. */
static void order_by_row_key(const uint32_t* col, uint64_t nnz, const uint64_t* row_key,
                             uint64_t nkeys, uint64_t* order) {
  uint64_t* start = (uint64_t*)calloc(nkeys + 1, sizeof(uint64_t));
  for (uint64_t i = 0; i < nnz; ++i) start[row_key[col[i]] + 1]++;
  for (uint64_t k = 0; k < nkeys; ++k) start[k + 1] += start[k];
  for (uint64_t i = 0; i < nnz; ++i) order[start[row_key[col[i]]]++] = i;
  free(start);
}

int orc_build_plan(uint32_t n, const uint32_t* dims, uint64_t nnz, const uint32_t* coords,
                   uint32_t mode, uint64_t kappa, int strategy, int policy, int* scheme,
                   uint64_t* order, uint64_t* offsets, uint32_t* owned_flat,
                   uint64_t* owned_offsets) {
  /* layout.hpp:135, layout.cpp:25-28, layout.hpp:139-146 */
  if (kappa < 1) FAIL("layout: kappa must be at least 1");
  if (mode >= n) FAIL("layout: mode out of range");
  const uint32_t extent = dims[mode];
  int s1 = policy == 1 ? 1 : (policy == 2 ? 0 : ((uint64_t)extent >= kappa));
  *scheme = s1 ? 1 : 2;

  /* tensor.hpp:87-92 mode_column */
  uint32_t* col = (uint32_t*)malloc((nnz ? nnz : 1) * sizeof(uint32_t));
  for (uint64_t i = 0; i < nnz; ++i) col[i] = coords[i * n + mode];
  uint64_t* row_key = (uint64_t*)malloc((uint64_t)extent * sizeof(uint64_t));

  if (s1) {
    /* layout.cpp:76-84 degrees */
    uint64_t* deg = (uint64_t*)calloc(extent, sizeof(uint64_t));
    for (uint64_t i = 0; i < nnz; ++i) deg[col[i]]++;
    /* layout.cpp:90-99 degree-ordered vertices */
    vdeg* verts = (vdeg*)malloc(((uint64_t)extent + 1) * sizeof(vdeg));
    uint64_t nv = 0;
    for (uint32_t i = 0; i < extent; ++i)
      if (deg[i]) {
        verts[nv].deg = deg[i];
        verts[nv].idx = i;
        ++nv;
      }
    qsort(verts, nv, sizeof(vdeg), cmp_vdeg);
    /* layout.cpp:125-138 assignment (cyclic k % kappa, or LPT with first-minimum ties) */
    uint32_t* part = (uint32_t*)malloc((uint64_t)extent * sizeof(uint32_t));
    uint64_t* load = (uint64_t*)calloc(kappa, sizeof(uint64_t));
    uint64_t* cnt = (uint64_t*)calloc(kappa + 1, sizeof(uint64_t));
    for (uint32_t i = 0; i < extent; ++i) part[i] = UINT32_MAX;
    for (uint64_t k = 0; k < nv; ++k) {
      uint64_t z;
      if (strategy == 0) {
        z = k % kappa;
      } else {
        z = 0;
        for (uint64_t q = 1; q < kappa; ++q)
          if (load[q] < load[z]) z = q;
      }
      part[verts[k].idx] = (uint32_t)z;
      load[z] += verts[k].deg;
      cnt[z + 1]++;
    }
    /* layout.cpp:139 owned sorted ascending; rows ordered by (partition, coordinate) */
    for (uint64_t z = 0; z < kappa; ++z) cnt[z + 1] += cnt[z];
    for (uint64_t z = 0; z <= kappa; ++z) owned_offsets[z] = cnt[z];
    uint64_t* fill = (uint64_t*)malloc((kappa + 1) * sizeof(uint64_t));
    memcpy(fill, cnt, (kappa + 1) * sizeof(uint64_t));
    for (uint32_t i = 0; i < extent; ++i)
      if (part[i] != UINT32_MAX) {
        uint64_t pos = fill[part[i]]++;
        owned_flat[pos] = i;
        row_key[i] = pos;
      } else {
        row_key[i] = 0; /* never referenced: degree 0 */
      }
    /* layout.cpp:141-151 element order */
    order_by_row_key(col, nnz, row_key, nv ? nv : 1, order);
    /* layout.cpp:153-155 sizes -> offsets */
    offsets[0] = 0;
    for (uint64_t z = 0; z < kappa; ++z) offsets[z + 1] = offsets[z] + load[z];
    free(deg);
    free(verts);
    free(part);
    free(load);
    free(cnt);
    free(fill);
  } else {
    /* layout.cpp:159-183 */
    for (uint32_t i = 0; i < extent; ++i) row_key[i] = i;
    order_by_row_key(col, nnz, row_key, extent, order);
    const uint64_t base = nnz / kappa, rem = nnz % kappa;
    offsets[0] = 0;
    for (uint64_t z = 0; z < kappa; ++z) offsets[z + 1] = offsets[z] + base + (z < rem ? 1 : 0);
    for (uint64_t z = 0; z <= kappa; ++z) owned_offsets[z] = 0;
  }
  free(col);
  free(row_key);
  return 0;
}

/* oracle.hpp:20-43 */
int orc_mttkrp(uint32_t n, const uint32_t* dims, uint64_t nnz, const uint32_t* coords,
               const float* values, uint64_t rank, const float* factors, uint32_t mode,
               float* out) {
  if (mode >= n) FAIL("oracle: mode out of range");
  const float* f[16];
  uint64_t off = 0;
  for (uint32_t w = 0; w < n && w < 16; ++w) {
    f[w] = factors + off;
    off += (uint64_t)dims[w] * rank;
  }
  memset(out, 0, (uint64_t)dims[mode] * rank * sizeof(float));
  for (uint64_t i = 0; i < nnz; ++i) {
    const uint32_t* c = coords + i * n;
    for (uint64_t r = 0; r < rank; ++r) {
      float term = values[i];
      for (uint32_t w = 0; w < n; ++w)
        if (w != mode) term *= f[w][(uint64_t)c[w] * rank + r];
      out[(uint64_t)c[mode] * rank + r] += term;
    }
  }
  return 0;
}

/* oracle.hpp:20-43 with T = double on the fp32 inputs widened exactly to double (the
 * reference's fp64 instantiation: SparseTensorCOO<double>, FactorMatrix<double>).  Each
 * output row is summed in element order, so splitting the OUTPUT ROWS across threads (every
 * thread scans all elements and keeps the ones whose row it owns) is bitwise identical to the
 * reference's single loop. */
typedef struct {
  uint32_t n, mode;
  const uint32_t* dims;
  uint64_t nnz, rank;
  const uint32_t* coords;
  const float* values;
  const float* f[16];
  double* out;
  uint32_t r0, r1;
} orc_f64_job;

static void* orc_f64_worker(void* arg) {
  const orc_f64_job* j = (const orc_f64_job*)arg;
  const uint32_t n = j->n, d = j->mode;
  const uint64_t R = j->rank;
  for (uint64_t i = 0; i < j->nnz; ++i) {
    const uint32_t* c = j->coords + i * n;
    const uint32_t row = c[d];
    if (row < j->r0 || row >= j->r1) continue;
    double* o = j->out + (uint64_t)row * R;
    for (uint64_t r = 0; r < R; ++r) {
      double term = (double)j->values[i];
      for (uint32_t w = 0; w < n; ++w)
        if (w != d) term *= (double)j->f[w][(uint64_t)c[w] * R + r];
      o[r] += term;
    }
  }
  return NULL;
}

int orc_mttkrp_f64(uint32_t n, const uint32_t* dims, uint64_t nnz, const uint32_t* coords,
                   const float* values, uint64_t rank, const float* factors, uint32_t mode,
                   double* out, uint32_t threads) {
  if (mode >= n) FAIL("oracle: mode out of range");
  if (n > 16) FAIL("oracle: too many modes");
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (threads > dims[mode]) threads = dims[mode];
  orc_f64_job jobs[256];
  pthread_t tids[256];
  uint64_t off = 0;
  const float* f[16];
  for (uint32_t w = 0; w < n; ++w) {
    f[w] = factors + off;
    off += (uint64_t)dims[w] * rank;
  }
  memset(out, 0, (uint64_t)dims[mode] * rank * sizeof(double));
  for (uint32_t t = 0; t < threads; ++t) {
    orc_f64_job* j = &jobs[t];
    j->n = n;
    j->mode = mode;
    j->dims = dims;
    j->nnz = nnz;
    j->rank = rank;
    j->coords = coords;
    j->values = values;
    memcpy(j->f, f, sizeof f);
    j->out = out;
    j->r0 = (uint32_t)((uint64_t)dims[mode] * t / threads);
    j->r1 = (uint32_t)((uint64_t)dims[mode] * (t + 1) / threads);
  }
  uint32_t started = 0;
  for (uint32_t t = 1; t < threads; ++t) {
    if (pthread_create(&tids[t], NULL, orc_f64_worker, &jobs[t]) != 0) break;
    started = t;
  }
  orc_f64_worker(&jobs[0]);
  for (uint32_t t = 1; t <= started; ++t) pthread_join(tids[t], NULL);
  for (uint32_t t = started + 1; t < threads; ++t) orc_f64_worker(&jobs[t]);
  return 0;
}

/* verify.hpp:21-39 against an fp64 want: max |g-w| / max(1,|w|). */
double orc_max_rel_err_f64(const float* got, const double* want, uint64_t count) {
  double worst = 0.0;
  for (uint64_t i = 0; i < count; ++i) {
    double g = got[i], w = want[i];
    double den = fabs(w) > 1.0 ? fabs(w) : 1.0;
    double e = fabs(g - w) / den;
    if (e != e) return INFINITY;
    if (e > worst) worst = e;
  }
  return worst;
}

/* verify.hpp:21-39 */
double orc_max_rel_err(const float* got, const float* want, uint64_t count) {
  double worst = 0.0;
  for (uint64_t i = 0; i < count; ++i) {
    double g = got[i], w = want[i];
    double den = fabs(w) > 1.0 ? fabs(w) : 1.0;
    double e = fabs(g - w) / den;
    if (e != e) return INFINITY;
    if (e > worst) worst = e;
  }
  return worst;
}
