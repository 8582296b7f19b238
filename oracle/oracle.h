/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the B200 spMTTKRP path.
 *
 * A plain-C restatement of the reference algorithm (arxiv 2503.18198 CPU model under
 * /root/reference/proj/core).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / reference arm may load it, and only as the checker.  The product
 * (paper_2503_18198_b200/) never links or calls anything in oracle/.
 *
 * Pinned against: the reference built from its own sources (oracle/_ref, see
 * oracle/Makefile) and the reference's golden fixtures (tests/golden/, made by
 * tests/golden/make_golden.py).  See DESIGN.md §3.
 */
#ifndef MK_ORACLE_H
#define MK_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);

/* rng.hpp:22-39 */
typedef struct {
  uint64_t mt[312];
  int mti;
} orc_engine;
void orc_seeded(orc_engine* g, uint64_t seed, uint64_t stream);
uint64_t orc_next(orc_engine* g);
uint64_t orc_bounded(orc_engine* g, uint64_t n);

/* synthetic.hpp:58-158.  dist 0 = uniform, 1 = mode_skewed. */
int orc_generate_synthetic(uint32_t n, const uint32_t* dims, uint64_t nnz, int dist,
                           uint64_t skew_mode, uint64_t skew_distinct, uint64_t seed,
                           uint32_t* coords_out, float* values_out);
/* Power-law generator specified in DESIGN.md §5 (no reference counterpart). */
int orc_generate_powerlaw(uint32_t n, const uint32_t* dims, uint64_t nnz, double exponent,
                          uint64_t seed, uint32_t* coords_out, float* values_out);
/* factor.hpp:71-84: concatenated row-major factors of every mode. */
int orc_random_factors(uint32_t n, const uint32_t* dims, uint64_t rank, uint64_t seed,
                       float* out);

/* layout.cpp:76-183 + layout.hpp:131-149.  strategy 0 cyclic / 1 least_loaded;
 * policy 0 adaptive / 1 s1-only / 2 s2-only.  scheme out: 1 or 2. */
int orc_build_plan(uint32_t n, const uint32_t* dims, uint64_t nnz, const uint32_t* coords,
                   uint32_t mode, uint64_t kappa, int strategy, int policy, int* scheme,
                   uint64_t* order, uint64_t* offsets, uint32_t* owned_flat,
                   uint64_t* owned_offsets);

/* oracle.hpp:20-43 (fp32, element order, term = val; term *= Y_w for w ascending). */
int orc_mttkrp(uint32_t n, const uint32_t* dims, uint64_t nnz, const uint32_t* coords,
               const float* values, uint64_t rank, const float* factors_concat, uint32_t mode,
               float* out);

/* oracle.hpp:20-43 with T = double (fp32 inputs widened exactly); output rows split across
 * `threads` threads, each row still summed in element order (bitwise = the reference). */
int orc_mttkrp_f64(uint32_t n, const uint32_t* dims, uint64_t nnz, const uint32_t* coords,
                   const float* values, uint64_t rank, const float* factors_concat,
                   uint32_t mode, double* out, uint32_t threads);
double orc_max_rel_err_f64(const float* got, const double* want, uint64_t count);

/* verify.hpp:21-39: max |g-w| / max(1,|w|). */
double orc_max_rel_err(const float* got, const float* want, uint64_t count);

#ifdef __cplusplus
}
#endif
#endif
