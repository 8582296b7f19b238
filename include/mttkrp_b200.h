/*
 * mttkrp_b200.h — C ABI of the B200-native all-mode spMTTKRP library
 * (libmttkrp_b200.so, built from paper_2503_18198_b200/csrc for sm_100a).
 *
 * The reference (arxiv 2503.18198 CPU model, /root/reference/proj/core) exposes no FFI:
 * its boundary is the header-only C++ template API in namespace `mttkrp`.  Every entry
 * point below replaces one call of that API; the reference file:line is cited on each.
 * The C++ drop-in layer include/mttkrp_b200/mttkrp.hpp re-exposes the reference's names
 * and exception messages on top of these functions.
 *
 * Conventions: plain pointers and sizes only; host buffers are caller-owned; every
 * function returns an mk_status and on failure stores a message retrievable with
 * mk_last_error() (thread-local).  A context is driven by one host thread at a time.
 * Index type is uint32 (types.hpp:14), values fp32.
 */
#ifndef MTTKRP_B200_H
#define MTTKRP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MK_OK = 0,
  MK_EINVAL = 1,     /* argument / shape / plan validation (reference: throw mttkrp::error) */
  MK_ENOMEM = 2,     /* device or host allocation failed */
  MK_ECUDA = 3,      /* CUDA runtime / launch failure */
  MK_ENONFINITE = 4, /* non-finite partial product (kernel.hpp:109-114) */
  MK_ESTATE = 5,     /* call-order error (e.g. no tensor uploaded) */
  MK_ENCCL = 6       /* multi-GPU collective failure */
} mk_status;

/* Scheme / Strategy / SchemePolicy enums (layout.hpp:17-24). */
enum { MK_SCHEME1 = 1, MK_SCHEME2 = 2 };
enum { MK_CYCLIC = 0, MK_LEAST_LOADED = 1 };
enum { MK_ADAPTIVE = 0, MK_SCHEME1_ONLY = 1, MK_SCHEME2_ONLY = 2 };

/* Execution flags for the MTTKRP entry points. */
enum {
  MK_EXEC_FAST = 0,          /* tile-parallel, atomics only on tile-split rows (1e-5 class) */
  MK_EXEC_DETERMINISTIC = 1, /* one owner per output row, element order, no FMA:
                                bitwise equal to ExecConfig{deterministic=true}
                                (kernel.hpp:26-28) and to oracle_mttkrp (oracle.hpp:20-43) */
  MK_EXEC_PARTITIONED = 2,   /* the reference's work split: partition z of the plan on CTA z
                                (for_each_partition, parallel.hpp:16-49; Algorithm 2), atomics
                                only where Scheme 2 partitions or the CTA-internal split cut a
                                row; the GPU form of the paper's scheme ablation (fp32 only) */
  MK_EXEC_REFERENCE = 3,     /* the reference's parallel-executor contract (
                                kernel.hpp:117-121): Scheme 1 copies own their rows and sum in
                                copy order, so they run the deterministic kernel (bitwise equal
                                to MK_EXEC_DETERMINISTIC); Scheme 2 copies run MK_EXEC_FAST.
                                The C++ drop-in's ExecConfig{deterministic=false} default */
};

typedef struct mk_context mk_context;

typedef struct {
  int scheme;              /* MK_SCHEME1 / MK_SCHEME2 (ModePlan::scheme, layout.hpp:49) */
  uint64_t kappa;          /* ModePlan::kappa */
  uint64_t nnz;            /* ModePlan::nnz() */
  uint64_t owned_total;    /* Σ owned_indices[z].size() (Scheme 1), 0 for Scheme 2 */
  uint64_t distinct_rows;  /* DegreeProfile::distinct() (layout.hpp:38-42) */
  uint64_t split_rows;     /* rows the fast kernel updates atomically (tile boundaries) */
  uint64_t device_bytes;   /* bytes of the materialised mode copy on the device */
} mk_plan_info;

/* How the fast path (MK_EXEC_FAST) runs one mode copy: which streaming kernel the one-time
 * timing chose and the level-ordered kernel's shared-memory plan. */
typedef struct {
  int kernel;               /* 0 level-ordered streaming, 1 fiber-ordered streaming,
                               2 generic tiles, -1 not chosen yet (no fast launch so far) */
  int blocked;              /* level-ordered: copy split into shared-memory blocks */
  uint32_t blocks;          /* level-ordered: blocks (1 when unblocked) */
  uint32_t staged_levels;   /* level-ordered: inner levels staged in shared memory */
  int outer_level;          /* level-ordered: outermost input level kept in registers */
  uint32_t launches;        /* kernel launches per fast call of this mode */
  uint64_t stream_bytes;    /* bytes streamed from HBM per call (records + slow keys) */
} mk_fast_info;

/* ---- library / context ------------------------------------------------------------ */
const char* mk_last_error(void);
const char* mk_version(void);
int mk_device_count(int* count);
/* streaming multiprocessors of `device` (the CLI's default kappa for the GPU backend) */
int mk_device_sm_count(int device, int* sms);
int mk_create(int device, mk_context** out);
int mk_destroy(mk_context* ctx);
/* Run all work on an external CUDA stream (cudaStream_t passed as void*).  NULL is the
 * CUDA default (legacy) stream, as everywhere in CUDA; MK_OWN_STREAM restores the
 * context's own non-blocking stream. */
#define MK_OWN_STREAM ((void*)(intptr_t)-1)
int mk_set_stream(mk_context* ctx, void* cuda_stream);
int mk_synchronize(mk_context* ctx);

/* ---- tensor: SparseTensorCOO<float>::from_parts (tensor.hpp:45-55) ---------------
 * coords_aos is nnz × n_modes (element-major, tensor.hpp:80-82).  Validated on device
 * with the reference's messages ("tensor: coordinate C out of range for mode H",
 * "tensor: non-finite element value"). */
int mk_tensor_upload(mk_context* ctx, uint32_t n_modes, const uint32_t* dims, uint64_t nnz,
                     const uint32_t* coords_aos, const float* values);
/* SparseTensorCOO<double>::from_parts (tensor.hpp:45-55, T = double).  An fp64 tensor is
 * driven through the _f64 entry points only (the fp32 ones fail with MK_EINVAL, as the
 * reference's templates do not mix T). */
int mk_tensor_upload_f64(mk_context* ctx, uint32_t n_modes, const uint32_t* dims, uint64_t nnz,
                         const uint32_t* coords_aos, const double* values);
/* Σ val² of the uploaded tensor (||X||_F², for the CPD fit). */
int mk_tensor_norm2(mk_context* ctx, double* norm2);

/* ---- format build + partition: build_mode_plans (layout.hpp:131-149) ---------------
 * Builds all N mode-specific copies on the device (GPU histogram + stable radix sorts,
 * layout.cpp:76-183) and materialises each as SoA (N uint32 index arrays + fp32 values)
 * in that mode's order. */
int mk_build_plans(mk_context* ctx, uint64_t kappa, int strategy, int policy);
int mk_get_plan_info(mk_context* ctx, uint32_t mode, mk_plan_info* info);
/* Fast-path kernel choice and plan of a mode copy (valid after a fast launch). */
int mk_fast_path_info(mk_context* ctx, uint32_t mode, mk_fast_info* info);
/* Force the fast path's kernel for every mode (0 level-ordered, 1 fiber-ordered, 2 generic
 * tiles) or restore the one-time timed choice (-1).  A forced kernel that has no
 * specialisation for the shape falls back along 0 -> 1 -> 2. */
int mk_set_fast_kernel(mk_context* ctx, int kernel);
/* How the fast path picks its kernel and shared-memory plan per mode copy (no reference
 * counterpart: the reference has one executor).  MK_PLAN_TIMED (default): the first fast call
 * of a mode times the candidates on the actual inputs (L2 flushed) and keeps the fastest.
 * MK_PLAN_MODEL: the cost model's choice, no timing -- a pure function of the tensor, rank,
 * kappa and device SM count, so the plan (and mk_fast_path_info) is the same on every run
 * and box.  Resets the per-mode choices. */
enum { MK_PLAN_TIMED = 0, MK_PLAN_MODEL = 1 };
int mk_set_plan_mode(mk_context* ctx, int mode);
/* ModePlan export (layout.hpp:47-64): order[nnz], partition_offsets[kappa+1],
 * owned_flat[owned_total] (concatenated owned_indices), owned_offsets[kappa+1].
 * Any output pointer may be NULL to skip it. */
int mk_plan_export(mk_context* ctx, uint32_t mode, uint64_t* order, uint64_t* partition_offsets,
                   uint32_t* owned_flat, uint64_t* owned_offsets);
/* mode_degrees (layout.hpp:106-111): degrees[extent]. */
int mk_mode_degrees(mk_context* ctx, uint32_t mode, uint64_t* degrees);
/* The materialised mode copy (parity/inspection): idx is n_modes × nnz, mode-major. */
int mk_copy_export(mk_context* ctx, uint32_t mode, uint32_t* idx, float* values);

/* ---- factors: FactorMatrix<float> (factor.hpp:16-48), row-major I_d × R --------------- */
int mk_factors_upload(mk_context* ctx, uint32_t rank, const float* const* factors);
int mk_factor_upload(mk_context* ctx, uint32_t mode, const float* factor);
int mk_factor_download(mk_context* ctx, uint32_t mode, float* factor);

/* ---- fp64 path: the reference's T = double instantiation ---------------
 * FactorMatrix<double> (factor.hpp:16-48); mttkrp_mode / mttkrp_all_modes<double>
 * (kernel.hpp:161-197).  Usable on an fp64 tensor and on an fp32 tensor (values widened
 * exactly).  MK_EXEC_DETERMINISTIC is bitwise equal to oracle_mttkrp<double>
 * (oracle.hpp:20-43); MK_EXEC_FAST is within verify_tolerance<double> = 1e-12. */
int mk_factors_upload_f64(mk_context* ctx, uint32_t rank, const double* const* factors);
int mk_mttkrp_mode_f64(mk_context* ctx, uint32_t mode, int exec, double* out);
int mk_mttkrp_all_modes_f64(mk_context* ctx, int chain, int exec, double* const* outs);

/* ---- spMTTKRP -------------------------------------------------------------------
 * mttkrp_mode (kernel.hpp:161-169): one mode from the current factors into out[I_d × R]. */
int mk_mttkrp_mode(mk_context* ctx, uint32_t mode, int exec, float* out);
/* mttkrp_all_modes (kernel.hpp:177-197); chain != 0 feeds each output to later modes. */
int mk_mttkrp_all_modes(mk_context* ctx, int chain, int exec, float* const* outs);
/* Device-resident sweep (Algorithm 1): enqueue only, outputs stay in
 * the context.  mk_synchronize() surfaces errors (non-finite detection). */
int mk_sweep_async(mk_context* ctx, int chain, int exec);
/* One mode of the sweep, enqueue only (reads the context's input factors). */
int mk_mttkrp_mode_async(mk_context* ctx, uint32_t mode, int exec);
int mk_output_download(mk_context* ctx, uint32_t mode, float* out);
/* End-to-end step as a caller sees it: H2D of all factors from host memory, the sweep,
 * D2H of all outputs, synchronise.  When the host matrices are packed in one allocation in
 * mode order (factor w at float offset sum_{v<w} I_v*R, every I_v*R a multiple of 32, e.g.
 * R = 32 or 64), each direction is ONE copy; otherwise one copy per mode. */
int mk_sweep_host(mk_context* ctx, const float* const* factors, float* const* outs, int chain,
                  int exec);
/* Whether the last all-mode sweep ran as one fused launch (1) or one launch per mode (0). */
int mk_last_sweep_fused(mk_context* ctx, int* fused);
/* run_timed analogue (kernel.hpp:239-287) timed with CUDA events on the context stream.
 * mode_ms[iters × N] and total_ms[iters]; flush_l2 writes a 2×L2 buffer between
 * iterations (outside the timed events).  *outputs_bit_identical (may be NULL) = whether
 * every iteration's outputs equal the first's bit for bit (TimingReport, kernel.hpp:271-276;
 * the fast path's float atomics need not be). */
int mk_run_timed(mk_context* ctx, uint64_t iters, int exec, int flush_l2, double* mode_ms,
                 double* total_ms, int* outputs_bit_identical);
/* L2 flush as used by mk_run_timed (enqueued on the context stream). */
int mk_flush_l2(mk_context* ctx);

/* ---- CPD-ALS (absent in the reference; hook kernel.hpp:171-176) ----------
 * One ALS iteration over all modes on the current factors: per mode d,
 * M = MTTKRP(d); V = ⊛_{w≠d} Y_wᵀY_w; Y_d = M V⁻¹; column 2-norms -> lambda; then the
 * fit 1 - ||X - X̂|| / ||X||.  lambda[R] may be NULL. */
int mk_cpd_als_iter(mk_context* ctx, double* fit, float* lambda);
/* Full driver: up to max_iters iterations, stops when |Δfit| < tol. */
int mk_cpd_als(mk_context* ctx, uint64_t max_iters, double tol, double* fit,
               uint64_t* iters_done, float* lambda);

/* ---- multi-GPU shards of the mode copies (no reference counterpart) --------
 * Rank `rank` of `world` owns, in every mode copy, the element range [e_rank, e_rank+1)
 * (mk_shard_split: nnz-balanced cuts moved to the next row start, except inside a heavy row
 * of more than nnz/(8 world) elements, which is split between ranks).  It touches the copy
 * rows [k0, k1) — whole rows plus at most one partial row at each end.  Subsequent fast,
 * deterministic and fp64 MTTKRP calls compute only the owned elements.  world = 1 restores
 * the full copy. */
int mk_set_shard(mk_context* ctx, uint32_t rank, uint32_t world);
/* Copy rows [k0, k1) touched by `rank` in `mode` (any rank of the current world). */
int mk_shard_rows(mk_context* ctx, uint32_t mode, uint32_t rank, uint64_t* k0, uint64_t* k1);
/* Element range [e0, e1) and touched copy rows [k0, k1) of `rank` (NULL outputs skipped). */
int mk_shard_range(mk_context* ctx, uint32_t mode, uint32_t rank, uint64_t* e0, uint64_t* e1,
                   uint64_t* k0, uint64_t* k1);
/* Pack this rank's output rows k0..k1-1 of `mode` (copy-row order, R floats each; the end
 * rows may be partial sums) into dst (device). */
int mk_shard_pack(mk_context* ctx, uint32_t mode, float* dst_device);
/* Scatter an all-gathered buffer (world blocks of stride_rows rows, device) into the output
 * of `mode` in row-index order, summing the partial sums of split rows in rank order. */
int mk_shard_unpack(mk_context* ctx, uint32_t mode, const float* src_device,
                    uint64_t stride_rows);
/* Host helpers on a CSR row pointer (row_ptr[nrows] = nnz), cuts[world + 1]:
 * mk_shard_cuts — copy-row cuts (first row starting at or after floor(r nnz / world));
 * mk_shard_split — the element cuts mk_set_shard uses (heavy rows split). */
int mk_shard_cuts(const uint32_t* row_ptr, uint64_t nrows, uint32_t world, uint64_t* cuts);
int mk_shard_split(const uint32_t* row_ptr, uint64_t nrows, uint32_t world, uint64_t* ecuts);
/* NCCL inside the library (one process per GPU; libnccl.so.2 is opened on first use).
 * Rank 0 creates the unique id (MK_NCCL_ID_BYTES opaque bytes) and the caller's launcher
 * hands it to every rank (any channel: MPI, a file, torch.distributed); mk_comm_init then
 * builds the communicator and applies mk_set_shard(rank, world) to the context's plans. */
#define MK_NCCL_ID_BYTES 128
int mk_comm_unique_id(void* id);
int mk_comm_init(mk_context* ctx, uint32_t world, uint32_t rank, const void* id);
int mk_comm_destroy(mk_context* ctx);
/* The sharded all-mode sweep (unchained, like run_timed, kernel.hpp:239-287): per mode the
 * rank's spMTTKRP, pack, ncclAllGather over NVLink, unpack — every rank ends with all N
 * outputs.  Enqueued on the context stream (mk_synchronize surfaces errors); captured into
 * a CUDA graph from the second call on (MKB_GRAPH=0 disables). */
int mk_sweep_sharded(mk_context* ctx);
/* One CPD-ALS iteration with the per-mode exchange; factors stay replicated. */
int mk_cpd_als_iter_sharded(mk_context* ctx, double* fit, float* lambda);
/* CPD-ALS pieces for a sharded driver: the Gram/solve/normalise update of mode d from the
 * (gathered) MTTKRP output, and the fit after the last mode. */
int mk_als_update_mode(mk_context* ctx, uint32_t mode);
int mk_als_fit(mk_context* ctx, double* fit, float* lambda);
/* Device pointer of the MTTKRP output of `mode` (I_d x R fp32), for external collectives. */
int mk_output_device_ptr(mk_context* ctx, uint32_t mode, void** ptr);

/* ---- host-side tensor ingest (synthetic.hpp:58-158, factor.hpp:71-84) ---------------
 * Bit-identical to the reference generator (same draw sequence), multi-threaded dedup.
 * dist: 0 uniform, 1 mode_skewed. */
int mk_generate_synthetic(uint32_t n_modes, const uint32_t* dims, uint64_t nnz, int dist,
                          uint64_t skew_mode, uint64_t skew_distinct, uint64_t seed,
                          uint32_t* coords_aos, float* values);
/* DESIGN.md §5 power-law (Zipf) generator for the nips-shaped config. */
int mk_generate_powerlaw(uint32_t n_modes, const uint32_t* dims, uint64_t nnz, double exponent,
                         uint64_t seed, uint32_t* coords_aos, float* values);
int mk_random_factors(uint32_t n_modes, const uint32_t* dims, uint64_t rank, uint64_t seed,
                      float* const* factors);
/* T = double variants (rng.hpp:37-39 unit_open_closed<double>; same draw sequence). */
int mk_generate_synthetic_f64(uint32_t n_modes, const uint32_t* dims, uint64_t nnz, int dist,
                              uint64_t skew_mode, uint64_t skew_distinct, uint64_t seed,
                              uint32_t* coords_aos, double* values);
int mk_random_factors_f64(uint32_t n_modes, const uint32_t* dims, uint64_t rank, uint64_t seed,
                          double* const* factors);

/* ---- FROSTT text and binary tensor cache (frostt.hpp:19-211) -----------
 * Multithreaded parse with the reference's semantics and error texts ("frostt: line N: ..."):
 * 1-based indices, '#' comments and blank lines skipped, values parsed in `prec` (32 / 64)
 * precision with std::from_chars, duplicates summed in file order into the first occurrence
 * (merge_duplicates != 0, FrosttOptions::merge_duplicates) or rejected, extents inferred
 * unless n_override > 0 (FrosttOptions::dims_override).  threads = 0: all host threads.
 * The result is a host tensor handle; read it with mk_host_tensor_info/_export, free it with
 * mk_host_tensor_free. */
typedef struct mk_host_tensor mk_host_tensor;
int mk_frostt_parse(const char* text, uint64_t len, int prec, int merge_duplicates,
                    const uint32_t* dims_override, uint32_t n_override, uint32_t threads,
                    mk_host_tensor** out);                       /* parse_frostt, frostt.hpp:74 */
int mk_frostt_read_file(const char* path, int prec, int merge_duplicates,
                        const uint32_t* dims_override, uint32_t n_override, uint32_t threads,
                        mk_host_tensor** out);                   /* read_frostt_file, :194-199 */
int mk_host_tensor_info(const mk_host_tensor* t, uint32_t* n_modes, uint32_t* dims,
                        uint32_t dims_capacity, uint64_t* nnz, uint64_t* duplicates_merged,
                        int* prec);                              /* FrosttParseResult, :31-35 */
/* coords_aos: nnz*n_modes uint32; values: nnz floats (prec 32) or doubles (prec 64). */
int mk_host_tensor_export(const mk_host_tensor* t, uint32_t* coords_aos, void* values);
int mk_host_tensor_free(mk_host_tensor* t);
/* write_frostt (frostt.hpp:165-186): 1-based indices, shortest round-trip values.  With
 * buf == NULL only *len (bytes) is returned. */
int mk_frostt_format(uint32_t n_modes, uint64_t nnz, const uint32_t* coords_aos,
                     const void* values, int prec, uint32_t threads, char* buf, uint64_t cap,
                     uint64_t* len);
int mk_frostt_write_file(const char* path, uint32_t n_modes, uint64_t nnz,
                         const uint32_t* coords_aos, const void* values, int prec,
                         uint32_t threads);                      /* write_frostt_file, :201-206 */
/* Binary tensor cache ("MKBT" v1, checksummed; no reference counterpart). */
int mk_tensor_cache_write(const char* path, uint32_t n_modes, const uint32_t* dims, uint64_t nnz,
                          const uint32_t* coords_aos, const void* values, int prec);
int mk_tensor_cache_read(const char* path, mk_host_tensor** out);

#ifdef __cplusplus
}
#endif
#endif /* MTTKRP_B200_H */
