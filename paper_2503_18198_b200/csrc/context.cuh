// Device-resident state of one mk_context: the uploaded tensor, the N mode-specific
// copies (the "tensor copies T_d" of Algorithm 1), factors and outputs.
//
// HBM layout per mode d (all arrays in copy order j = 0..nnz-1, i.e. the order of
// ModePlan::order, layout.hpp:51-52):
//   idx[w][j]   uint32  coordinate of mode w of element order[j]       (N arrays, SoA)
//   val[j]      fp32    value of element order[j]
//   order[j]    uint32  original element position (exported as uint64)
//   row_seq[k]  uint32  k-th non-empty output row in copy order       (V entries)
//   row_ptr[k]  uint32  first copy position of row_seq[k]               (V+1 entries)
//   zero_rows   uint32  rows the fast kernel must pre-zero: empty rows + tile-split rows
// A Scheme 1 copy has rows grouped by partition (owned rows ascending inside a partition);
// a Scheme 2 copy has rows ascending.  Both are one contiguous run per output row, which
// is what lets one kernel serve both schemes.
#pragma once

#include <cstdint>
#include <vector>

#include "common.cuh"
#include "sort.cuh"

namespace mkb {

constexpr int kMaxModes = 8;

struct ModeCopy {
  int scheme = MK_SCHEME1;
  uint64_t kappa = 1;
  uint64_t owned_total = 0;
  uint64_t distinct = 0;  // V: rows with degree > 0
  DevBuf<uint32_t> idx[kMaxModes];
  DevBuf<float> val;
  DevBuf<double> val64;  // fp64 path (mttkrp64.cu): values in copy order, built on first use
  DevBuf<uint32_t> order;
  DevBuf<uint32_t> row_seq;  // rows in copy order: [0,V) non-empty, [V,extent) empty
  DevBuf<uint32_t> row_ptr;  // V+1
  DevBuf<uint32_t> zero_rows;
  uint64_t n_zero_rows = 0;
  uint64_t n_split_rows = 0;
  uint32_t tile = 256;  // fast-kernel tile length (nnz), chosen per copy at build time
  std::vector<uint64_t> partition_offsets;  // kappa+1 (host)
  std::vector<uint64_t> owned_offsets;      // kappa+1 (host); rows = row_seq[...]
  DevBuf<uint32_t> degrees;                 // extent
  // partitioned executor (mttkrp.cu launch_partitioned): per-lane-group tile bounds
  DevBuf<uint64_t> part_tiles;
  uint32_t part_gpb = 0;
  uint64_t part_tiles_kappa = 0;
  // packed element records for the streaming kernel (stream.cu): part A 16 B/element,
  // part B 0/4/8/16 B/element; padded to a multiple of 4 elements
  DevBuf<uint32_t> recA, recB;
  DevBuf<uint32_t> kperm;  // kernel (fiber) order -> reference copy position
  uint32_t fiber_mode = kMaxModes;  // input mode accumulated per fiber (== n: off)
  uint32_t rec_modes[kMaxModes] = {};  // record word q -> input mode (extent descending)
  uint64_t fibers = 0;              // (row, c_fiber) runs in kernel order
  // pre-zero row lists (empty rows + rows split by the kernel's segmentation), cached per
  // (kernel, segment length, shard range)
  struct ZeroList {
    DevBuf<uint32_t> rows;
    uint64_t n = 0;
    uint64_t key_seg = 0, key_tile = 0, key_e0 = ~0ull, key_e1 = ~0ull;
  };
  ZeroList zl_stream, zl_tiles;
  // deterministic kernel: copy rows long enough for the one-CTA-per-row path (mttkrp.cu
  // k_mttkrp_rows_long), cached per (threshold, shard range)
  DevBuf<uint32_t> det_long;
  uint64_t det_long_n = 0, det_long_key_min = 0, det_long_key_e0 = ~0ull, det_long_key_e1 = ~0ull;
  // fast-path kernel chosen for this copy by a one-time timing of the candidates
  // (mttkrp.cu): -1 undecided, 0 level-ordered streaming kernel, 1 fiber-ordered streaming
  // kernel, 2 generic tile kernel; keyed by factor rank and shard range
  int fast_kernel = -1;
  uint32_t fast_rank = 0;
  // level-ordered plan autotune: staged-level count to plan for (-1: cost model), and the
  // timed milliseconds of the best plan per staged-level count (< 0: none)
  int s2_force_k = -1;
  bool s2_no_os = false;  // fused sweep: plan without staging the outer factor
  float s2_ms[5] = {-1.f, -1.f, -1.f, -1.f, -1.f};
  uint64_t fast_e0 = ~0ull, fast_e1 = ~0ull;
  // level-ordered, shared-memory-blocked records of the streaming kernel (stream2_plan.cu),
  // built per (factor rank, shard range) on first use
  struct Stream2 {
    bool tried = false, ok = false;
    int k_req = -1;                            // requested staged-level count (-1: model)
    bool no_os = false;                        // planned with the outer factor unstaged
    uint32_t rank = 0;
    uint64_t key_e0 = ~0ull, key_e1 = ~0ull;  // shard range the plan was built for
    unsigned key_grid = 0;                     // CTAs the work split was built for
    uint32_t ni = 0, nout = 0, k = 0, aw = 2;  // input levels, outer levels, staged levels
    uint32_t nt = 512;                         // threads per CTA
    bool os = false;                           // outer factor staged in shared memory
    uint32_t levels[kMaxModes] = {};           // level -> input mode (outermost first)
    uint32_t rowbits = 0, b0 = 0, m0 = 0, m1 = 0, ob = 0, om = 0;
    uint32_t stage_off[4] = {};
    uint32_t outer_off = 0, outer_bytes = 0;
    size_t staged_end = 0;
    bool blocked = false;
    uint32_t nblocks = 1;
    uint64_t outer_runs = 0;                   // distinct (row, level-0 coordinate) pairs
    DevBuf<uint32_t> blk_dev;                  // s2::Blk table
    DevBuf<uint32_t> tiles, kperm;             // tile stream (records + slow keys), kperm
    DevBuf<uint32_t> wdesc, items, cta_items;  // work schedule (grid = SM count)
    uint32_t nitems = 0;
    unsigned grid = 0;
    DevBuf<uint32_t> zero_rows;                // rows to pre-zero (unblocked plans)
    uint64_t n_zero_rows = 0;
  } s2;
  // multi-GPU row-range shard of this copy: copy rows [k0, k1) = elements [e0, e1)
  uint64_t shard_k0 = 0, shard_k1 = 0, shard_e0 = 0, shard_e1 = 0;
  std::vector<uint64_t> shard_cuts;  // world+1: first copy row touched by each rank (+ V)
  std::vector<uint64_t> shard_ecuts;   // world+1 element cut points (mk_shard_split)
  std::vector<uint64_t> shard_krange;  // 2*world: copy rows [k0_r, k1_r) touched by rank r
  bool shard_split_row = false;        // this rank's range starts or ends inside a row
  std::vector<uint32_t> row_ptr_host;
  bool built = false;
};

struct Context {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  size_t l2_bytes = 0;

  // tensor
  uint32_t n = 0;
  std::vector<uint32_t> dims;
  uint64_t nnz = 0;
  DevBuf<uint32_t> cols[kMaxModes];  // original element order, SoA
  DevBuf<float> values;
  DevBuf<double> values64;  // mk_tensor_upload_f64: the fp64 values (original order)
  bool tensor_f64 = false;  // the tensor was uploaded as SparseTensorCOO<double>
  double norm2 = 0.0;

  // plans
  ModeCopy copies[kMaxModes];
  bool plans_built = false;
  uint64_t kappa = 0;
  uint32_t shard_rank = 0, shard_world = 1;
  DevBuf<uint64_t> shard_cuts_dev[kMaxModes];

  // factors / outputs (row-major I_d x R)
  uint32_t rank = 0;
  // factors[w] / outputs[w] are windows into one arena each, at 128-B aligned offsets
  // arena_off[w] (floats): a host layout with the same offsets moves in one copy
  DevBuf<float> factor_arena, output_arena;
  size_t arena_off[kMaxModes + 1] = {};
  DevBuf<float> factors[kMaxModes];
  DevBuf<float> outputs[kMaxModes];
  bool factors_set[kMaxModes] = {};
  // fp64 path: FactorMatrix<double> inputs / outputs
  uint32_t rank64 = 0;
  DevBuf<double> factor64_arena, output64_arena;
  double* factors64[kMaxModes] = {};
  double* outputs64[kMaxModes] = {};

  // device scalars: [0] = min non-finite copy position (uint64, ~0 = none), [1] = mode
  DevBuf<unsigned long long> nonfinite;
  PinnedWord nonfinite_host;
  DevBuf<uint8_t> flush_buf;
  int plan_mode = MK_PLAN_TIMED;  // mk_set_plan_mode
  int s2_grid = 0;  // level-ordered CTAs (0: SM count; CPD-ALS leaves one SM to its inverse)
  int force_fast_kernel = -1;  // mk_set_fast_kernel: -1 timed choice, else 0 / 1 / 2
  DevBuf<uint32_t> s2sync;  // streaming kernel: finished-CTA counter + non-finite flag
  SortScratch scratch;

  // CPD-ALS state
  DevBuf<double> gram;    // N x R x R (fp64)
  DevBuf<double> mtm;     // MᵀM of the current update (fp64; 2 x R x R allocated)
  DevBuf<double> als_ppart;  // per-CTA partial MᵀM (SM count x R x R), reduced in CTA order
  uint32_t mtm_rank = 0;  // rank the accumulators were laid out (and zeroed) for
  DevBuf<unsigned int> als_bar;  // grid barrier counter of the fused update (monotonic)
  unsigned int als_bar_count = 0;
  uint64_t als_epoch = 0;
  DevBuf<float> solve;    // R x R inverse of V (fp32 for the row apply)
  DevBuf<float> lambda;   // R
  DevBuf<double> als_scalars;
  DevBuf<int> als_status;
  DevBuf<unsigned long long> als_prof;  // MKB_ALS_PROF: phase timestamps of the update
  // overlapped inverse: V_d⁻¹ computed on a side stream (one CTA) while mode d's spMTTKRP runs
  // on the other SMs (als.cu als_iteration)
  cudaStream_t als_side = nullptr;
  cudaEvent_t als_ev_upd = nullptr, als_ev_inv = nullptr;
  DevBuf<double> als_vinv;  // R x R
  DevBuf<int> als_vinv_status;  // 1: the Jacobi pseudo-inverse ran
  // host-buffer pipeline of mk_sweep_host (abi.cu): H2D and D2H copy streams, flags
  cudaStream_t io_h2d = nullptr, io_d2h = nullptr;
  cudaEvent_t io_ev_main = nullptr, io_ev_h2d = nullptr, io_ev_d2h = nullptr;
  cudaEvent_t io_ev_f[kMaxModes] = {}, io_ev_done[kMaxModes] = {};  // per-mode pipeline
  DevBuf<uint32_t> io_flags;  // [0, kMaxModes): factor H2D epochs; [kMaxModes, 2k): mode done
  uint32_t io_epoch = 0;
  // the iteration captured as a CUDA graph (als.cu): replayed while the key and the device
  // memory epoch match the capture; the eager iteration before it records its own epoch
  void* als_graph_exec = nullptr;  // cudaGraphExec_t
  uint64_t als_graph_key = ~0ull;
  unsigned long long als_graph_epoch = ~0ull, als_eager_epoch = ~0ull;
  bool grams_valid = false;
  bool last_sweep_fused = false;  // the last sweep() ran as one k_sweep2 launch
  bool sweep_tuned = false;       // tune_sweep decided fused-vs-mix for the current choices

  // NCCL communicator and the sharded sweep's exchange buffers / CUDA graph (comm.cu)
  void* nccl_comm = nullptr;
  uint32_t comm_world = 0;
  DevBuf<float> xsend, xrecv;
  uint64_t xstride[kMaxModes] = {};
  void* graph_exec = nullptr;  // cudaGraphExec_t of the captured sharded sweep
  bool graph_warm = false;     // one eager sweep ran (the fast path's kernel choice is made)
  unsigned long long graph_epoch = 0;  // g_devmem_epoch when the eager sweep / capture ran
};

// One CPD-ALS iteration over all modes (als.cu); fit and optional lambda[R] to host.
void als_iteration(Context& c, double* fit, float* lambda_host);

// Fast-kernel tile length: ~one tile per resident lane group, clamped to [32, 1024].
uint32_t choose_tile(uint64_t nnz, int num_sms);

void tensor_upload(Context& c, uint32_t n, const uint32_t* dims, uint64_t nnz,
                   const uint32_t* coords_aos, const float* values);
void build_plans(Context& c, uint64_t kappa, int strategy, int policy);

// Enqueue MTTKRP of `mode` reading factors in[w] and writing out (I_d x R).
void launch_mttkrp(Context& c, uint32_t mode, const float* const* in, float* out, int exec);
void reset_nonfinite(Context& c);
// Empty rows + rows that continue across a segment start.  Segment starts are
// e0a + t*tile + g*seg (g < tile/seg) inside [e0, e1).
void ensure_zero_list(Context& c, uint32_t mode, ModeCopy::ZeroList& zl, uint32_t seg,
                      uint32_t tile, uint64_t e0a, uint64_t e0, uint64_t e1);
// Multi-GPU row-range shards (shard.cu).
void set_shard(Context& c, uint32_t rank, uint32_t world);
void shard_pack(Context& c, uint32_t mode, float* dst);
void shard_unpack(Context& c, uint32_t mode, const float* src, uint64_t stride_rows);
// NCCL communicator + sharded sweep / ALS iteration (comm.cu)
void comm_unique_id(void* id128);
void comm_init(Context& c, uint32_t world, uint32_t rank, const void* unique_id);
void comm_destroy(Context& c);
void invalidate_graph(Context& c);
void sweep_sharded(Context& c);
void als_iteration_sharded(Context& c, double* fit, float* lambda_host);
// ALS pieces (als.cu), used by the single-GPU iteration and the sharded driver.
void als_prepare(Context& c);
void als_update_mode(Context& c, uint32_t d, bool pre_inverse = false);
void als_fit(Context& c, double* fit, float* lambda_host);
// Streaming TMA kernel (stream.cu); false when the shape has no specialisation.
bool launch_stream(Context& c, uint32_t mode, const float* const* in, float* out);
bool prepare_stream(Context& c, uint32_t mode);  // builds its records; false: no specialisation
// Fast-path kernel selection (mttkrp.cu): 0 level-ordered, 1 fiber-ordered, 2 tiles.
int choose_fast_kernel(Context& c, uint32_t mode, const float* const* in, float* out);
// Unchained fast sweep whose per-mode timed choices mix kernels: time that mix against every
// mode on the level-ordered kernel as ONE fused launch, keep the faster (mttkrp.cu).
void tune_sweep(Context& c, const float* const* in, float* const* outs);
void flush_l2(Context& c);  // write 2x the L2 size on the context's stream
void pack_records(Context& c, uint32_t mode, const uint32_t* rank_of_row);
// v2 level-ordered streaming kernel (stream2_plan.cu): records built per factor rank on first
// use (or eagerly by prepare_stream2); false when the shape has no specialisation.
bool prepare_stream2(Context& c, uint32_t mode);
bool launch_stream2(Context& c, uint32_t mode, const float* const* in, float* out);
// One fused launch for an unchained all-mode sweep (when every mode shares the level-ordered
// kernel's specialisation); false if not applicable (nothing launched).
// Host-buffer pipeline of an unchained fused sweep (abi.cu mk_sweep_host): the modes run in
// `order`; slot m waits for the H2D flags of the factors it reads, and each finished mode
// raises its done flag for the D2H copy stream.
struct SweepIO {
  const uint32_t* fin;   // per factor: epoch of its last H2D copy
  uint32_t* fdone;       // per mode: epoch of its last completed output
  uint32_t epoch;
  uint32_t order[kMaxModes];
};
bool launch_sweep2(Context& c, const float* const* in, float* const* outs,
                   const SweepIO* io = nullptr);
// rank_of_row[row_seq[k]] = k for the copy's non-empty rows
void rank_of_row_build(Context& c, uint32_t mode, DevBuf<uint32_t>& rank);
void check_nonfinite(Context& c);  // synchronises; throws MK_ENONFINITE
// fp64 path (mttkrp64.cu)
void ensure_val64(Context& c, uint32_t mode);
void launch_mttkrp64(Context& c, uint32_t mode, const double* const* in, double* out, int exec);

}  // namespace mkb
