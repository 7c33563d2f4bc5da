/*
 * lscat.h — C ABI of the B200-native LS-CAT hot path (arXiv 2103.14409).
 *
 * Citations: P:n = line n of the paper text (PAPER.md, final IEEE version P:46-324),
 * S:n = SPEC.md line n (interfaces/test ideas only), DESIGN.md §x = this repo's readings.
 *
 * The hot path is the paper's thread-block-size sweep and the analysis of
 * its runtime table:
 *   register suite (a1) -> plan/shard (a2) -> launch (a3) + time (a4) -> emit table (a5)
 *   -> per-group reduce (a6) -> global accumulate (a7) -> percentiles (a8)
 *   -> multi-GPU merge (a9) -> finalize stats (a10).
 *
 * Conventions for every function below
 *   - Returns lscat_status; LSCAT_OK == 0.  Never aborts the process, never prints.
 *   - On LSCAT_ERR_INVALID_ARG no output is written (arguments are checked first).
 *   - A sticky CUDA error (e.g. an illegal address) poisons the context: every later call
 *     on it returns LSCAT_ERR_CUDA.  lscat_last_error() gives the message.
 *   - `stream` is a cudaStream_t passed as an opaque pointer (NULL = legacy default stream).
 *   - Device pointers are plain CUDA device addresses (e.g. torch tensor data_ptr()).
 *     "CALLER-OWNED" buffers stay owned by the caller; the library never frees them.
 *   - With world > 1 (lscat_comm_init), lscat_reduce_table and lscat_stats are collective:
 *     every rank calls them in the same order with the same options.  lscat_sweep is not a
 *     collective; each rank sweeps the points lscat_plan assigns to it.
 *   - There is no CPU fallback: without a CUDA device every compute call returns
 *     LSCAT_ERR_CUDA.  Host-only helpers (plan, work model, status strings) need no GPU.
 */
#ifndef LSCAT_H
#define LSCAT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSCAT_ABI_VERSION 2

typedef enum {
  LSCAT_OK = 0,
  LSCAT_ERR_INVALID_ARG = 1, /* bad argument; nothing written (maps to SPEC exit 2) */
  LSCAT_ERR_CUDA = 2,        /* CUDA runtime/driver error, or ctx poisoned */
  LSCAT_ERR_OOM = 3,         /* device or pinned-host allocation failed */
  LSCAT_ERR_NCCL = 4,        /* NCCL error during a collective */
  LSCAT_ERR_STATE = 5,       /* call out of order (e.g. sweep before register_suite) */
  LSCAT_ERR_UNSUPPORTED = 6  /* feature not built in / not available on this device */
} lscat_status;

/* Row status of one sweep point (S:233 RunOutcome; NaN runtime iff status != OK). */
typedef enum {
  LSCAT_ROW_OK = 0,
  LSCAT_ROW_TIMEOUT = 1,        /* predicted or measured point time > timeout_s */
  LSCAT_ROW_LAUNCH_ERROR = 2,   /* cudaLaunch* returned an error for this configuration */
  LSCAT_ROW_INVALID_CONFIG = 3  /* the kernel has no implementation at this block size */
} lscat_row_status;

/* The self-written suite (the paper's scraped kernels are unavailable, its
   only named kernel is euclidean_kernel). */
typedef enum {
  LSCAT_K_EUCLID = 0,    /* d[i] = sqrt(sum_j (A[i][j]-q[j])^2)                       */
  LSCAT_K_MATVEC = 1,    /* y[i] = sum_j A[i][j] x[j]                                 */
  LSCAT_K_GEMM_BF16 = 2, /* C = A Bt^T, bf16 in, fp32 accumulate (TMEM), bf16 out     */
  LSCAT_K_TRANSPOSE = 3, /* B[j][i] = A[i][j]                                         */
  LSCAT_K_AXPY = 4,      /* z = 0.5 x + y over N*N elements                           */
  LSCAT_K_ROWSUM = 5,    /* r[i] = sum_j A[i][j]                                      */
  LSCAT_K_COLSUM = 6,    /* c[j] = sum_i A[i][j]                                      */
  LSCAT_K_STENCIL5 = 7,  /* 5-point average, interior; border copied                  */
  LSCAT_K_COUNT = 8,
  LSCAT_K_SPIN = 100     /* TEST ONLY: spins `spin_ns` ns per launch (timeout tests)  */
} lscat_kernel;

/* Suite buffer slots. in0 = A (or x for axpy), in1 = q / x / Bt / y, out = result. */
typedef enum { LSCAT_SLOT_IN0 = 0, LSCAT_SLOT_IN1 = 1, LSCAT_SLOT_OUT = 2 } lscat_slot;

typedef enum { LSCAT_MEM_DEVICE = 0, LSCAT_MEM_HOST = 1 } lscat_mem;
/* How a bracket's R launches are issued (the paper's generated main loops on the host):
   GRAPH      pre-instantiated CUDA graphs of <= 128 launches (no host launch overhead);
   STREAM     one launch call per launch (the paper's host loop);
   GRAPH_PDL  graphs whose consecutive launches carry programmatic-dependent-launch edges:
              launch i+1 is scheduled and reads its (read-only) inputs while launch i drains,
              and waits for launch i to complete before its first global store.  Results are
              identical; the bracket time excludes the launch gap (R-3). */
typedef enum { LSCAT_LAUNCH_GRAPH = 0, LSCAT_LAUNCH_STREAM = 1, LSCAT_LAUNCH_GRAPH_PDL = 2 } lscat_launch_mode;
typedef enum { LSCAT_SHARD_POINT_LPT = 0, LSCAT_SHARD_GROUP = 1 } lscat_shard;
/* Bracket clock (P:201-205 times a loop of 1000 launches):
   EVENT        a CUDA event pair around the bracket on `stream`;
   GLOBALTIMER  two one-thread stamp kernels reading %globaltimer (ns) around the bracket,
                copied back asynchronously.  Events are recorded in both modes (the timeout
                budget uses them), so the two clocks can be compared on the same brackets. */
typedef enum { LSCAT_TIMER_EVENT = 0, LSCAT_TIMER_GLOBALTIMER = 1 } lscat_timer;
/* L2 state of the timed launches:
   WARM    the paper's loop: every launch of a point reuses the same buffers, so what one launch
           leaves in the 126 MB L2 serves the next (the suite kernels keep re-read inputs with
           L2 cache policies).  This is the runtime-table definition (R-3).
   ROTATE  cold-HBM measurement: c = clamp(ceil(2 x L2 / footprint), 2, 128) copies of the
           point's buffers (inputs copied from the registered suite before the warm-up, not
           timed) are cycled launch by launch, and no L2 keep policies are used; a launch's
           inputs were last touched >= 2 x L2 bytes of traffic earlier (for footprints of at
           least 2 x L2 / 128, i.e. N >= 512 for the 4N^2-byte kernels). */
typedef enum { LSCAT_L2_WARM = 0, LSCAT_L2_ROTATE = 1 } lscat_l2_mode;
typedef enum { LSCAT_SKIPNA = 0, LSCAT_COMPLETE_ONLY = 1 } lscat_nan_policy;

typedef struct lscat_ctx lscat_ctx; /* one per process/rank and device; opaque */

/* ---------------------------------------------------------------- context ---------- */
int lscat_abi_version(void);
const char* lscat_status_string(lscat_status s);

/* Create a context on CUDA device `device`.  `seed` seeds the on-device input generator
   (DESIGN.md §6).  *out receives the context (CALLEE-OWNED; free with lscat_ctx_destroy). */
lscat_status lscat_ctx_create(int device, uint64_t seed, lscat_ctx** out);
void lscat_ctx_destroy(lscat_ctx* ctx);
/* Message of the last failing call on ctx ("" if none).  Valid until the next call on ctx. */
const char* lscat_last_error(const lscat_ctx* ctx);
/* Number of device kernels the library has launched on ctx so far (graph-launched kernels
   counted one by one).  Used by bench.py for its gpu_launches claim. */
lscat_status lscat_launch_count(const lscat_ctx* ctx, uint64_t* out);

/* Multi-GPU (a9).  lscat_comm_unique_id writes a 128-byte ncclUniqueId into `out` (rank 0
   calls it and broadcasts the bytes, e.g. with torch.distributed).  lscat_comm_init creates
   the NCCL communicator of `world` ranks; world == 1 is valid and makes collectives no-ops. */
lscat_status lscat_comm_unique_id(void* out /* 128 bytes */);
lscat_status lscat_comm_init(lscat_ctx* ctx, const void* unique_id, int rank, int world);
/* TEST TRANSPORT: the `world` ranks are threads of this process (usually sharing one device)
   that each own a ctx and call this with the same `name`.  The merge collectives of
   lscat_reduce_table / lscat_stats then exchange buffers through host memory with a barrier
   instead of NCCL; the merge code path is otherwise identical, so multi-rank merges can be
   checked on a single GPU.  Not for production use. */
lscat_status lscat_comm_init_local(lscat_ctx* ctx, const char* name, int rank, int world);

/* ------------------------------------------------------------- a1: suite ------------ */
/* Materialise the inputs of every (kernel, N) pair: N x N row-major matrices (fp32, bf16 for
   the GEMM) filled on the device with a counter-based generator, uniform in [-1, 1)
   (reading R-15).  Outputs are allocated too.  The library owns these buffers until
   lscat_ctx_destroy.  Re-registering replaces the previous suite.  Sizes: 1 <= N <= 16384.
   (the generated main "initialize[s] all the needed variables".) */
lscat_status lscat_register_suite(lscat_ctx* ctx, const uint32_t* kernels, uint32_t n_kernels,
                                  const uint32_t* matrix_sizes, uint32_t n_sizes, void* stream);

/* Device address and byte size of a registered suite buffer (for verification).  Returns
   LSCAT_ERR_INVALID_ARG if the kernel/N/slot is not registered or the slot is unused. */
lscat_status lscat_suite_buffer(lscat_ctx* ctx, uint32_t kernel, uint32_t n, uint32_t slot,
                                void** dev_ptr, uint64_t* bytes);

/* Overwrite a registered input slot from `src` (host or device per `src_mem`), `bytes` must
   equal the slot size.  Host sources should be pinned for asynchronous copies. */
lscat_status lscat_suite_upload(lscat_ctx* ctx, uint32_t kernel, uint32_t n, uint32_t slot,
                                const void* src, uint64_t bytes, uint32_t src_mem, void* stream);

/* ------------------------------------------------------------- a3: launch ----------- */
/* One launch of suite kernel `kernel` over N at `block_threads` threads per block
   (32..1024, multiple of 32: P:98).  Asynchronous.  Returns LSCAT_ERR_INVALID_ARG for
   an illegal block and LSCAT_ERR_UNSUPPORTED when the kernel has no implementation at that
   block size (the GEMM needs >= 128 threads; the sweep records such points as
   LSCAT_ROW_INVALID_CONFIG). */
lscat_status lscat_launch(lscat_ctx* ctx, uint32_t kernel, uint32_t n, uint32_t block_threads,
                          void* stream);

/* Algorithmic work of one launch: bytes that must cross HBM and FLOPs.
   Host-only; needs no GPU. */
lscat_status lscat_kernel_work(uint32_t kernel, uint32_t n, uint64_t* bytes, uint64_t* flops);

/* ------------------------------------------------------------- a2: plan ------------- */
typedef struct {
  const uint32_t* kernels;  uint32_t n_kernels;   /* in sweep order                       */
  const uint32_t* sizes;    uint32_t n_sizes;     /* ascending N                          */
  const uint16_t* blocks;   uint32_t n_blocks;    /* threads; unique, ascending, %32 == 0, */
                                                  /* 32..1024    */
  uint32_t warmup, brackets, launches_per_bracket;/* paper: 1, 10, 1000    */
  uint32_t shard;                                 /* lscat_shard                          */
  double launch_overhead_s;                       /* cost model t_launch (0 -> 2e-6)      */
  double hbm_bytes_per_s, tensor_flops_per_s;     /* cost model peaks (0 -> defaults)     */
} lscat_plan_opts;

/* Points are numbered p = (kernel_index * n_sizes + size_index) * n_blocks + block_index
   (kernel-major canonical order); group g = p / n_blocks.  Writes the ids of the points owned
   by `rank` of `world`, ascending, into out_points[cap]; *n_out = their count.  Sharding is
   LPT on the cost model (W + K*R) * max(bytes/BW, flops/TC, t_launch), ties broken by point
   id then rank for LSCAT_SHARD_POINT_LPT, or LPT over whole groups for
   LSCAT_SHARD_GROUP.  Deterministic; host-only; needs no GPU.  ("By using
   cudaSetDevice, the additional GPUs could run the script in parallel".) */
lscat_status lscat_plan(const lscat_plan_opts* opts, int rank, int world, uint32_t* out_points,
                        uint64_t cap, uint64_t* n_out);

/* ------------------------------------------------------------- a4/a5: sweep --------- */
typedef struct {
  const uint16_t* blocks;   uint32_t n_blocks;    /* as lscat_plan_opts                   */
  uint32_t warmup;                                /* preheat launches (1)          */
  uint32_t brackets;                              /* K timed brackets (median: 10) */
  uint32_t launches_per_bracket;                  /* R launches per bracket (1000) */
  double timeout_s;                               /* per point (30; 2 on GTX 980)  */
  uint32_t launch_mode;                           /* lscat_launch_mode                    */
  uint32_t shard;                                 /* lscat_shard (world > 1)              */
  double launch_overhead_s;                       /* cost model, as lscat_plan_opts       */
  uint64_t spin_ns;                               /* LSCAT_K_SPIN only                    */
  float* bracket_ms_host;                         /* optional [cap_rows * brackets] host:  */
                                                  /* per-launch ms of every bracket by     */
                                                  /* `timer` (NaN = bracket not run)       */
  uint32_t timer;                                 /* lscat_timer (default EVENT)          */
  uint32_t l2_mode;                               /* lscat_l2_mode (default WARM)         */
  float* bracket_ms_event_host;                   /* optional [cap_rows * brackets] host:  */
                                                  /* the CUDA-event clock of the same     */
                                                  /* brackets (timer agreement check)     */
  uint32_t verify;                                /* 1: copy every point's output buffer  */
                                                  /* (the last timed launch's) to host    */
  void* verify_host;                              /* [verify_cap_bytes] host (pinned for  */
  uint64_t verify_cap_bytes;                      /* asynchronous copies)                 */
  uint64_t* verify_offsets;                       /* [cap_rows + 1] host: row i's bytes   */
                                                  /* at [off[i], off[i+1]) (empty if NaN) */
} lscat_sweep_opts;

/* Runtime table, structure of arrays (a5; the paper's dataframe rows).
   Group g owns rows [group_offset[g], group_offset[g+1]), or rows [g*rows_per_group, ...)
   when rows_per_group != 0 (then group_offset may be NULL).  Rows of a group need not be
   sorted; (group, block_id) pairs must be unique.  Buffers are CALLER-OWNED and live in
   device memory (mem == LSCAT_MEM_DEVICE) or host memory (LSCAT_MEM_HOST; the library
   stages them through device scratch, copies counted in the e2e measurement). */
typedef struct {
  float* runtime_ms;        /* [cap_rows] per-launch milliseconds; NaN = no result        */
  uint16_t* block_id;       /* [cap_rows] index into the block list (ascending threads)   */
  uint8_t* status;          /* [cap_rows] lscat_row_status (written by sweep/gen; may be  */
                            /*            NULL for reduce, which never reads it)          */
  int64_t* group_offset;    /* [cap_groups + 1]                                           */
  uint32_t* group_kernel;   /* [cap_groups] kernel id (may be NULL for reduce)           */
  uint32_t* group_matrix;   /* [cap_groups] matrix-size index; NULL -> (first_group+g) %  */
                            /*              n_matrices                                    */
  uint64_t cap_rows, cap_groups;
  uint64_t n_rows, n_groups;/* out of sweep/gen, in to reduce                             */
  uint32_t rows_per_group;  /* != 0 -> uniform groups                                     */
  uint32_t mem;             /* lscat_mem                                                  */
  uint64_t first_group;     /* global index of this table's group 0 (group-aligned shards)*/
} lscat_table;

/* Run this rank's points: per point `warmup` launches, then `brackets` brackets of
   `launches_per_bracket` launches each timed by `timer` on `stream`; runtime = median over
   brackets of (bracket ms / R) (even count -> midpoint).  Timeout
   budget (R-18): a point whose warm-up predicts more than timeout_s gets
   NaN + TIMEOUT without running its brackets; a point without a warm-up prediction (warmup
   == 0) or predicted above half the budget runs its brackets one at a time (one queued ahead)
   and stops as soon as the elapsed time, or the first bracket x K, exceeds timeout_s ("skip
   the rest" -> NaN + TIMEOUT); any point whose measured total exceeds it is NaN + TIMEOUT.
   verify requires verify_host / verify_offsets and enough capacity (ERR_INVALID_ARG).  Writes ALL groups of the plan (n_groups = n_kernels * n_sizes, canonical order,
   groups without local rows are empty) and this rank's rows, grouped, ascending block id.
   Synchronous with respect to the host.  Requires lscat_register_suite for every kernel/N. */
lscat_status lscat_sweep(lscat_ctx* ctx, const uint32_t* kernels, uint32_t n_kernels,
                         const uint32_t* sizes, uint32_t n_sizes, const lscat_sweep_opts* opts,
                         lscat_table* out, void* stream);

/* ------------------------------------------------------------- a6-a9: reduce -------- */
typedef struct {
  uint32_t n_blocks;          /* |L|                                                        */
  uint32_t largest_block_id;  /* l = id of the 1024-thread block             */
  uint32_t n_matrices;        /* rows of best_block_hist                                    */
  uint32_t nan_policy;        /* lscat_nan_policy; SKIPNA = pandas semantics        */
  uint32_t bins_per_unit;     /* 100 -> 1 % bins                                            */
  uint32_t gain_cap;          /* 10 -> gain bins [0, 10) + one overflow bin                 */
  uint32_t gain_gt_num, gain_gt_den;   /* 1/5: "more than 20 %", strict             */
  uint32_t perf_lt_num, perf_lt_den;   /* 17/20: "less than 85 %", strict           */
  uint32_t band_lo_num, band_lo_den;   /* 2/5: "from 40 to 85 %", [2/5, 17/20)      */
  uint32_t point_sharded;     /* 1 -> groups are split across ranks: per-group merge first  */
  uint32_t keep_values;       /* 1 -> keep per-group perf/gain (caller arrays or ctx        */
                              /*      scratch) for the percentiles of lscat_stats           */
  uint32_t block_profile;     /* 1 -> also accumulate the block profile of Figs. 2/4        */
                              /*      (P:240-247): per (matrix, block) the sum   */
                              /*      of floor(RN(best / r_b) * 2^31) over the ok rows of   */
                              /*      defined groups, and their count (R-22); one */
                              /*      extra read of the table                               */
  uint32_t kernel_rollup;     /* 1 -> also the per-kernel roll-up of P:258 ("83 % of the    */
                              /*      kernels", "1 % of the kernels ... from 40 to 85 %",  */
                              /*      DESIGN.md R-26): per kernel id (group_kernel, or      */
                              /*      (first_group + g) / n_matrices when NULL) over its    */
                              /*      ratio-defined groups: some best block != l, and the  */
                              /*      exact kernel-mean perf S_k / (c_k 2^52) against the  */
                              /*      thresholds and in 1 % bins.  Precondition: a kernel's */
                              /*      groups are contiguous in table order (sweep, generator */
                              /*      and ingest tables are); 8 extra bytes per group       */
  uint32_t n_percentiles;     /* > 0 (<= 64): lscat_reduce_table also enqueues the a8       */
                              /*      selection of these percentiles on its stream, right   */
                              /*      behind the reduction (one rank, not point-sharded,    */
                              /*      per-group values kept; R-27), and           */
                              /*      lscat_stats called with the same list only collects   */
                              /*      the result (a later selection of another list         */
                              /*      replaces it).  Otherwise lscat_stats selects as       */
                              /*      usual.  0: off                                        */
  uint32_t pad0;
  const double* percentiles;  /* HOST [n_percentiles] in [0, 1], read during the call      */
} lscat_reduce_opts;

/* Fills `opts` with the defaults above for a block list of n_blocks with largest id l. */
void lscat_reduce_opts_default(lscat_reduce_opts* opts, uint32_t n_blocks, uint32_t n_matrices);

/* Per-group outputs, device, CALLER-OWNED, each [n_groups] and each may be NULL. */
typedef struct {
  uint16_t* best_block_id;  /* argmin block id; 0xFFFF if the group is not defined        */
  float* best_runtime;      /* min runtime; NaN if not defined                             */
  double* perf;             /* RN(best / r_l); NaN unless ratio_defined           */
  double* gain;             /* RN(RN(r_l / best) - 1); NaN unless ratio_defined    */
  uint32_t* flags;          /* LSCAT_GF_* bits                                             */
  uint64_t* partials;       /* [lscat_partials_len] merged packed partials, or NULL        */
                            /* (the library keeps its own copy for lscat_stats either way) */
} lscat_reduce_out;

/* Layout of the packed partial vector (uint64 words), LSCAT_P_* counter slots first, then
   perf_hist [bins_per_unit+1], gain_hist [gain_cap*bins_per_unit+1], best_block_hist
   [n_matrices*n_blocks], and with block_profile: profile_sum [n_matrices*n_blocks],
   profile_count [n_matrices*n_blocks], and with kernel_rollup: 8 words (n_kernels,
   n_kernels_largest_not_best, n_kernels_perf_lt, n_kernels_perf_band, kernel_mean_fx_hi,
   kernel_mean_fx_lo, 0, 0) and kernel_perf_hist [bins_per_unit+1]. */
enum {
  LSCAT_P_ROWS = 0, LSCAT_P_OK, LSCAT_P_NAN, LSCAT_P_INVALID,
  LSCAT_P_GROUPS, LSCAT_P_DEFINED, LSCAT_P_ALL_NAN, LSCAT_P_COMPLETE, LSCAT_P_INCOMPLETE,
  LSCAT_P_LARGEST_MISSING, LSCAT_P_RATIO_DEFINED,
  LSCAT_P_LARGEST_IS_BEST, LSCAT_P_LARGEST_SLOWER, LSCAT_P_GAIN_GT, LSCAT_P_PERF_LT,
  LSCAT_P_PERF_BAND, LSCAT_P_PERF_FX_HI, LSCAT_P_PERF_FX_LO, LSCAT_P_GAIN_FX_HI,
  LSCAT_P_GAIN_FX_LO,
  LSCAT_P_BAD_IDS,   /* defined groups whose best row has block_id >= n_blocks or whose
                        matrix index >= n_matrices (a table violating the id ranges; such
                        groups are left out of the best-block histogram and lscat_stats
                        returns LSCAT_ERR_INVALID_ARG) */
  LSCAT_P_NCOUNTERS = 24 /* padded */
};

#define LSCAT_GF_DEFINED 0x001u
#define LSCAT_GF_COMPLETE 0x002u
#define LSCAT_GF_ALL_NAN 0x004u
#define LSCAT_GF_RATIO_DEFINED 0x008u
#define LSCAT_GF_LARGEST_IS_BEST 0x010u
#define LSCAT_GF_LARGEST_SLOWER 0x020u
#define LSCAT_GF_GAIN_GT 0x040u
#define LSCAT_GF_PERF_LT 0x080u
#define LSCAT_GF_PERF_BAND 0x100u
#define LSCAT_GF_LARGEST_MISSING 0x200u

/* Number of uint64 words of the packed partial vector (the NCCL payload of a9). */
size_t lscat_partials_len(const lscat_reduce_opts* opts);

/* Reduce a runtime table to per-group results and packed integer partials (DESIGN.md §4,
   steps O3.1-O3.9).  Integer outputs are exact and independent of row order, block order
   within a group and shard count.  With world > 1 the partials are summed over ranks (and,
   if point_sharded, per-group minima/maxima/counts are merged first) with NCCL.  The result
   stays in the context for lscat_stats.  Asynchronous unless table->mem == HOST. */
lscat_status lscat_reduce_table(lscat_ctx* ctx, const lscat_table* table,
                                const lscat_reduce_opts* opts, lscat_reduce_out* out,
                                void* stream);

/* ------------------------------------------------------------- a8/a10: stats -------- */
typedef struct {
  /* exact counters */
  uint64_t n_rows, n_ok, n_nan, n_invalid;
  uint64_t n_groups, n_defined, n_all_nan, n_complete, n_incomplete;
  uint64_t n_largest_missing, n_ratio_defined;
  uint64_t n_largest_is_best, n_largest_strictly_slower;
  uint64_t n_gain_gt, n_perf_lt, n_perf_band;
  /* fixed-point sums: sum floor(perf*2^52) and sum floor(min(gain,2^20)*2^32), each as
     hi = sum(fx >> 21), lo = sum(fx & (2^21-1)) */
  uint64_t perf_fx_hi, perf_fx_lo, gain_fx_hi, gain_fx_lo;
  /* derived on the host */
  double frac_nonnan;           /* n_ok / n_rows ("97% non NaN")                     */
  double frac_largest_not_best; /* (ratio_defined - largest_is_best) / ratio_defined */
  double frac_gain_gt;          /* n_gain_gt / n_ratio_defined ("10 %")             */
  double frac_perf_lt;          /* n_perf_lt / n_ratio_defined ("12 %")             */
  double frac_perf_band;        /* n_perf_band / n_ratio_defined ("1 %")            */
  double mean_perf;             /* P:258 "98.7 %", "86 %"                           */
  double mean_gain;             /* P:307 "6 %"                                            */
  /* optional caller-owned HOST arrays (NULL to skip) */
  uint64_t* perf_hist;          /* [bins_per_unit + 1]; bin k: k*t <= nb*b < (k+1)*t      */
  uint64_t* gain_hist;          /* [gain_cap*bins_per_unit + 1]; last = overflow          */
  uint64_t* best_block_hist;    /* [n_matrices * n_blocks]                                 */
  const double* percentiles;    /* [n_percentiles] in [0, 1]; nearest rank                 */
  uint32_t n_percentiles;       /* <= 64                                                   */
  double* pct_perf;             /* [n_percentiles] out; NaN if no ratio-defined group     */
  double* pct_gain;             /* [n_percentiles] out                                     */
  /* with opts->block_profile (else untouched): [n_matrices * n_blocks], row-major by matrix */
  double* profile_mean;         /* mean of best / r_b ((double)sum * 2^-31 / count); NaN  */
                                /* where count == 0                                        */
  uint64_t* profile_count;      /* number of rows averaged                                 */
  /* with opts->kernel_rollup (else untouched): the per-kernel roll-up (R-26) */
  uint64_t n_kernels;                    /* kernels with >= 1 ratio-defined group        */
  uint64_t n_kernels_largest_not_best;   /* ... some such group's best block != l        */
  uint64_t n_kernels_perf_lt;            /* ... kernel-mean perf < perf_lt               */
  uint64_t n_kernels_perf_band;          /* ... kernel-mean perf in [band_lo, perf_lt)   */
  uint64_t kernel_mean_fx_hi, kernel_mean_fx_lo;  /* sum_k floor(S_k / c_k), 21-bit limbs */
  double frac_kernels_largest_not_best;  /* P:258 "83 % of the kernels"                   */
  double frac_kernels_perf_lt;
  double frac_kernels_perf_band;         /* P:258 "around 1 % of the kernels"             */
  double mean_kernel_perf;               /* mean over kernels of the kernel-mean perf      */
  uint64_t* kernel_perf_hist;            /* optional HOST [bins_per_unit + 1]             */
} lscat_stats_out;

/* Finalize the statistics of the last lscat_reduce_table on ctx (a10) and, when
   out->n_percentiles > 0, select the exact nearest-rank percentiles of perf and gain over
   ratio-defined groups (a8).  Synchronizes `stream`; collective when world > 1. */
lscat_status lscat_stats(lscat_ctx* ctx, const lscat_reduce_opts* opts, lscat_stats_out* out,
                         void* stream);

/* ------------------------------------------------- table ingest (8f #3) ------------ */
/* Group an unordered runtime dataframe (the paper's Pandas rows) into a table: DEVICE
   inputs [n] kernel id, matrix index, block id, runtime (status may be NULL); `out` (device,
   CALLER-OWNED, cap_rows >= n, cap_groups >= number of distinct (kernel, matrix)) receives
   groups in ascending (kernel, matrix) order, rows ascending by block id (a stable radix sort,
   so equal keys keep their input order), group_offset / group_kernel / group_matrix (the
   latter two may be NULL).  n < 2^32.  Duplicated (kernel, matrix, block) rows violate the
   table precondition: the table is still written, *n_duplicates (may be NULL) counts them,
   and LSCAT_ERR_INVALID_ARG is returned.  Synchronous. */
lscat_status lscat_ingest(lscat_ctx* ctx, const uint32_t* kernel, const uint32_t* matrix,
                          const uint16_t* block_id, const float* runtime, const uint8_t* status,
                          uint64_t n, lscat_table* out, uint64_t* n_duplicates, void* stream);

/* ------------------------------------------------- side analyses (8f #4) ----------- */
/* The block the CUDA occupancy calculator picks for `kernel` ("The
   cudaOccupancyMaxPotentialBlockSize is Nvidias own solution to find the optimal thread block
   size for a kernel"; "insensitive to matrix sizes").  The suite is templated on the block
   size, so every candidate B has its own compiled function f_B.  For each candidate the
   library calls cudaOccupancyMaxPotentialBlockSizeVariableSMem(f_B, its dynamic smem, limit B)
   (info.api_block / api_min_grid) and cudaOccupancyMaxActiveBlocksPerMultiprocessor(f_B, B)
   (info.blocks_per_sm); the choice is the API's rule applied across the family: the candidate
   with the most resident threads (warps) per SM, ties -> the larger block (R-24).
   Independent of N by construction.  *out_block_id = its index in `blocks`; info (HOST
   [n_blocks], may be NULL) receives every candidate's attributes.  Evaluate the choice with
   lscat_reduce_table by setting largest_block_id to it. */
typedef struct {
  uint32_t threads;           /* candidate block size B                                     */
  int32_t regs_per_thread;    /* cudaFuncAttributes.numRegs of f_B                          */
  int32_t static_smem;        /* cudaFuncAttributes.sharedSizeBytes                         */
  int32_t dynamic_smem;       /* dynamic shared memory of the default launch at B           */
  int32_t max_threads_per_block; /* cudaFuncAttributes.maxThreadsPerBlock (launch bounds)   */
  int32_t blocks_per_sm;      /* cudaOccupancyMaxActiveBlocksPerMultiprocessor(f_B, B, dyn) */
  int32_t warps_per_sm;       /* blocks_per_sm * B / 32                                     */
  int32_t api_block;          /* cudaOccupancyMaxPotentialBlockSizeVariableSMem, limit B    */
  int32_t api_min_grid;       /* its minGridSize (= blocks per SM at api_block x SMs)       */
} lscat_occupancy_info;
lscat_status lscat_occupancy_block(lscat_ctx* ctx, uint32_t kernel, const uint16_t* blocks,
                                   uint32_t n_blocks, uint32_t* out_block_id,
                                   lscat_occupancy_info* info);

/* Timeout economics ("for two seconds of timeout around one third of the kernels had
   enough time to execute"): counts[i] (HOST) = number of rows of the (device) table that have
   a result and whose point time (warmup + brackets * launches_per_bracket) x runtime_ms x 1e-3
   (computed in double, rounded per operation) is <= taus[i] seconds (HOST, <= 64 values). */
lscat_status lscat_timeout_curve(lscat_ctx* ctx, const lscat_table* table, uint32_t warmup,
                                 uint32_t brackets, uint32_t launches_per_bracket,
                                 const double* taus, uint32_t n_taus, uint64_t* counts,
                                 void* stream);

/* ------------------------------------------------- aggregation experiment (8f #2) --- */
/* The paper's choice of the median: from a pool of runtimes (device, n_pool fp32)
   draw `reps` samples of k values without replacement (Floyd's algorithm on a counter-based
   generator seeded by `seed`), aggregate each with the five methods {mean, median, min, max,
   20 % trimmed mean} and report per method the variation = population standard deviation of
   its reps aggregates divided by their mean (R-23).  spread[5] and
   mean_of_aggregates[5] (may be NULL) are HOST arrays; aggregates (may be NULL) is a DEVICE
   array [5 * reps], method-major.  1 <= k <= 64 <= ... k <= n_pool.  Synchronizes `stream`. */
lscat_status lscat_aggregation_experiment(lscat_ctx* ctx, const float* pool, uint64_t n_pool,
                                          uint32_t k, uint32_t reps, uint64_t seed,
                                          double* spread, double* mean_of_aggregates,
                                          double* aggregates, void* stream);

/* ------------------------------------------------- synthetic tables (test/bench) ---- */
typedef enum { LSCAT_PRESET_T4 = 0, LSCAT_PRESET_GTX980 = 1 } lscat_preset;

typedef struct {
  uint64_t n_rows_global;   /* total rows of the global table (layout rule) */
  uint32_t n_kernels;       /* kernel ids K                                                */
  uint32_t n_blocks;        /* |L| (block ids 0..|L|-1, threads 32*(id+1))                 */
  uint32_t largest_block_id;
  uint32_t n_matrices;      /* matrix index = position within the kernel's groups         */
  uint32_t preset;          /* lscat_preset                                                */
  double nan_rate;          /* iid per row (3 %)                                    */
  uint64_t seed;
  /* shard selection: rows of global groups [group_begin, group_end) ...                   */
  uint64_t group_begin, group_end;  /* group_end == 0 -> all groups                        */
  uint32_t block_mod, block_rem;    /* ... keeping only block ids with id % mod == rem     */
                                    /* (mod 0 or 1 -> all; point-sharded tables)           */
} lscat_gen_opts;

/* Write a synthetic runtime table shaped like the paper's dataset (planted-best runtime
   model) into `out` (device memory).  Bit-identical to synth/tables.py. */
lscat_status lscat_gen_table(lscat_ctx* ctx, const lscat_gen_opts* opts, lscat_table* out,
                             void* stream);
/* Sizes the buffers lscat_gen_table needs for `opts` (host-only). */
lscat_status lscat_gen_table_shape(const lscat_gen_opts* opts, uint64_t* n_rows,
                                   uint64_t* n_groups);

#ifdef __cplusplus
}
#endif
#endif /* LSCAT_H */
