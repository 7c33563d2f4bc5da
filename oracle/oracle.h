/* oracle.h — CPU oracle interface.  TEST INFRASTRUCTURE ONLY (see lscat_oracle.c).
   Independent of include/lscat.h: its own types, its own counter order. */
#ifndef LSCAT_ORACLE_H
#define LSCAT_ORACLE_H
#include <stddef.h>
#include <stdint.h>

enum { ORACLE_OK = 0, ORACLE_EINVAL = 1, ORACLE_EDUP = 2, ORACLE_ENOMEM = 3 };
enum { ORACLE_SKIPNA = 0, ORACLE_COMPLETE_ONLY = 1 };

/* counter slots of oracle_result.counters */
enum {
  OC_N_ROWS = 0, OC_N_OK, OC_N_NAN, OC_N_INVALID,
  OC_N_GROUPS, OC_N_DEFINED, OC_N_ALL_NAN, OC_N_COMPLETE, OC_N_INCOMPLETE,
  OC_N_LARGEST_MISSING, OC_N_RATIO_DEFINED,
  OC_N_LARGEST_IS_BEST, OC_N_LARGEST_SLOWER, OC_N_GAIN_GT, OC_N_PERF_LT, OC_N_PERF_BAND,
  OC_PERF_FX_HI, OC_PERF_FX_LO, OC_GAIN_FX_HI, OC_GAIN_FX_LO,
  ORACLE_NCOUNTERS
};

typedef struct {
  const float* runtime_ms;
  const uint16_t* block_id;
  uint64_t n_rows;
  const int64_t* group_offset; /* [n_groups+1], unused if rows_per_group != 0 */
  uint64_t n_groups;
  uint32_t rows_per_group;
  const uint32_t* group_matrix; /* may be NULL -> (first_group + g) % n_matrices */
  uint64_t first_group;
} oracle_table;

typedef struct {
  uint32_t n_blocks, largest_block_id, n_matrices, nan_policy;
  uint32_t bins_per_unit, gain_cap;
  uint32_t gain_gt_num, gain_gt_den, perf_lt_num, perf_lt_den, band_lo_num, band_lo_den;
} oracle_opts;

typedef struct {
  uint64_t counters[ORACLE_NCOUNTERS];
  uint64_t* perf_hist;       /* [bins+1]            caller-owned */
  uint64_t* gain_hist;       /* [cap*bins+1]        caller-owned */
  uint64_t* best_block_hist; /* [n_matrices*n_blocks] caller-owned */
  uint64_t* profile_sum;     /* [n_matrices*n_blocks] caller-owned, or NULL (no block profile) */
  uint64_t* profile_count;   /* [n_matrices*n_blocks] caller-owned, or NULL */
} oracle_result;

typedef struct {
  uint16_t* best_block; float* best_runtime; double* perf; double* gain; uint32_t* flags;
} oracle_group_out;

typedef struct {
  double frac_nonnan, frac_largest_not_best, frac_gain_gt, frac_perf_lt, frac_perf_band;
  double mean_perf, mean_gain;
} oracle_derived;

int oracle_reduce_table(const oracle_table* T, const oracle_opts* o, oracle_result* R,
                        oracle_group_out* G);

/* Per-kernel roll-up (P:258 counts *kernels*: "this was also true for 83% of the kernels",
   "in around 1% of the kernels this ranges from 40 to 85%"; R-26). */
enum {
  OK_N_KERNELS = 0,          /* kernels with >= 1 ratio-defined group                       */
  OK_N_NOT_BEST,             /* ... in which some ratio-defined group's best block != l     */
  OK_N_PERF_LT,              /* ... whose mean performance is < perf_lt (17/20)            */
  OK_N_PERF_BAND,            /* ... whose mean performance is in [band_lo, perf_lt)        */
  OK_MEAN_FX_HI, OK_MEAN_FX_LO,  /* sum over kernels of floor(S_k / c_k), two 21-bit limbs   */
  ORACLE_NKCOUNTERS
};
typedef struct {
  uint64_t counters[ORACLE_NKCOUNTERS];
  uint64_t* perf_hist;       /* [bins+1] caller-owned: bin j = largest j with j c 2^52 <= nb S */
} oracle_rollup;
/* group_kernel[g] (NULL -> (first_group + g) / n_matrices) names each group's kernel; G holds
   oracle_reduce_table's per-group outputs of the same table. */
int oracle_kernel_rollup(const oracle_table* T, const uint32_t* group_kernel, const oracle_opts* o,
                         const oracle_group_out* G, oracle_rollup* K);
void oracle_finalize(const oracle_result* R, oracle_derived* D);
double oracle_percentile(const double* values, uint64_t n, double p);
size_t oracle_partials_len(uint32_t bins_per_unit, uint32_t gain_cap, uint32_t n_matrices,
                           uint32_t n_blocks);
#endif
