/*
 * lscat_oracle.c — CPU ORACLE for the LS-CAT runtime-table analysis.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * / --impl reference legs may load this library.  It shares no code, header, table or
 * constant generator with the CUDA path (paper_2103_14409_b200/csrc), and never reads any of
 * its outputs.  Plain, slow, single-threaded C: every step is written the way the paper (and
 * the readings listed in DESIGN.md §4) state it, in that order.
 *
 * Citations: P:n = PAPER.md line n.  R-n = DESIGN.md reading n.
 *
 * What it computes, per group g = one (kernel, matrix size) slice of the runtime table
 * (the paper's Figs. 3/5 unit):
 *   1. row validity: a row has a result iff its runtime is finite and > 0; NaN rows are the
 *      paper's failed / timed-out runs ("97% non NaN data").
 *   2. the best block = the block with the smallest runtime, ties -> smaller block id (R-8)
 *      ("the best performing thread block was not the largest one").
 *   3. the largest block l (1024 threads) and its runtime t; best runtime b.
 *   4. performance of the largest block = b / t ("performance of 98.7 % of the best block",
 *      P:258, R-5) and the gain of the optimal block = t / b - 1 ("6 % performance increase",
 *      P:307).
 *   5. thresholds: gain > 1/5 ("more than 20 %"), perf < 17/20 ("less than 85 %",
 *      P:282), 2/5 <= perf < 17/20 ("from 40 to 85 %"), all as exact rational
 *      comparisons of b and t (R-10).
 *   6. 1 % histograms of perf and gain (R-13) with the bin edges exact (largest k with
 *      k*t <= nb*b), a per-matrix histogram of best block ids (Figs. 2/4 data).
 *   7. fixed-point sums floor(perf*2^52), floor(min(gain,2^20)*2^32) for exact means (R-13).
 *   8. nearest-rank percentiles of perf and gain over ratio-defined groups (R-13).
 *   9. (optional) the block profile of Figs. 2/4: mean of best / r_b per (matrix, block) (R-22).
 *
 * Exactness argument used in steps 5-6: b and t are float32 values widened to double; every
 * product k*t with integer k < 2^29 has at most 24+29 = 53 significant bits, so it is exact
 * in double and the comparisons below are exact rational comparisons.
 *
 * Parity status: every function here is pinned by tests/test_oracle_table.py against
 * pandas groupby / fractions.Fraction brute force, SPEC examples (tests/golden/) and
 * invariants.  See DESIGN.md §8.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* ---- step 1: row validity ------------------------------------------------------------ */
static int row_ok(float r) { return isfinite(r) && r > 0.0f; }

/* ---- step 6: histogram bins, by the definition "largest integer k with k*t <= nb*b" ---- */
static uint32_t perf_bin(double b, double t, uint32_t nb) {
  /* perf = b/t in (0, 1]: the bin is the largest k in [0, nb] with k*t <= nb*b.  Scan down
     from nb; the first k that satisfies the inequality is the largest. */
  for (uint32_t k = nb;; k--) {
    if ((double)k * t <= (double)nb * b) return k;
    if (k == 0) return 0;
  }
}

static uint32_t gain_bin(double b, double t, uint32_t nb, uint32_t cap) {
  /* gain = t/b - 1 >= 0.  Overflow bin (index cap*nb) iff gain >= cap, i.e. t >= (cap+1)*b.
     Otherwise the bin is m - nb for the largest integer m with m*b <= nb*t; m >= nb since
     t >= b.  Scan up from nb. */
  if (t >= (double)(cap + 1) * b) return cap * nb;
  uint32_t m = nb;
  while ((double)(m + 1) * b <= (double)nb * t) m++;
  return m - nb;
}

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

double oracle_percentile(const double* values, uint64_t n, double p) {
  /* Nearest rank (R-13): the value at sorted position ceil(p*n) (1-based), clamped to
     [1, n].  Empty -> NaN. */
  if (n == 0) return NAN;
  double* s = (double*)malloc(n * sizeof(double));
  memcpy(s, values, n * sizeof(double));
  qsort(s, n, sizeof(double), cmp_double);
  double r = ceil(p * (double)n);
  uint64_t k = r < 1.0 ? 1 : (r > (double)n ? n : (uint64_t)r);
  double v = s[k - 1];
  free(s);
  return v;
}

size_t oracle_partials_len(uint32_t bins_per_unit, uint32_t gain_cap, uint32_t n_matrices,
                           uint32_t n_blocks) {
  return (size_t)ORACLE_NCOUNTERS + (bins_per_unit + 1) + ((size_t)gain_cap * bins_per_unit + 1) +
         (size_t)n_matrices * n_blocks;
}

int oracle_reduce_table(const oracle_table* T, const oracle_opts* o, oracle_result* R,
                        oracle_group_out* G) {
  const uint32_t nb = o->bins_per_unit;
  const uint32_t L = o->n_blocks;
  const uint32_t ell = o->largest_block_id;
  if (nb == 0 || L == 0 || ell >= L || o->gain_cap == 0) return ORACLE_EINVAL;
  memset(R->counters, 0, sizeof(R->counters));
  memset(R->perf_hist, 0, sizeof(uint64_t) * (nb + 1));
  memset(R->gain_hist, 0, sizeof(uint64_t) * ((size_t)o->gain_cap * nb + 1));
  memset(R->best_block_hist, 0, sizeof(uint64_t) * (size_t)o->n_matrices * L);
  if (R->profile_sum) memset(R->profile_sum, 0, sizeof(uint64_t) * (size_t)o->n_matrices * L);
  if (R->profile_count) memset(R->profile_count, 0, sizeof(uint64_t) * (size_t)o->n_matrices * L);
  uint64_t* C = R->counters;
  unsigned char* seen = (unsigned char*)malloc(L);
  if (!seen) return ORACLE_ENOMEM;

  C[OC_N_ROWS] = T->n_rows;
  C[OC_N_GROUPS] = T->n_groups;
  for (uint64_t g = 0; g < T->n_groups; g++) {
    uint64_t r0, r1;
    if (T->rows_per_group) {
      r0 = g * T->rows_per_group;
      r1 = r0 + T->rows_per_group;
      if (r1 > T->n_rows) r1 = T->n_rows;
    } else {
      r0 = (uint64_t)T->group_offset[g];
      r1 = (uint64_t)T->group_offset[g + 1];
    }
    /* step 1 + precondition: (group, block) unique */
    memset(seen, 0, L);
    uint64_t n_ok = 0, n_nan = 0, n_rows = r1 - r0;
    int have_best = 0;
    float best = 0.0f;
    uint32_t best_block = 0;
    int have_ell = 0, ell_ok = 0;
    float t_ell = 0.0f;
    for (uint64_t r = r0; r < r1; r++) {
      uint32_t bid = T->block_id[r];
      float rt = T->runtime_ms[r];
      if (bid >= L || seen[bid]) { free(seen); return ORACLE_EDUP; }
      seen[bid] = 1;
      if (isnan(rt)) n_nan++;
      else if (row_ok(rt)) n_ok++;
      if (bid == ell) { have_ell = 1; ell_ok = row_ok(rt); t_ell = rt; }
      /* step 2: smallest runtime; equal runtimes -> the smaller block id */
      if (row_ok(rt)) {
        if (!have_best || rt < best || (rt == best && bid < best_block)) {
          have_best = 1; best = rt; best_block = bid;
        }
      }
    }
    C[OC_N_OK] += n_ok;
    C[OC_N_NAN] += n_nan;
    C[OC_N_INVALID] += n_rows - n_ok - n_nan;

    /* step 3: completeness and definedness (R-4) */
    int complete = (n_rows == L) && (n_ok == n_rows);
    int defined = (o->nan_policy == ORACLE_COMPLETE_ONLY) ? complete : (n_ok >= 1);
    uint32_t flags = 0;
    if (n_ok == 0) { C[OC_N_ALL_NAN]++; flags |= 0x004u; }
    if (complete) { C[OC_N_COMPLETE]++; flags |= 0x002u; } else C[OC_N_INCOMPLETE]++;
    uint32_t matrix = T->group_matrix ? T->group_matrix[g]
                                      : (uint32_t)((T->first_group + g) % o->n_matrices);
    double perf = NAN, gain = NAN;
    if (defined) {
      flags |= 0x001u;
      C[OC_N_DEFINED]++;
      R->best_block_hist[(size_t)matrix * L + best_block]++;
      /* block profile (Figs. 2/4; reading R-22): performance best / r_b of every
         block that has a result, as floor(RN(best / r_b) * 2^31), per (matrix, block) */
      if (R->profile_sum && R->profile_count) {
        for (uint64_t r = r0; r < r1; r++) {
          if (!row_ok(T->runtime_ms[r])) continue;
          double pb = (double)best / (double)T->runtime_ms[r];
          size_t at = (size_t)matrix * L + T->block_id[r];
          R->profile_sum[at] += (uint64_t)floor(pb * 2147483648.0);
          R->profile_count[at] += 1;
        }
      }
      /* step 3: the largest block's row must exist and have a result */
      if (have_ell && ell_ok) {
        double b = (double)best, t = (double)t_ell;
        flags |= 0x008u;
        C[OC_N_RATIO_DEFINED]++;
        /* step 4 */
        perf = b / t;
        gain = t / b - 1.0;
        /* step 5 */
        if (best_block == ell) { C[OC_N_LARGEST_IS_BEST]++; flags |= 0x010u; }
        if (t > b) { C[OC_N_LARGEST_SLOWER]++; flags |= 0x020u; }
        /* gain > p/q  <=>  t/b > 1 + p/q  <=>  q*t > (q+p)*b */
        if ((double)o->gain_gt_den * t > (double)(o->gain_gt_den + o->gain_gt_num) * b) {
          C[OC_N_GAIN_GT]++; flags |= 0x040u;
        }
        /* perf < p/q  <=>  q*b < p*t */
        int perf_lt = (double)o->perf_lt_den * b < (double)o->perf_lt_num * t;
        if (perf_lt) { C[OC_N_PERF_LT]++; flags |= 0x080u; }
        /* p_lo <= perf  <=>  q_lo*b >= p_lo*t ; band = [lo, perf_lt) */
        if (perf_lt && (double)o->band_lo_den * b >= (double)o->band_lo_num * t) {
          C[OC_N_PERF_BAND]++; flags |= 0x100u;
        }
        /* step 6 */
        R->perf_hist[perf_bin(b, t, nb)]++;
        R->gain_hist[gain_bin(b, t, nb, o->gain_cap)]++;
        /* step 7: fixed point; perf*2^52 and gain*2^32 are exact scalings */
        uint64_t fxp = (uint64_t)floor(perf * 4503599627370496.0);
        double gc = gain < 1048576.0 ? gain : 1048576.0;
        uint64_t fxg = (uint64_t)floor(gc * 4294967296.0);
        C[OC_PERF_FX_HI] += fxp >> 21;
        C[OC_PERF_FX_LO] += fxp & ((1ull << 21) - 1);
        C[OC_GAIN_FX_HI] += fxg >> 21;
        C[OC_GAIN_FX_LO] += fxg & ((1ull << 21) - 1);
      } else {
        C[OC_N_LARGEST_MISSING]++;
        flags |= 0x200u;
      }
    }
    if (G) {
      if (G->best_block) G->best_block[g] = defined ? (uint16_t)best_block : 0xFFFFu;
      if (G->best_runtime) G->best_runtime[g] = defined ? best : NAN;
      if (G->perf) G->perf[g] = perf;
      if (G->gain) G->gain[g] = gain;
      if (G->flags) G->flags[g] = flags;
    }
  }
  free(seen);
  return ORACLE_OK;
}

void oracle_finalize(const oracle_result* R, oracle_derived* D) {
  /* step a10 (host): fractions over the ratio-defined groups (R-7, R-9), non-NaN share over
     all rows, exact fixed-point means rounded to double (R-13). */
  const uint64_t* C = R->counters;
  double nrd = (double)C[OC_N_RATIO_DEFINED];
  D->frac_nonnan = C[OC_N_ROWS] ? (double)C[OC_N_OK] / (double)C[OC_N_ROWS] : NAN;
  D->frac_largest_not_best =
      nrd > 0 ? (double)(C[OC_N_RATIO_DEFINED] - C[OC_N_LARGEST_IS_BEST]) / nrd : NAN;
  D->frac_gain_gt = nrd > 0 ? (double)C[OC_N_GAIN_GT] / nrd : NAN;
  D->frac_perf_lt = nrd > 0 ? (double)C[OC_N_PERF_LT] / nrd : NAN;
  D->frac_perf_band = nrd > 0 ? (double)C[OC_N_PERF_BAND] / nrd : NAN;
  unsigned __int128 tp = ((unsigned __int128)C[OC_PERF_FX_HI] << 21) + C[OC_PERF_FX_LO];
  unsigned __int128 tg = ((unsigned __int128)C[OC_GAIN_FX_HI] << 21) + C[OC_GAIN_FX_LO];
  D->mean_perf = nrd > 0 ? ((double)tp * 0x1p-52) / nrd : NAN;
  D->mean_gain = nrd > 0 ? ((double)tg * 0x1p-32) / nrd : NAN;
}

/* ---- per-kernel roll-up (R-26) ----------------------------------------- */
typedef struct { uint64_t kernel, group; } kg_pair;

static int cmp_kg(const void* a, const void* b) {
  const kg_pair *x = (const kg_pair*)a, *y = (const kg_pair*)b;
  if (x->kernel != y->kernel) return x->kernel < y->kernel ? -1 : 1;
  return (x->group > y->group) - (x->group < y->group);
}

int oracle_kernel_rollup(const oracle_table* T, const uint32_t* group_kernel, const oracle_opts* o,
                         const oracle_group_out* G, oracle_rollup* K) {
  /* The paper states two results over kernels: the share of kernels for which "the
     best performing thread block was not the largest one", and the share whose largest-block
     performance "ranges from 40 to 85%".  For each kernel k, over its ratio-defined groups
     (the matrix sizes where perf = best / t_l is defined, R-5/R-6):
       c_k     = their number (a kernel with c_k = 0 is not counted);
       S_k     = sum of floor(perf * 2^52) (the exact fixed-point values of O3 step 9);
       not_best(k)  <=> some such group's best block != l;
       mean perf    P_k = S_k / (c_k 2^52), compared exactly:
       perf_lt(k)   <=> P_k < perf_lt_num / perf_lt_den;
       band(k)      <=> band_lo <= P_k < perf_lt  (half-open, as R-10);
       histogram bin = the largest j in [0, nb] with j c_k 2^52 <= nb S_k;
       mean over kernels = sum_k floor(S_k / c_k) / (2^52 n_kernels), kept as two limbs.
     Groups are collected per kernel id by sorting (kernel, group) pairs, so the roll-up does
     not depend on the table's group order. */
  if (!G || !G->perf || !G->flags || !G->best_block || o->bins_per_unit == 0 || o->n_matrices == 0)
    return ORACLE_EINVAL;
  const uint32_t nb = o->bins_per_unit;
  memset(K->counters, 0, sizeof(K->counters));
  memset(K->perf_hist, 0, sizeof(uint64_t) * (nb + 1));
  uint64_t n = T->n_groups;
  kg_pair* pr = (kg_pair*)malloc((n ? n : 1) * sizeof(kg_pair));
  if (!pr) return ORACLE_ENOMEM;
  for (uint64_t g = 0; g < n; g++) {
    pr[g].kernel = group_kernel ? group_kernel[g] : (T->first_group + g) / o->n_matrices;
    pr[g].group = g;
  }
  qsort(pr, n, sizeof(kg_pair), cmp_kg);
  const unsigned __int128 one = (unsigned __int128)1 << 52;
  uint64_t i = 0;
  while (i < n) {
    uint64_t j = i, c = 0;
    unsigned __int128 S = 0;
    int not_best = 0;
    while (j < n && pr[j].kernel == pr[i].kernel) {
      uint64_t g = pr[j].group;
      if (G->flags[g] & 0x008u) {            /* ratio-defined */
        c++;
        S += (uint64_t)floor(G->perf[g] * 4503599627370496.0);
        if (G->best_block[g] != o->largest_block_id) not_best = 1;
      }
      j++;
    }
    if (c > 0) {
      uint64_t* C = K->counters;
      C[OK_N_KERNELS]++;
      if (not_best) C[OK_N_NOT_BEST]++;
      unsigned __int128 cd = (unsigned __int128)c * one;  /* P_k = S / cd */
      int lt = (unsigned __int128)o->perf_lt_den * S < (unsigned __int128)o->perf_lt_num * cd;
      if (lt) C[OK_N_PERF_LT]++;
      if (lt && (unsigned __int128)o->band_lo_den * S >= (unsigned __int128)o->band_lo_num * cd)
        C[OK_N_PERF_BAND]++;
      uint32_t bin = nb;
      while (bin > 0 && (unsigned __int128)bin * cd > (unsigned __int128)nb * S) bin--;
      K->perf_hist[bin]++;
      uint64_t kfx = (uint64_t)(S / c);
      C[OK_MEAN_FX_HI] += kfx >> 21;
      C[OK_MEAN_FX_LO] += kfx & ((1ull << 21) - 1);
    }
    i = j;
  }
  free(pr);
  return ORACLE_OK;
}
