/*
 * lscat_oracle_omp.c — the C oracle of lscat_oracle.c run on all host cores.
 *
 * TEST / BASELINE INFRASTRUCTURE ONLY (bench.py's cpu_baseline and its test): it adds no
 * arithmetic of the method.  The table is cut into group-aligned chunks; every chunk is
 * reduced by the unchanged single-threaded oracle_reduce_table (a sub-table of the same rows,
 * first_group shifted so the implicit matrix index is unchanged), and the integer partials
 * (counters, histograms) are summed.  Every partial is an integer sum over groups, so the
 * totals equal the whole-table oracle exactly for any chunking (the same shard
 * invariance the multi-GPU merge uses; pinned by tests/test_oracle_table.py).
 */
#include <omp.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

int oracle_reduce_table_omp(const oracle_table* T, const oracle_opts* o, oracle_result* R,
                            oracle_group_out* G, int nthreads) {
  const size_t nb = o->bins_per_unit, ng = (size_t)o->gain_cap * nb, nbb = (size_t)o->n_matrices * o->n_blocks;
  const uint64_t n_groups = T->n_groups;
  if (nthreads < 1) nthreads = omp_get_max_threads();
  uint64_t nch = (uint64_t)nthreads * 8;
  if (nch > n_groups) nch = n_groups ? n_groups : 1;
  memset(R->counters, 0, sizeof(R->counters));
  memset(R->perf_hist, 0, (nb + 1) * 8);
  memset(R->gain_hist, 0, (ng + 1) * 8);
  memset(R->best_block_hist, 0, nbb * 8);
  int err = ORACLE_OK;
#pragma omp parallel num_threads(nthreads)
  {
    uint64_t* ph = (uint64_t*)calloc(nb + 1, 8);
    uint64_t* gh = (uint64_t*)calloc(ng + 1, 8);
    uint64_t* bh = (uint64_t*)calloc(nbb ? nbb : 1, 8);
    uint64_t* acc = (uint64_t*)calloc(ORACLE_NCOUNTERS + nb + 1 + ng + 1 + nbb, 8);
    int lerr = (ph && gh && bh && acc) ? ORACLE_OK : ORACLE_ENOMEM;
#pragma omp for schedule(dynamic, 1)
    for (int64_t c = 0; c < (int64_t)nch; c++) {
      if (lerr) continue;
      const uint64_t g0 = n_groups * (uint64_t)c / nch, g1 = n_groups * (uint64_t)(c + 1) / nch;
      oracle_table S = *T;
      S.n_groups = g1 - g0;
      S.first_group = T->first_group + g0;
      if (T->group_matrix) S.group_matrix = T->group_matrix + g0;
      if (T->rows_per_group) {
        const uint64_t r0 = g0 * T->rows_per_group;
        uint64_t r1 = g1 * T->rows_per_group;
        if (r1 > T->n_rows) r1 = T->n_rows;
        S.runtime_ms = T->runtime_ms + r0;
        S.block_id = T->block_id + r0;
        S.n_rows = r1 - r0;
      } else {
        S.group_offset = T->group_offset + g0;  /* absolute row indices into the same arrays */
        S.n_rows = (uint64_t)(T->group_offset[g1] - T->group_offset[g0]);
      }
      oracle_result P;
      memset(&P, 0, sizeof P);
      P.perf_hist = ph;
      P.gain_hist = gh;
      P.best_block_hist = bh;
      oracle_group_out GS, *gp = NULL;
      if (G) {
        GS.best_block = G->best_block ? G->best_block + g0 : NULL;
        GS.best_runtime = G->best_runtime ? G->best_runtime + g0 : NULL;
        GS.perf = G->perf ? G->perf + g0 : NULL;
        GS.gain = G->gain ? G->gain + g0 : NULL;
        GS.flags = G->flags ? G->flags + g0 : NULL;
        gp = &GS;
      }
      lerr = oracle_reduce_table(&S, o, &P, gp);
      if (lerr) continue;
      for (int i = 0; i < ORACLE_NCOUNTERS; i++) acc[i] += P.counters[i];
      for (size_t i = 0; i <= nb; i++) acc[ORACLE_NCOUNTERS + i] += ph[i];
      for (size_t i = 0; i <= ng; i++) acc[ORACLE_NCOUNTERS + nb + 1 + i] += gh[i];
      for (size_t i = 0; i < nbb; i++) acc[ORACLE_NCOUNTERS + nb + 1 + ng + 1 + i] += bh[i];
    }
#pragma omp critical
    {
      if (lerr) err = lerr;
      if (acc) {
        for (int i = 0; i < ORACLE_NCOUNTERS; i++) R->counters[i] += acc[i];
        for (size_t i = 0; i <= nb; i++) R->perf_hist[i] += acc[ORACLE_NCOUNTERS + i];
        for (size_t i = 0; i <= ng; i++) R->gain_hist[i] += acc[ORACLE_NCOUNTERS + nb + 1 + i];
        for (size_t i = 0; i < nbb; i++) R->best_block_hist[i] += acc[ORACLE_NCOUNTERS + nb + 1 + ng + 1 + i];
      }
    }
    free(ph); free(gh); free(bh); free(acc);
  }
  return err;
}
