// gen.cu — synthetic runtime tables (test/bench input; not on the timed path).
//
// Counter-based twin of synth/tables.py: the same splitmix64 streams and the
// same IEEE double operations in the same order, each written with an explicit _rn intrinsic
// so that no FMA contraction can change a rounding; the result is bit-identical to numpy.
// One warp per group; lane 0's draws are broadcast; lanes write the group's rows.
#include <cmath>

#include "common.h"

namespace lscat {
namespace {

__device__ __forceinline__ uint64_t smix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double unif(uint64_t s_stream, uint64_t idx) {
  return __dmul_rn(__ull2double_rn(smix(idx ^ s_stream) >> 11), 0x1p-53);
}

struct GP {
  uint64_t G, n_rows_global, gb, ge;
  uint32_t K, L, ell, M, mod, rem;
  uint32_t cnt_full, cnt_last;  // kept rows per full / last (global) group
  uint64_t q, r;                // kernel layout
  double nan_rate;
  double c0, c1, c2, lo1, hi1, lo2, hi2, lo3, hi3;
  uint64_t s[6];                // per-stream seeds
  float* rt; uint16_t* bid; uint8_t* st; int64_t* off; uint32_t* gk; uint32_t* gm;
};

__global__ void gen_kernel(GP p) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const uint64_t nG = p.ge - p.gb;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t j = warp; j < nG; j += nw) {
    const uint64_t g = p.gb + j;
    // kernel / matrix position of g (layout rule)
    const uint64_t big = p.r * (p.q + 1);
    uint64_t kern, pos;
    if (g < big) { kern = g / (p.q + 1); pos = g % (p.q + 1); }
    else { const uint64_t q = p.q ? p.q : 1; kern = p.r + (g - big) / q; pos = (g - big) % q; }
    const uint32_t mat = (uint32_t)(pos % p.M);
    const double u0 = unif(p.s[0], g), u1 = unif(p.s[1], g), u2 = unif(p.s[2], g), u3 = unif(p.s[3], g);
    const double scale = (double)(1ull << (2 * mat));
    const double T0 = __dmul_rn(__dmul_rn(1e-3, scale), __dadd_rn(0.5, u0));
    const bool best_is_l = u1 < p.c0;
    int64_t bstar = (int64_t)floor(__dmul_rn(u2, (double)(p.L - 1)));
    if (bstar >= (int64_t)p.ell) bstar += 1;
    if (best_is_l) bstar = p.ell;
    const double lo = u1 < p.c1 ? p.lo1 : (u1 < p.c2 ? p.lo2 : p.lo3);
    const double hi = u1 < p.c1 ? p.hi1 : (u1 < p.c2 ? p.hi2 : p.hi3);
    const double glarge = __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u3));
    const double thr_b = __dmul_rn(32.0, __dadd_rn((double)bstar, 1.0));
    const double thr_l = __dmul_rn(32.0, __dadd_rn((double)p.ell, 1.0));
    const double dl = __ddiv_rn(__dsub_rn(thr_l, thr_b), 1024.0);
    const double a = best_is_l ? __dadd_rn(0.01, __dmul_rn(0.09, u3)) : __ddiv_rn(glarge, __dmul_rn(dl, dl));
    const bool last = (g == p.G - 1);
    const uint32_t cnt = last ? p.cnt_last : p.cnt_full;
    const int64_t o0 = (int64_t)(j * p.cnt_full);
    if (lane == 0) {
      if (p.off) { p.off[j] = o0; if (j == nG - 1) p.off[nG] = o0 + cnt; }
      if (p.gk) p.gk[j] = (uint32_t)kern;
      if (p.gm) p.gm[j] = mat;
    }
    for (uint32_t i = lane; i < cnt; i += 32) {
      const uint32_t b = p.mod > 1 ? p.rem + i * p.mod : i;
      const uint64_t row = g * p.L + b;
      const double u4 = unif(p.s[4], row), u5 = unif(p.s[5], row);
      const double thr = __dmul_rn(32.0, __dadd_rn((double)b, 1.0));
      const double d = __ddiv_rn(__dsub_rn(thr, thr_b), 1024.0);
      double r = __dmul_rn(T0, __dadd_rn(1.0, __dmul_rn(a, __dmul_rn(d, d))));
      r = __dmul_rn(r, __dadd_rn(1.0, __dmul_rn(0.005, u4)));
      const double sep = __dmul_rn(T0, 1.0001);
      if (r < sep) r = sep;
      if ((int64_t)b == bstar) r = T0;
      const bool isnan_ = u5 < p.nan_rate;
      const uint64_t at = (uint64_t)o0 + i;
      p.rt[at] = isnan_ ? __int_as_float(0x7FC00000) : __double2float_rn(r);
      p.bid[at] = (uint16_t)b;
      if (p.st) p.st[at] = isnan_ ? LSCAT_ROW_TIMEOUT : LSCAT_ROW_OK;
    }
  }
  (void)FULL;
}

uint64_t host_smix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

bool shape(const lscat_gen_opts* o, uint64_t* G, uint64_t* gb, uint64_t* ge, uint32_t* cf,
           uint32_t* cl) {
  if (!o || o->n_blocks == 0 || o->n_blocks > 65535 || o->n_kernels == 0 || o->n_matrices == 0 ||
      o->largest_block_id >= o->n_blocks || o->n_rows_global == 0 || o->preset > 1)
    return false;
  *G = (o->n_rows_global + o->n_blocks - 1) / o->n_blocks;
  *gb = o->group_begin;
  *ge = o->group_end ? o->group_end : *G;
  if (*gb > *ge || *ge > *G) return false;
  const uint32_t mod = o->block_mod > 1 ? o->block_mod : 1, rem = o->block_mod > 1 ? o->block_rem : 0;
  if (rem >= mod) return false;
  const uint32_t last_rows = (uint32_t)(o->n_rows_global - (*G - 1) * o->n_blocks);
  auto kept = [&](uint32_t nrows) { return nrows > rem ? (nrows - rem + mod - 1) / mod : 0u; };
  *cf = kept(o->n_blocks);
  *cl = kept(last_rows);
  return true;
}

}  // namespace
}  // namespace lscat

using namespace lscat;

extern "C" {

lscat_status lscat_gen_table_shape(const lscat_gen_opts* o, uint64_t* n_rows, uint64_t* n_groups) {
  uint64_t G, gb, ge;
  uint32_t cf, cl;
  if (!n_rows || !n_groups || !shape(o, &G, &gb, &ge, &cf, &cl)) return LSCAT_ERR_INVALID_ARG;
  *n_groups = ge - gb;
  *n_rows = (ge - gb) * cf;
  if (ge == G && ge > gb) *n_rows = *n_rows - cf + cl;
  return LSCAT_OK;
}

lscat_status lscat_gen_table(lscat_ctx* ctx, const lscat_gen_opts* o, lscat_table* out, void* stream) {
  LSCAT_CHECK_CTX(ctx);
  uint64_t G, gb, ge, nrows, ngroups;
  uint32_t cf, cl;
  if (!out || !shape(o, &G, &gb, &ge, &cf, &cl) || lscat_gen_table_shape(o, &nrows, &ngroups))
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "gen_table: bad options");
  if (out->mem != LSCAT_MEM_DEVICE || !out->runtime_ms || !out->block_id || out->cap_rows < nrows ||
      out->cap_groups < ngroups)
    return fail(ctx, LSCAT_ERR_INVALID_ARG, "gen_table: device table of %llu rows / %llu groups needed",
                (unsigned long long)nrows, (unsigned long long)ngroups);
  GP p{};
  p.G = G; p.n_rows_global = o->n_rows_global; p.gb = gb; p.ge = ge;
  p.K = o->n_kernels; p.L = o->n_blocks; p.ell = o->largest_block_id; p.M = o->n_matrices;
  p.mod = o->block_mod > 1 ? o->block_mod : 1; p.rem = o->block_mod > 1 ? o->block_rem : 0;
  p.cnt_full = cf; p.cnt_last = cl;
  p.q = G / o->n_kernels; p.r = G % o->n_kernels;
  p.nan_rate = o->nan_rate;
  if (o->preset == LSCAT_PRESET_T4) {
    p.c0 = 0.17; p.c1 = 0.88; p.c2 = 0.90;
    p.lo1 = 0.0; p.hi1 = 0.074; p.lo2 = 0.1765; p.hi2 = 0.2; p.lo3 = 0.2; p.hi3 = 0.4;
  } else {
    p.c0 = 0.17; p.c1 = 0.99; p.c2 = 1.00;
    p.lo1 = 0.0; p.hi1 = 0.02; p.lo2 = 0.18; p.hi2 = 1.5; p.lo3 = 0.18; p.hi3 = 1.5;
  }
  for (uint64_t i = 0; i < 6; i++) p.s[i] = host_smix(o->seed ^ (i * 0x9E3779B97F4A7C15ull));
  p.rt = out->runtime_ms; p.bid = out->block_id; p.st = out->status; p.off = out->group_offset;
  p.gk = out->group_kernel; p.gm = out->group_matrix;
  cudaStream_t s = (cudaStream_t)stream;
  LSCAT_CUDA(ctx, cudaSetDevice(ctx->device));
  if (ngroups) {
    const uint64_t warps = ngroups;
    const int grid = (int)std::min<uint64_t>((warps + 7) / 8, (uint64_t)ctx->sm_count * 32);
    gen_kernel<<<grid, 256, 0, s>>>(p);
    ctx->launches++;
    LSCAT_CUDA(ctx, cudaGetLastError());
  } else if (out->group_offset) {
    LSCAT_CUDA(ctx, cudaMemsetAsync(out->group_offset, 0, 8, s));
  }
  out->n_rows = nrows;
  out->n_groups = ngroups;
  out->first_group = gb;
  out->rows_per_group = (p.mod == 1 && (ge < G || cl == cf)) ? o->n_blocks : 0;
  return LSCAT_OK;
}

}  // extern "C"
