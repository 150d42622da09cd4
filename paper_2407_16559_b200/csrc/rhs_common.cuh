// rhs_common.cuh — device helpers shared by the RHS kernels (rhs.cu, rhs_w.cu).
#pragma once
#include "internal.h"

namespace agk {

constexpr int kSwap = 1000000;  // rank_map code offset for swapped folds

// Sum NV doubles over the CTA (fixed shuffle tree + fixed warp order); result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&x)[NV], double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) x[k] += __shfl_xor_sync(0xffffffffu, x[k], off);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) red[warp * NV + k] = x[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += red[w * NV + k];
      x[k] = s;
    }
  }
  __syncthreads();
}

// Reduce the per-CTA moment partials [ub][blk][4] into tot[ub*4+q] (global or shared scratch)
// in a fixed order, by all warps of the calling CTA (blockDim a multiple of 32): a warp sums 8
// outputs at once, lane l taking blocks l, l+32, ... with all 64 loads of a 256-block chunk in
// flight, then a shuffle tree. Bitwise reproducible; ~one memory round trip per chunk.
__device__ __forceinline__ void reduce_partials_wide(const RhsArgs& a, int nblk, double* tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nout = a.rf * 4;
  for (int p0 = warp; p0 < nout; p0 += 8 * nw) {
    double s[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int b0 = 0; b0 < nblk; b0 += 256) {
      double x[8][8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int p = p0 + j * nw;
        const double* __restrict__ src = a.partials + (int64_t)(p >> 2) * nblk * 4 + (p & 3);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int b = b0 + lane + 32 * u;
          x[j][u] = (p < nout && b < nblk) ? src[(int64_t)b * 4] : 0.0;
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int u = 0; u < 8; ++u) s[j] += x[j][u];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s[j] += __shfl_xor_sync(0xffffffffu, s[j], off);
      const int p = p0 + j * nw;
      if (lane == 0 && p < nout) tot[p] = s[j];
    }
  }
}

// Register-light variant for kernels that carry transforms (one warp per output, fixed order).
// Reduce the per-CTA moment partials [ub][blk][4] into tot[ub*4+q] (global scratch), fixed
// order, by all warps of the calling CTA (blockDim a multiple of 32).
__device__ __forceinline__ void reduce_partials(const RhsArgs& a, int nblk, double* tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int p = warp; p < a.rf * 4; p += nw) {
    const int ub = p >> 2, q = p & 3;
    double s = 0.0;
    for (int b = lane; b < nblk; b += 32) s += a.partials[((int64_t)ub * nblk + b) * 4 + q];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) tot[p] = s;
  }
}

// w_a for every rank (folded ranks read their partner's sums), pair and monomer gains
// (rhs.cpp:24-36 and 185-196), written to a.scalars by one thread.
__device__ __forceinline__ void finalize_scalars(const RhsArgs& a, const double* tot, double n0) {
  double pair = 0.0, mono = 0.0;
  for (int ra = 0; ra < a.r; ++ra) {
    const int code = a.rank_map[ra];
    const bool sw = code >= kSwap;
    const int ub = sw ? code - kSwap : code;
    const double A0 = tot[ub * 4 + 0], A1 = tot[ub * 4 + 1];
    const double B0 = tot[ub * 4 + 2], B1 = tot[ub * 4 + 3];
    const double su0 = sw ? B0 : A0, su1 = sw ? B1 : A1;
    const double sv0 = sw ? A0 : B0, sv1 = sw ? A1 : B1;
    a.scalars[ra] = sv0 + a.v0[ra] * n0;  // w_a = sum_j V_aj n_j
    pair += su1 * sv0 + su0 * sv1;
    mono += a.u0[ra] * sv1;
  }
  a.scalars[a.r] = pair;
  a.scalars[a.r + 1] = mono;
}

// The same, by a whole CTA: each thread finishes its ranks' w_a and gain terms (the loads of
// all ranks in flight together), then thread 0 sums the gains in rank order. sh: 2 r doubles.
__device__ __forceinline__ void finalize_scalars_to(const RhsArgs& a, const double* tot, double n0, double* sh,
                                                    double* scal) {
  for (int ra = threadIdx.x; ra < a.r; ra += blockDim.x) {
    const int code = a.rank_map[ra];
    const bool sw = code >= kSwap;
    const int ub = sw ? code - kSwap : code;
    const double A0 = tot[ub * 4 + 0], A1 = tot[ub * 4 + 1];
    const double B0 = tot[ub * 4 + 2], B1 = tot[ub * 4 + 3];
    const double su0 = sw ? B0 : A0, su1 = sw ? B1 : A1;
    const double sv0 = sw ? A0 : B0, sv1 = sw ? A1 : B1;
    scal[ra] = sv0 + a.v0[ra] * n0;  // w_a = sum_j V_aj n_j
    sh[2 * ra] = su1 * sv0 + su0 * sv1;
    sh[2 * ra + 1] = a.u0[ra] * sv1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double pair = 0.0, mono = 0.0;
    for (int ra = 0; ra < a.r; ++ra) {
      pair += sh[2 * ra];
      mono += sh[2 * ra + 1];
    }
    scal[a.r] = pair;
    scal[a.r + 1] = mono;
  }
}
__device__ __forceinline__ void finalize_scalars_cta(const RhsArgs& a, const double* tot, double n0, double* sh) {
  for (int ra = threadIdx.x; ra < a.r; ra += blockDim.x) {
    const int code = a.rank_map[ra];
    const bool sw = code >= kSwap;
    const int ub = sw ? code - kSwap : code;
    const double A0 = tot[ub * 4 + 0], A1 = tot[ub * 4 + 1];
    const double B0 = tot[ub * 4 + 2], B1 = tot[ub * 4 + 3];
    const double su0 = sw ? B0 : A0, su1 = sw ? B1 : A1;
    const double sv0 = sw ? A0 : B0, sv1 = sw ? A1 : B1;
    a.scalars[ra] = sv0 + a.v0[ra] * n0;  // w_a = sum_j V_aj n_j
    sh[2 * ra] = su1 * sv0 + su0 * sv1;
    sh[2 * ra + 1] = a.u0[ra] * sv1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double pair = 0.0, mono = 0.0;
    for (int ra = 0; ra < a.r; ++ra) {
      pair += sh[2 * ra];
      mono += sh[2 * ra + 1];
    }
    a.scalars[a.r] = pair;
    a.scalars[a.r + 1] = mono;
  }
}

// Epilogue for output index jo >= 1: S = birth - death [+ shattering loss] [+ sources], with the
// death row sum sum_a U_sa w_a given (ascending a, as rhs.cpp:24-46 accumulates it)
__device__ __forceinline__ double epilogue_rsn(const RhsArgs& a, double nn, int64_t jo, double birth, double rowsum) {
  double res = (a.flags & T_BIRTH) ? birth : 0.0;
  if (a.flags & (T_DEATH | T_DEATH_POS | T_SHATTER)) {
    if (a.flags & T_DEATH) res = res - nn * rowsum;
    if (a.flags & T_DEATH_POS) res = nn * rowsum;
    if (a.flags & T_SHATTER) res = res + (-a.lambda * nn) * rowsum;
  }
  if (a.flags & T_SOURCES) {
    for (int q = 0; q < a.nsrc; ++q)
      if (a.src_k[q] - 1 == jo) res += a.src_rate[q];
  }
  return res;
}
__device__ __forceinline__ double epilogue_rs(const RhsArgs& a, const double* __restrict__ n, int64_t jo,
                                              double birth, double rowsum) {
  return epilogue_rsn(a, (a.flags & (T_DEATH | T_DEATH_POS | T_SHATTER)) ? n[jo] : 0.0, jo, birth, rowsum);
}
__device__ __forceinline__ double epilogue(const RhsArgs& a, const double* __restrict__ n,
                                           int64_t jo, double birth) {
  double rowsum = 0.0;
  if (a.flags & (T_DEATH | T_DEATH_POS | T_SHATTER)) {
    // loads batched 8 deep (the compiler otherwise issues them one FMA at a time); sum order kept
    int ra = 0;
    for (; ra + 8 <= a.r; ra += 8) {
      double u[8], w[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        u[k] = __ldg(a.ut + (int64_t)(ra + k) * a.m + jo);
        w[k] = a.scalars[ra + k];
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) rowsum += u[k] * w[k];
    }
    for (; ra < a.r; ++ra) rowsum += __ldg(a.ut + (int64_t)ra * a.m + jo) * a.scalars[ra];
  }
  return epilogue_rs(a, n, jo, birth, rowsum);
}

// D = the non-birth part of S at output index jo >= 1 (death, shattering loss, sources) from the
// row sum and n_jo, for term flags `fl` (epilogue_rsn with T_BIRTH cleared, without an RhsArgs copy)
__device__ __forceinline__ double dvalue(const RhsArgs& a, int fl, double nn, int64_t jo, double rowsum) {
  double res = 0.0;
  if (fl & T_DEATH) res = res - nn * rowsum;
  if (fl & T_DEATH_POS) res = nn * rowsum;
  if (fl & T_SHATTER) res = res + (-a.lambda * nn) * rowsum;
  if (fl & T_SOURCES) {
    for (int q = 0; q < a.nsrc; ++q)
      if (a.src_k[q] - 1 == jo) res += a.src_rate[q];
  }
  return res;
}
// D at index 0 (epilogue0 with the scalars w_a, pair, mono in `scal`)
__device__ __forceinline__ double dvalue0(const RhsArgs& a, int fl, const double* scal, double n0) {
  double res = 0.0;
  if (fl & (T_DEATH | T_DEATH_POS)) {
    double rowsum = 0.0;
    for (int ra = 0; ra < a.r; ++ra) rowsum += a.ut[(int64_t)ra * a.m] * scal[ra];
    if (fl & T_DEATH) res = res - n0 * rowsum;
    if (fl & T_DEATH_POS) res = n0 * rowsum;
  }
  if (fl & T_SHATTER) res = res + (0.5 * a.lambda * scal[a.r] + a.lambda * n0 * scal[a.r + 1]);
  if (fl & T_SOURCES) {
    for (int q = 0; q < a.nsrc; ++q)
      if (a.src_k[q] == 1) res += a.src_rate[q];
  }
  return res;
}

// out[0]: no birth; death; shattering gain at s = 1 (rhs.cpp:208); sources at k = 1.
__device__ __forceinline__ double epilogue0(const RhsArgs& a, const double* __restrict__ n) {
  double res = 0.0;
  const double n0 = n[0];
  if (a.flags & (T_DEATH | T_DEATH_POS)) {
    double rowsum = 0.0;
    for (int ra = 0; ra < a.r; ++ra) rowsum += a.ut[(int64_t)ra * a.m] * a.scalars[ra];
    if (a.flags & T_DEATH) res = res - n0 * rowsum;
    if (a.flags & T_DEATH_POS) res = n0 * rowsum;
  }
  if (a.flags & T_SHATTER) {
    const double pair = a.scalars[a.r], mono = a.scalars[a.r + 1];
    res = res + (0.5 * a.lambda * pair + a.lambda * n0 * mono);
  }
  if (a.flags & T_SOURCES) {
    for (int q = 0; q < a.nsrc; ++q)
      if (a.src_k[q] == 1) res += a.src_rate[q];
  }
  return res;
}

// conjugate-pair split and product of one packed spectrum bin (rhs.cpp:138-144):
// A = (Z + conj Zp)/2, B = -i/2 (Z - conj Zp), returns A*B
__device__ __forceinline__ double2 split_product(double2 z, double2 zp) {
  const double mr = zp.x, mi = -zp.y;
  const double ar = 0.5 * (z.x + mr), ai = 0.5 * (z.y + mi);
  const double dr = z.x - mr, di = z.y - mi;
  const double br = 0.5 * di, bi = -0.5 * dr;
  return make_double2(ar * br - ai * bi, ar * bi + ai * br);
}

// acc += w4 * A*B for the bin pair (z, zp) as split_product, with 4 A*B = -i (z + conj zp)(z - conj zp)
// formed directly (the factors 1/2 are powers of two: the same roundings) and w4 = weight / 4
__device__ __forceinline__ void split_product_acc4(double2& acc, double w4, double2 z, double2 zp) {
  const double sx = z.x + zp.x, sy = z.y - zp.y, dx = z.x - zp.x, dy = z.y + zp.y;
  acc.x = fma(w4, fma(sx, dy, sy * dx), acc.x);
  acc.y = fma(w4, fma(sy, dy, -(sx * dx)), acc.y);
}

// Four-step twiddles W_P^{SIGN e} for e = e0 + r*de, r = 0..E-1, by a short recurrence from two
// accurate two-level lookups (error ~r ulp, no per-element table loads).
template <int SIGN>
struct TwSeries {
  double2 w, st;
  __device__ __forceinline__ TwSeries(const TwoLevel& t, uint32_t e0, uint32_t de)
      : w(tw_p<SIGN>(t, e0)), st(tw_p<SIGN>(t, de)) {}
  __device__ __forceinline__ double2 next() {
    const double2 cur = w;
    w = cmul(w, st);
    return cur;
  }
};


}  // namespace agk
