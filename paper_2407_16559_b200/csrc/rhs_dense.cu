// rhs_dense.cu — the RHS for a DenseKernel (free-molecular and other kernels without an exact
// finite-rank form): the DenseKernel branches of the reference's
//   kernel_row_sums   rhs.cpp:37-45    rowsum_s = sum_j K(s,j) n_j
//   birth_term        rhs.cpp:153-159  birth_s  = 1/2 sum_{i<s} K(i,s-i) n_i n_{s-i}
//   shattering_terms  rhs.cpp:197-205  pair = sum_{i,j>=2} (i+j) K(i,j) n_i n_j,
//                                      mono = sum_{j>=2} j K(1,j) n_j
// with the same epilogue as the low-rank path (death, sources, shattering; rhs.cpp:212-235).
// O(M^2) work, HBM-bound: one pass over K for the row sums and one over its upper-left triangle
// (i + j <= M) for the birth sums. Every reduction is in a fixed order (bitwise reproducible).
//   k_dense_rows  : one warp per row: rowsum, and the row's shattering-gain term
//   k_dense_birth : CTA (256 consecutive output sizes s) x (chunk of 1024 rows i): thread s sums
//                   K(i, s-i) n_i n_{s-i} over the chunk — for fixed i consecutive threads read
//                   consecutive K entries — into a per-chunk partial
//   k_dense_pair  : one CTA: pair and mono gains
//   k_dense_epi   : birth = 1/2 sum of the chunk partials (ascending chunk), S = birth - death ...
#include "rhs_common.cuh"

namespace agk {

constexpr int kDenseS = 256;    // output sizes per birth CTA
constexpr int kDenseCh = 1024;  // rows per birth chunk

int dense_chunks(int64_t m) { return (int)((m + kDenseCh - 1) / kDenseCh); }

__device__ __forceinline__ double warp_sum_d(double x) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
  return x;
}

// row s (0-based) is size i = s + 1: rowsum[s] = sum_j K(i,j) n_j; pairc[s] = n_i (i sum_{j>=2}
// K(i,j) n_j + sum_{j>=2} j K(i,j) n_j) for i >= 2; pairc[0] = mono = sum_{j>=2} j K(1,j) n_j
__global__ void __launch_bounds__(256) k_dense_rows(RhsArgs a) {
  if (a.skip && *a.skip) return;
  const double* __restrict__ n = a.n.get();
  const int64_t m = a.m;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const bool shat = (a.flags & T_SHATTER) != 0;
  for (int64_t s = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); s < m; s += nw) {
    const double* __restrict__ kr = a.kd + s * m;
    double acc = 0.0, g0 = 0.0, g1 = 0.0;
    int64_t j = lane;
    for (; j + 96 < m; j += 128) {  // 4 loads in flight per lane
      double kv[4], nv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        kv[q] = __ldg(kr + j + 32 * q);
        nv[q] = n[j + 32 * q];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t jj = j + 32 * q;
        const double t = kv[q] * nv[q];
        acc += t;
        if (jj >= 1) {
          g0 += t;
          g1 += (double)(jj + 1) * t;
        }
      }
    }
    for (; j < m; j += 32) {
      const double t = __ldg(kr + j) * n[j];
      acc += t;
      if (j >= 1) {
        g0 += t;
        g1 += (double)(j + 1) * t;
      }
    }
    acc = warp_sum_d(acc);
    if (shat) {
      g0 = warp_sum_d(g0);
      g1 = warp_sum_d(g1);
    }
    if (lane == 0) {
      a.drow[s] = acc;
      if (shat) a.dpair[s] = s == 0 ? g1 : n[s] * ((double)(s + 1) * g0 + g1);
    }
  }
}

// partial[c][s - 1] = sum over rows i of chunk c, i < s, of K(i, s-i) n_i n_{s-i} (1-based sizes)
__global__ void __launch_bounds__(kDenseS) k_dense_birth(RhsArgs a) {
  if (a.skip && *a.skip) return;
  const double* __restrict__ n = a.n.get();
  const int64_t m = a.m;
  const int64_t s = (int64_t)blockIdx.x * kDenseS + threadIdx.x + 1;  // output size
  const int64_t smax = (int64_t)blockIdx.x * kDenseS + kDenseS;
  const int64_t i0 = (int64_t)blockIdx.y * kDenseCh + 1;
  if (i0 >= (smax < m ? smax : m)) return;  // chunk starts past every size of this CTA
  const int64_t i1 = i0 + kDenseCh - 1 < m ? i0 + kDenseCh - 1 : m;
  double acc = 0.0;
  int64_t i = i0;
  for (; i + 3 <= i1; i += 4) {
    double kv[4], nj[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t ii = i + q;
      const bool ok = ii < s && s <= m;
      kv[q] = ok ? __ldg(a.kd + (ii - 1) * m + (s - ii - 1)) : 0.0;
      nj[q] = ok ? n[s - ii - 1] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) acc += kv[q] * n[i + q - 1] * nj[q];
  }
  for (; i <= i1; ++i)
    if (i < s && s <= m) acc += __ldg(a.kd + (i - 1) * m + (s - i - 1)) * n[i - 1] * n[s - i - 1];
  if (s <= m) a.dpart[(int64_t)blockIdx.y * m + (s - 1)] = acc;
}

// scalars[r], scalars[r + 1] = pair, mono (fixed order: strided per thread, then a shuffle tree)
__global__ void __launch_bounds__(256) k_dense_pair(RhsArgs a) {
  if (a.skip && *a.skip) return;
  __shared__ double red[8];
  double t = 0.0;
  for (int64_t s = 1 + threadIdx.x; s < a.m; s += blockDim.x) t += a.dpair[s];
  t = warp_sum_d(t);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double p = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) p += red[q];
    a.scalars[0] = p;
    a.scalars[1] = a.dpair[0];
  }
}

__global__ void __launch_bounds__(256) k_dense_epi(RhsArgs a) {
  if (a.skip && *a.skip) return;
  const double* __restrict__ n = a.n.get();
  const int64_t m = a.m;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < m; o += (int64_t)gridDim.x * blockDim.x) {
    const double rs = a.drow[o];
    if (o == 0) {  // out[0]: no birth; death; shattering gains; sources at k = 1
      double res = 0.0;
      const double n0 = n[0];
      if (a.flags & T_DEATH) res = res - n0 * rs;
      if (a.flags & T_DEATH_POS) res = n0 * rs;
      if (a.flags & T_SHATTER) res = res + (0.5 * a.lambda * a.scalars[0] + a.lambda * n0 * a.scalars[1]);
      if (a.flags & T_SOURCES)
        for (int q = 0; q < a.nsrc; ++q)
          if (a.src_k[q] == 1) res += a.src_rate[q];
      a.out[0] = res;
      continue;
    }
    double birth = 0.0;
    if (a.flags & T_BIRTH) {
      // chunks c with c * 1024 + 1 <= s - 1 = o contributed to size s = o + 1
      const int nc = (int)((o - 1) / kDenseCh) + 1;
      double acc = 0.0;
      for (int c = 0; c < nc; ++c) acc += a.dpart[(int64_t)c * m + o];
      birth = 0.5 * acc;
    }
    a.out[o] = epilogue_rs(a, n, o, birth, rs);
  }
}

// Row-sum maximum partials for euler_stability_bound (rhs.cpp:284-294): rmax[b] = max over this
// CTA's rows of rowsum, from 0 (the reference's std::max fold), NaN-ignoring like it.
__global__ void __launch_bounds__(256) k_dense_rowmax(const double* rowsum, int64_t m, double* rmax) {
  __shared__ double red[8];
  double pk = 0.0;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m; s += (int64_t)gridDim.x * blockDim.x)
    pk = (pk < rowsum[s]) ? rowsum[s] : pk;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double o = __shfl_xor_sync(0xffffffffu, pk, off);
    pk = (pk < o) ? o : pk;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = pk;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < 8; ++q) t = (t < red[q]) ? red[q] : t;
    rmax[blockIdx.x] = t;
  }
}

static int rows_grid(int64_t m) {
  const int64_t g = (m + 7) / 8;
  return (int)(g < 148 * 8 ? g : 148 * 8);
}

cudaError_t rhs_dense_launch(const RhsPlan& p, const RhsArgs& a, cudaStream_t s, void (*mark)(void*, int, cudaStream_t),
                             void* mk) {
  (void)p;
  const int64_t m = a.m;
  k_dense_rows<<<rows_grid(m), 256, 0, s>>>(a);
  if (mark) mark(mk, K_DENSE_ROWS, s);
  if (a.flags & T_BIRTH) {
    k_dense_birth<<<dim3((unsigned)((m + kDenseS - 1) / kDenseS), (unsigned)dense_chunks(m)), kDenseS, 0, s>>>(a);
    if (mark) mark(mk, K_DENSE_BIRTH, s);
  }
  if (a.flags & T_SHATTER) k_dense_pair<<<1, 256, 0, s>>>(a);
  int64_t eg = (m + 255) / 256;
  k_dense_epi<<<(int)(eg < 148 * 4 ? eg : 148 * 4), 256, 0, s>>>(a);
  if (mark) mark(mk, K_COL_INV, s);
  return cudaGetLastError();
}

cudaError_t launch_dense_rowmax(const RhsArgs& md, VecRef n, double* rmax, int nblk, cudaStream_t s) {
  RhsArgs a = md;
  a.n = n;
  a.skip = nullptr;
  a.flags = T_DEATH;  // row sums only
  k_dense_rows<<<rows_grid(a.m), 256, 0, s>>>(a);
  k_dense_rowmax<<<nblk, 256, 0, s>>>(a.drow, a.m, rmax);
  return cudaGetLastError();
}

}  // namespace agk
