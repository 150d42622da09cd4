// rhs_w.cu — warp-synchronous fast path of the RHS for P = 2^21 (N1 = 1024 columns x N2 = 2048),
// the M = 2^20 shape of BASELINE configs 4 and 5.
//
// Same algebra as rhs.cu's four-step path (reference rhs.cpp:87-151 birth, 24-46 death,
// 170-210 shattering), restructured so every 1024-point transform is owned by ONE warp
// (warp_fft1024: two register radix-32 DFTs around one warp-private shared-memory exchange) —
// no block-wide barrier inside a transform, 2x fewer shared-memory passes than the radix-16
// Stockham path:
//   k_transpose_n : n -> column-major grid layout ng (so each column's operands are contiguous)
//   k_colw        : per (column, rank): z = (U_a n, V_a n) from the column-major UV copy (cp.async
//                   prefetch of the next rank), 1024-pt forward FFT (upper half zero), four-step
//                   twiddle, block-cooperative coalesced store of the Y tile; moment partials.
//   k_roww        : per row pair (k1, N1-k1), 4 warps: radix-2 DIF across two warps per row +
//                   1024-pt FFTs, conjugate-pair split, w*A*B summed over ranks in registers; then
//                   the inverse row transform of the Hermitian half-row and the inverse twiddle -> G.
//   k_colinvw     : per column pair, 1024-pt inverse FFT of G_a + i G_b (two real outputs),
//                   epilogue (birth/death/sources/shattering) block-cooperative and coalesced.
#include "rhs_common.cuh"

namespace agk {

constexpr int kW_N1 = 1024, kW_N2 = 2048, kW_H = kW_N1 / 2;
constexpr int kCW = 8;            // warps (columns) per column-kernel CTA
constexpr int kXR = kXS + 1;      // region stride (double2): successive regions on different banks


__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
  return x;
}

// n (natural, m) -> ng[n2 * 512 + n1] = n[n1 * 2048 + n2] (0 past m). 32x32 tiles.
__global__ void __launch_bounds__(256) k_transpose_n(RhsArgs a) {
  if (a.skip && *a.skip) return;
  __shared__ double t[32][33];
  const double* __restrict__ n = a.n.get();
  const int bx = blockIdx.x % (kW_N2 / 32), by = blockIdx.x / (kW_N2 / 32);  // n2 tile, n1 tile
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int n1 = by * 32 + ty + 8 * q, n2 = bx * 32 + tx;
    const int64_t i = (int64_t)n1 * kW_N2 + n2;
    t[ty + 8 * q][tx] = i < a.m ? n[i] : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int n2 = bx * 32 + ty + 8 * q, n1 = by * 32 + tx;
    a.ng[(int64_t)n2 * kW_H + n1] = t[tx][ty + 8 * q];
  }
}

template <int kCW, bool STAGE>
__global__ void __launch_bounds__(kCW * 32, STAGE ? 1 : 2) k_colw(RhsArgs a, int g0, int gcount) {
  extern __shared__ double2 smem[];
  double2* X = smem;                       // kCW exchange / output regions
  double2* S = X + kCW * kXR;              // kCW staging regions (512 x (U,V)), STAGE only
  double2* tw = S + (STAGE ? kCW * kW_H : 0);  // W_1024^{l k1}, [k1][l]
  __shared__ double red[kCW][4];
  __shared__ double2 tk[kCW][32];  // four-step factors W_P^{32 n2 k} of the warp's column
  if (a.skip && *a.skip) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int ngroups = kW_N2 / kCW;
  // persistent over (column group, rank) items, rank-minor so n is reloaded only per group
  const int items = ngroups * gcount;
  const int it0 = (int)((int64_t)blockIdx.x * items / gridDim.x);
  const int it1 = (int)((int64_t)(blockIdx.x + 1) * items / gridDim.x);
  for (int i = tid; i < 1024; i += blockDim.x) tw[i] = __ldg(a.tw32 + i);
  double2* Sw = S + w * kW_H;
  double2* Xw = X + w * kXR;
  auto prefetch = [&](int item) {
    if constexpr (STAGE) {
      const int grp = item / gcount, ub = g0 + item % gcount;
      const int n2 = grp * kCW + w;
      const double2* src = a.uvg + ((int64_t)ub * kW_N2 + n2) * kW_H;
#pragma unroll
      for (int r = 0; r < 16; ++r) cp_async16(Sw + lane + 32 * r, src + lane + 32 * r);
      cp_async_commit();
    }
  };
  if (it0 < it1) prefetch(it0);
  __syncthreads();
  double nl[16];
  double2 base = czero();
  int cur_grp = -1;
  const int64_t P = (int64_t)kW_N1 * kW_N2;
  for (int item = it0; item < it1; ++item) {
    const int grp = item / gcount, g = item % gcount, ub = g0 + g;
    const int n2 = grp * kCW + w;
    if (grp != cur_grp) {
      cur_grp = grp;
#pragma unroll
      for (int r = 0; r < 16; ++r) nl[r] = a.ng[(int64_t)n2 * kW_H + lane + 32 * r];
      base = tw_p<-1>(a.twp, (uint32_t)(n2 * lane));
      tk[w][lane] = tw_p<-1>(a.twp, (uint32_t)(32 * n2 * lane));
    }
    if constexpr (STAGE) {
      cp_async_wait_all();
      __syncwarp();
    }
    const double2* uvsrc = STAGE ? Sw : a.uvg + ((int64_t)ub * kW_N2 + n2) * kW_H;
    double2 v[32];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const double2 uv = uvsrc[lane + 32 * r];
      const double x = uv.x * nl[r], y = uv.y * nl[r];
      v[r] = make_double2(x, y);
      const int64_t i = (int64_t)(lane + 32 * r) * kW_N2 + n2;  // zero-filled past m
      if (i >= 1) {
        const double sz = (double)(i + 1);
        s0 += x;
        s1 += sz * x;
        s2 += y;
        s3 += sz * y;
      }
    }
#pragma unroll
    for (int r = 16; r < 32; ++r) v[r] = czero();
    __syncwarp();
    if (item + 1 < it1) prefetch(item + 1);
    if (!(a.dbg & 1)) warp_fft1024<-1, true>(v, Xw, tw, lane);
    // four-step twiddle W_P^{n2 k1c} = W_P^{n2 lane} W_P^{32 n2 k}, k1c = lane + 32 k
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 32; ++k) Xw[lane + 32 * k] = cmul(v[k], cmul(base, tk[w][k]));
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    s3 = warp_sum(s3);
    if (lane == 0) {
      red[w][0] = s0;
      red[w][1] = s1;
      red[w][2] = s2;
      red[w][3] = s3;
    }
    __syncthreads();
    // coalesced store of the tile: rows k1c, kCW consecutive columns
    double2* __restrict__ yg = a.y + (int64_t)g * P + (int64_t)grp * kCW;
    if (!(a.dbg & 2))
    for (int idx = tid; idx < kW_N1 * kCW; idx += blockDim.x) {
      const int k1c = idx / kCW, ww = idx % kCW;
      yg[(int64_t)k1c * kW_N2 + ww] = X[ww * kXR + k1c];
    }
    if (tid < 4) {
      double t = 0.0;
      for (int q = 0; q < kCW; ++q) t += red[q][tid];
      a.partials[((int64_t)ub * a.nblk_colfwd + grp) * 4 + tid] = t;
    }
    __syncthreads();
  }
}

// row pair (k1, N1-k1): warps (rho, h): rho = row, h = output parity of the radix-2 DIF split.
// One CTA of 4 warps per SM; the next rank's two rows are staged by cp.async while this rank's
// transforms run (the warp FFT keeps ~90% of its throughput at one warp per SMSP).
template <bool STAGE>
__global__ void __launch_bounds__(128, STAGE ? 1 : 2) k_roww(RhsArgs a, int g0, int gcount, int first) {
  extern __shared__ double2 smem[];
  double2* X = smem;               // 4 regions
  double2* tw = X + 4 * kXR;       // W_1024^{l k1}, [k1][l]
  double2* twh = tw + 1024;        // W_2048^{l + 32 r}, [r][l]
  double2* St = twh + 1024;        // staging: 2 rows x 2048
  if (a.skip && *a.skip) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, rho = w >> 1, h = w & 1;
  const int n1 = a.n1;
  const int P = kW_N1 * kW_N2;
  const int nrows = n1 / 2 + 1;
  // items: (row pair k1, rank g), rank-minor; a CTA owns whole row pairs (acc in registers)
  auto prefetch = [&](int k1, int g) {
    if constexpr (!STAGE) return;
    if (a.dbg & 64) return;
    const double2* y0 = a.y + (int64_t)g * P + (int64_t)k1 * kW_N2;
    const double2* y1 = a.y + (int64_t)g * P + (int64_t)((n1 - k1) & (n1 - 1)) * kW_N2;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int e = tid + 128 * q;
      cp_async16(St + e, y0 + e);
      cp_async16(St + kW_N2 + e, y1 + e);
    }
    cp_async_commit();
  };
  if ((int)blockIdx.x < nrows && gcount > 0) prefetch(blockIdx.x, 0);
  for (int i = tid; i < 1024; i += blockDim.x) {
    tw[i] = __ldg(a.tw32 + i);
    twh[i] = __ldg(a.tw2048h + i);
  }
  double2* Xw = X + w * kXR;
  const double2* Sr = St + rho * kW_N2;
  for (int k1 = blockIdx.x; k1 < nrows; k1 += gridDim.x) {
    double2 acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = first ? czero() : a.acc[(int64_t)k1 * kW_N2 + tid + 128 * j];
    for (int g = 0; g < gcount; ++g) {
      const double wt = a.uniq_weight[g0 + g];
      if constexpr (STAGE) { if (!(a.dbg & 64)) cp_async_wait_all(); }
      __syncthreads();  // staged rows visible; previous split done with X
      double2 v[32];
      const double2* src = STAGE ? Sr : a.y + (int64_t)g * P + (int64_t)(rho == 0 ? k1 : (n1 - k1) & (n1 - 1)) * kW_N2;
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const double2 lo = src[lane + 32 * r], hi = src[1024 + lane + 32 * r];
        v[r] = h == 0 ? cadd(lo, hi) : cmul(csub(lo, hi), twh[r * 32 + lane]);
      }
      __syncthreads();  // everyone has read the staging buffer
      if (g + 1 < gcount) {
        prefetch(k1, g + 1);
      } else if (k1 + (int)gridDim.x < nrows && gcount > 0) {
        prefetch(k1 + gridDim.x, 0);
      }
      if (!(a.dbg & 16)) warp_fft1024<-1, false>(v, Xw, tw, lane);
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 32; ++k) Xw[lane + 32 * k] = v[k];  // X_row[2(lane + 32k) + h]
      __syncthreads();
      if (!(a.dbg & 32))
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int q = tid + 128 * j;
        const int pq = (k1 == 0) ? ((kW_N2 - q) & (kW_N2 - 1)) : (kW_N2 - 1 - q);
        const double2 z = X[(q & 1) * kXR + (q >> 1)];
        const double2 zp = X[(2 + (pq & 1)) * kXR + (pq >> 1)];
        const double2 pr = split_product(z, zp);
        acc[j].x += wt * pr.x;
        acc[j].y += wt * pr.y;
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) a.acc[(int64_t)k1 * kW_N2 + tid + 128 * j] = acc[j];
  }
}

// inverse row transform of the Hermitian half-rows k1 = 0..N1/2 (2 warps per row, radix-2 DIF),
// inverse four-step twiddle -> G rows; block 0 also reduces the moment partials into the scalars
__global__ void __launch_bounds__(128) k_rowinvw(RhsArgs a) {
  extern __shared__ double2 smem[];
  double2* X = smem;               // 4 regions: two rows' halves
  double2* tw = X + 4 * kXR;
  double2* twh = tw + 1024;
  __shared__ double2 tkk[4][32];
  if (a.skip && *a.skip) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, sub = w >> 1, h = w & 1;
  const int P = kW_N1 * kW_N2;
  for (int i = tid; i < 1024; i += blockDim.x) {
    tw[i] = __ldg(a.tw32 + i);
    twh[i] = __ldg(a.tw2048h + i);
  }
  __syncthreads();
  const int nrows = kW_N1 / 2 + 1;
  for (int k1b = 2 * blockIdx.x; k1b < nrows; k1b += 2 * gridDim.x) {
    const int k1 = k1b + sub;
    double2 v[32];
    if (k1 < nrows) {
      const double2* __restrict__ ar = a.acc + (int64_t)k1 * kW_N2;
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] = ar[lane + 32 * r];
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const double2 hi = ar[1024 + lane + 32 * r];
        v[r] = h == 0 ? cadd(v[r], hi) : cmul(csub(v[r], hi), cconj(twh[r * 32 + lane]));
      }
      warp_fft1024<+1, false>(v, X + w * kXR, tw, lane);
    }
    __syncthreads();  // all rows of this pass loaded before G overwrites acc rows
    if (k1 < nrows) {
      // T[c2], c2 = 2(lane + 32k) + h; G = T W_P^{-c2 k1} = T W_P^{-(2 lane + h) k1} W_P^{-64 k1 k}
      const double2 base = tw_p<+1>(a.twp, (uint32_t)((2 * lane + h) * k1));
      tkk[w][lane] = tw_p<+1>(a.twp, (uint32_t)((64 * k1 * lane) & (P - 1)));
      __syncwarp();
      double2* __restrict__ gr = a.acc + (int64_t)k1 * kW_N2;
#pragma unroll
      for (int k = 0; k < 32; ++k) gr[2 * (lane + 32 * k) + h] = cmul(v[k], cmul(base, tkk[w][k]));
    }
    __syncthreads();
  }
}

// w_a, pair and monomer gains from the column pass' partials (one CTA, fixed order)
__global__ void __launch_bounds__(256) k_scalars_w(RhsArgs a) {
  if (a.skip && *a.skip) return;
  double* tot = a.scalars + a.r + 2;
  reduce_partials(a, a.nblk_colfwd, tot);
  __syncthreads();
  if (threadIdx.x == 0) finalize_scalars(a, tot, a.n.get()[0]);
}

// The non-birth part of S for every size: -n_s sum_a U_sa w_a [+ shattering] [+ sources]
// (rhs.cpp:24-46, 162-168, 170-210, 227-229). A pure stream over U (R x M) at full occupancy;
// it runs on the side stream while the row transforms run.
__global__ void __launch_bounds__(256) k_dvec(RhsArgs a) {
  if (a.skip && *a.skip) return;
  const double* __restrict__ n = a.n.get();
  RhsArgs b = a;
  b.flags = a.flags & ~T_BIRTH;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < a.m; s += (int64_t)gridDim.x * blockDim.x)
    a.dvec[s] = s == 0 ? epilogue0(b, n) : epilogue(b, n, s, 0.0);
}

// Inverse column pass: two real columns per complex 1024-pt inverse FFT, then S = birth + D.
template <int kCW>
__global__ void __launch_bounds__(kCW * 32, kCW == 8 ? 1 : 2) k_colinvw(RhsArgs a) {
  extern __shared__ double2 smem[];
  double2* X = smem;
  double2* tw = X + kCW * kXR;
  if (a.skip && *a.skip) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i < 1024; i += blockDim.x) tw[i] = __ldg(a.tw32 + i);
  __syncthreads();
  const double2* __restrict__ G = a.acc;
  const double scale = ldexp(0.5, -a.log2p);
  const bool birth = (a.flags & T_BIRTH) != 0;
  double* tile = reinterpret_cast<double*>(X);  // [512][2 kCW + 1] birth values, after the FFTs
  constexpr int TS = 2 * kCW + 1;
  for (int grp = blockIdx.x; grp < kW_N2 / (2 * kCW); grp += gridDim.x) {
    const int col = (grp * kCW + w) * 2;
    double2 v[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int k1 = lane + 32 * r;
      const bool refl = k1 > kW_N1 / 2;
      const int rowi = refl ? kW_N1 - k1 : k1;
      const double4 g4 = *reinterpret_cast<const double4*>(G + (int64_t)rowi * kW_N2 + col);
      double2 ga = make_double2(g4.x, g4.y), gb = make_double2(g4.z, g4.w);
      if (refl) {
        ga = cconj(ga);
        gb = cconj(gb);
      }
      v[r] = make_double2(ga.x - gb.y, ga.y + gb.x);
    }
    warp_fft1024<+1, false>(v, X + w * kXR, tw, lane);
    __syncthreads();  // all exchanges done: the regions become the birth tile
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int nn1 = lane + 32 * k;
      tile[nn1 * TS + 2 * w] = scale * v[k].x;
      tile[nn1 * TS + 2 * w + 1] = scale * v[k].y;
    }
    __syncthreads();
    for (int idx = tid; idx < kW_H * 2 * kCW; idx += blockDim.x) {
      const int nn1 = idx / (2 * kCW), c = idx % (2 * kCW);
      const int64_t jo = (int64_t)nn1 * kW_N2 + grp * 2 * kCW + c + 1;
      if (jo < a.m) a.out[jo] = (birth ? tile[nn1 * TS + c] : 0.0) + a.dvec[jo];
    }
    if (grp == 0 && tid == 0) a.out[0] = a.dvec[0];
    __syncthreads();
  }
}

template <int CW, bool STAGE>
static size_t smem_colw() { return (size_t)(CW * kXR + (STAGE ? CW * kW_H : 0) + 1024) * sizeof(double2); }
template <bool STAGE>
static size_t smem_roww() { return (size_t)(4 * kXR + 2048 + (STAGE ? 2 * kW_N2 : 0)) * sizeof(double2); }
static size_t smem_rowinvw() { return (size_t)(4 * kXR + 2048) * sizeof(double2); }
template <int CW>
static size_t smem_colinvw() { return (size_t)(CW * kXR + 1024) * sizeof(double2); }

// tuning knobs (AGK_WVAR): 0 = staged 8-warp column CTAs + staged row CTAs (1/SM);
// 1 = unstaged 4-warp column CTAs and row CTAs (2/SM); 2 = column staged, row unstaged
static int wvar() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("AGK_WVAR");
    v = e ? atoi(e) : 0;
  }
  return v;
}

cudaError_t rhs_w_set_smem_limits() {
  cudaError_t e;
#define SET(fn, bytes) \
  if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(bytes))) != cudaSuccess) return e;
  SET((k_colw<8, true>), (smem_colw<8, true>()));
  SET((k_colw<4, false>), (smem_colw<4, false>()));
  SET((k_roww<true>), (smem_roww<true>()));
  SET((k_roww<false>), (smem_roww<false>()));
  SET(k_rowinvw, smem_rowinvw());
  SET((k_colinvw<8>), (smem_colinvw<8>()));
  SET((k_colinvw<4>), (smem_colinvw<4>()));
#undef SET
  return cudaSuccess;
}

cudaError_t rhs_w_launch(const RhsPlan& p, const RhsArgs& a0, cudaStream_t s, void (*mark)(void*, int, cudaStream_t),
                         void* mk) {
  RhsArgs a = a0;
  if (const char* e = getenv("AGK_DBG")) a.dbg = atoi(e);
  const int nsm = 148;
  const int v = wvar();
  if (v == 3 && p.colstream) {
    // rank pipeline: col(g) on colstream into Y[g % 2], row(g) on s; col(g+2) waits row(g)
    const int64_t P = (int64_t)kW_N1 * kW_N2;
    a.nblk_colfwd = kW_N2 / 8;
    cudaEventRecord(p.ev_start, s);
    cudaStreamWaitEvent(p.colstream, p.ev_start, 0);
    k_transpose_n<<<(kW_H / 32) * (kW_N2 / 32), 256, 0, p.colstream>>>(a);
    for (int g = 0; g < a.rf; ++g) {
      RhsArgs ag = a;
      ag.y = a.y + (g & 1) * P;
      if (g >= 2) cudaStreamWaitEvent(p.colstream, p.ev_row[g & 1], 0);
      k_colw<8, true><<<nsm, 256, smem_colw<8, true>(), p.colstream>>>(ag, g, 1);
      cudaEventRecord(p.ev_col[g & 1], p.colstream);
      if (g + 1 == a.rf) {
        cudaStreamWaitEvent(p.side, p.ev_col[g & 1], 0);
        k_scalars_w<<<1, 256, 0, p.side>>>(a);
        k_dvec<<<4 * nsm, 256, 0, p.side>>>(a);
        cudaEventRecord(p.ev_join, p.side);
      }
      cudaStreamWaitEvent(s, p.ev_col[g & 1], 0);
      k_roww<true><<<nsm, 128, smem_roww<true>(), s>>>(ag, g, 1, g == 0);
      if (mark) mark(mk, K_ROW, s);
      cudaEventRecord(p.ev_row[g & 1], s);
    }
    k_rowinvw<<<(kW_N1 / 2 + 2) / 2 < 2 * nsm ? (kW_N1 / 2 + 2) / 2 : 2 * nsm, 128, smem_rowinvw(), s>>>(a);
    if (mark) mark(mk, K_ROW, s);
    cudaStreamWaitEvent(s, p.ev_join, 0);
    k_colinvw<8><<<kW_N2 / 16, 256, smem_colinvw<8>(), s>>>(a);
    if (mark) mark(mk, K_COL_INV, s);
    return cudaGetLastError();
  }
  const bool col8 = v != 1, rowstage = v == 0;
  const int cw = col8 ? 8 : 4;
  a.nblk_colfwd = kW_N2 / cw;
  k_transpose_n<<<(kW_H / 32) * (kW_N2 / 32), 256, 0, s>>>(a);
  if (mark) mark(mk, K_TRANSPOSE, s);
  for (int g0 = 0; g0 < a.rf; g0 += p.gsize) {
    const int gc = (a.rf - g0) < p.gsize ? (a.rf - g0) : p.gsize;
    const int items = (kW_N2 / cw) * gc;
    if (col8) {
      k_colw<8, true><<<items < nsm ? items : nsm, 256, smem_colw<8, true>(), s>>>(a, g0, gc);
    } else {
      k_colw<4, false><<<items < 2 * nsm ? items : 2 * nsm, 128, smem_colw<4, false>(), s>>>(a, g0, gc);
    }
    if (mark) mark(mk, K_COL_FWD, s);
    if (g0 + gc >= a.rf) {
      // fork: all column partials exist -> scalars and the non-birth part on the side stream
      cudaEventRecord(p.ev_fork, s);
      cudaStreamWaitEvent(p.side, p.ev_fork, 0);
      k_scalars_w<<<1, 256, 0, p.side>>>(a);
      k_dvec<<<4 * nsm, 256, 0, p.side>>>(a);
      cudaEventRecord(p.ev_join, p.side);
    }
    const int rows = kW_N1 / 2 + 1;
    if (rowstage) {
      k_roww<true><<<rows < nsm ? rows : nsm, 128, smem_roww<true>(), s>>>(a, g0, gc, g0 == 0);
    } else {
      k_roww<false><<<rows < 2 * nsm ? rows : 2 * nsm, 128, smem_roww<false>(), s>>>(a, g0, gc, g0 == 0);
    }
    if (mark) mark(mk, K_ROW, s);
  }
  k_rowinvw<<<(kW_N1 / 2 + 2) / 2 < 2 * nsm ? (kW_N1 / 2 + 2) / 2 : 2 * nsm, 128, smem_rowinvw(), s>>>(a);
  if (mark) mark(mk, K_ROW, s);
  // join the side stream (scalars + D) before the inverse column pass
  cudaStreamWaitEvent(s, p.ev_join, 0);
  if (col8) {
    k_colinvw<8><<<kW_N2 / 16, 256, smem_colinvw<8>(), s>>>(a);
  } else {
    k_colinvw<4><<<kW_N2 / 8, 128, smem_colinvw<4>(), s>>>(a);
  }
  if (mark) mark(mk, K_COL_INV, s);
  return cudaGetLastError();
}

}  // namespace agk
