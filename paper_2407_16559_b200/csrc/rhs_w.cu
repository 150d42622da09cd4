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

// EOI: the group is columns {4 grp + j} and {1024 + 4 grp + j}, j < 4, and the tile store applies
// the first radix-2 DIF stage of the row transform, E[j] = y[j] + y[j + 1024] and
// O[j] = (y[j] - y[j + 1024]) W_2048^j, written interleaved in 64-byte chunks so each row of the
// tile is one full 128-byte line: Y row k1 = [E 0..3 | O 0..3 | E 4..7 | O 4..7 | ...]. The row
// kernel's warps then load their 1024-point half-row directly and run no combine pass.
template <int kCW, bool STAGE, bool EOI = false>
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
      const int n2 = EOI ? (w < 4 ? 4 * grp + w : kW_N2 / 2 + 4 * grp + w - 4) : grp * kCW + w;
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
    const int n2 = EOI ? (w < 4 ? 4 * grp + w : kW_N2 / 2 + 4 * grp + w - 4) : grp * kCW + w;
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
    if constexpr (EOI) {
      static_assert(!EOI || kCW == 8, "EOI groups are 4 + 4 columns");
      const int j = tid & 3;
      const double2 wj = a.tw2048h[4 * grp + j];  // W_2048^{4 grp + j}
      if (!(a.dbg & 2)) {
#pragma unroll 4
        for (int it = 0; it < kW_N1 / 64; ++it) {
          const int k1c = (tid >> 2) + 64 * it;
          const double2 lo = X[j * kXR + k1c], hi = X[(4 + j) * kXR + k1c];
          yg[(int64_t)k1c * kW_N2 + j] = cadd(lo, hi);
          yg[(int64_t)k1c * kW_N2 + 4 + j] = cmul(csub(lo, hi), wj);
        }
      }
    } else if (!(a.dbg & 2)) {
      for (int idx = tid; idx < kW_N1 * kCW; idx += blockDim.x) {
        const int k1c = idx / kCW, ww = idx % kCW;
        yg[(int64_t)k1c * kW_N2 + ww] = X[ww * kXR + k1c];
      }
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

// W_64^r = exp(-2 pi i r / 64) for r < 32, a compile-time constant after unrolling
__device__ __forceinline__ double2 w64(int r) {
  constexpr double c[17] = {1.0,
                            0.99518472667219688624,
                            0.98078528040323044913,
                            0.95694033573220886494,
                            0.92387953251128675613,
                            0.88192126434835502971,
                            0.83146961230254523708,
                            0.77301045336273696081,
                            0.70710678118654752440,
                            0.63439328416364549822,
                            0.55557023301960222474,
                            0.47139673682599764856,
                            0.38268343236508977173,
                            0.29028467725446236764,
                            0.19509032201612826785,
                            0.09801714032956060199,
                            0.0};
  // cos(2 pi r / 64) and sin(2 pi r / 64) = cos(2 pi (16 - r) / 64)
  const double cs = r <= 16 ? c[r] : -c[32 - r];
  const double sn = r <= 16 ? c[16 - r] : c[r - 16];
  return make_double2(cs, -sn);
}

// Row kernel: 8 warps = two independent halves (named barriers), each half owning one row pair
// (k1, N1-k1) at a time with warps (rho, h) = (row, output parity of the radix-2 DIF split).
// Every warp loads its own quarter of the row pair straight from global memory -- lo[j], hi[j]
// for 512 consecutive j -- forms E[j] = lo + hi and O[j] = (lo - hi) W_2048^j in registers and
// swaps the half its partner warp needs through its shared-memory region, so global loads are
// full-line coalesced, nothing is staged, and each 2048-point row costs two 1024-point warp FFTs.
// The two halves drift out of phase: one half's loads overlap the other half's transforms. The
// conjugate-pair split and w*A*B accumulate in registers over all ranks.
// Launched with 2 row pairs per half (grid = ceil(513 / 4) = 129 CTAs at N1 = 1024) so the SMs
// left over run the non-birth part D concurrently (k_dvec, programmatic dependent launch).
template <bool EOI>
__global__ void __launch_bounds__(256, 1) k_rown(RhsArgs a, int g0, int gcount, int first) {
  extern __shared__ double2 smem[];
  double2* X = smem;               // 8 regions: per half, row k1 (h = 0, 1) and row N1-k1 (h = 0, 1)
  double2* tw = X + 8 * kXR;       // W_1024^{l k1}, [k1][l]
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (a.skip && *a.skip) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, hf = w >> 2, hw = w & 3, rho = hw >> 1,
            h = hw & 1, ht = tid & 127;
  const int n1 = a.n1;
  const int64_t P = (int64_t)kW_N1 * kW_N2;
  const int nrows = n1 / 2 + 1;
  for (int i = tid; i < 1024; i += blockDim.x) tw[i] = __ldg(a.tw32 + i);
  const double2 wl = tw_p<-1>(a.twp, (uint32_t)(lane * (P / kW_N2)));  // W_2048^lane
  __syncthreads();
  double2* Xh = X + hf * 4 * kXR;
  double2* Xw = X + w * kXR;
  const double2* Xp = X + (w ^ 1) * kXR;
  const int bar = 1 + hf, pbar = 3 + (w >> 1);
  for (int k1 = 2 * blockIdx.x + hf; k1 < nrows; k1 += 2 * gridDim.x) {
    const int row = rho == 0 ? k1 : (n1 - k1) & (n1 - 1);
    const double2* rsrc = a.y + (int64_t)g0 * P + (int64_t)row * kW_N2 + h * (kW_N2 / 4);
    double2 acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = first ? czero() : a.acc[(int64_t)k1 * kW_N2 + ht + 128 * j];
    for (int g = 0; g < gcount; ++g) {
      const double wt = a.uniq_weight[g0 + g];
      const double2* __restrict__ src = rsrc + (int64_t)g * P;
      double2 v[32];
      if constexpr (EOI) {
        // element e of E (h = 0) / O (h = 1) sits at (e / 4) * 8 + 4 h + e % 4 of the row
        const double2* __restrict__ sh = src - h * (kW_N2 / 4) + 4 * h + (lane & 3) + 2 * (lane & ~3);
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = sh[64 * r];
      } else {
        // j = 512 h + lane + 32 r: E -> FFT slot (j mod 1024) / 32 of warp 0, O -> of warp 1
        if (h == 0) {
  #pragma unroll
          for (int r = 0; r < 16; ++r) {
            const double2 lo = src[lane + 32 * r], hi = src[kW_N2 / 2 + lane + 32 * r];
            v[r] = cadd(lo, hi);
            Xw[32 * r + lane] = cmul(csub(lo, hi), cmul(wl, w64(r)));
          }
        } else {
  #pragma unroll
          for (int r = 0; r < 16; ++r) {
            const double2 lo = src[lane + 32 * r], hi = src[kW_N2 / 2 + lane + 32 * r];
            v[16 + r] = cmul(csub(lo, hi), cmul(wl, w64(16 + r)));
            Xw[32 * r + lane] = cadd(lo, hi);
          }
        }
        asm volatile("bar.sync %0, 64;" ::"r"(pbar) : "memory");
        if (h == 0) {
  #pragma unroll
          for (int r = 0; r < 16; ++r) v[16 + r] = Xp[32 * r + lane];
        } else {
  #pragma unroll
          for (int r = 0; r < 16; ++r) v[r] = Xp[32 * r + lane];
        }
        asm volatile("bar.sync %0, 64;" ::"r"(pbar) : "memory");
      }
      if (!(a.dbg & 16)) warp_fft1024<-1, false>(v, Xw, tw, lane);
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 32; ++k) Xw[lane + 32 * k] = v[k];  // X_row[2(lane + 32k) + h]
      asm volatile("bar.sync %0, 128;" ::"r"(bar) : "memory");
      if (!(a.dbg & 32))
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int q = ht + 128 * j;
        const int pq = (k1 == 0) ? ((kW_N2 - q) & (kW_N2 - 1)) : (kW_N2 - 1 - q);
        const double2 z = Xh[(q & 1) * kXR + (q >> 1)];
        const double2 zp = Xh[(2 + (pq & 1)) * kXR + (pq >> 1)];
        const double2 pr = split_product(z, zp);
        acc[j].x += wt * pr.x;
        acc[j].y += wt * pr.y;
      }
      asm volatile("bar.sync %0, 128;" ::"r"(bar) : "memory");
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) a.acc[(int64_t)k1 * kW_N2 + ht + 128 * j] = acc[j];
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
  if (!(a.skip && *a.skip)) {
    const double* __restrict__ n = a.n.get();
    RhsArgs b = a;
    b.flags = a.flags & ~T_BIRTH;
    const bool rs = (a.flags & (T_DEATH | T_DEATH_POS | T_SHATTER)) != 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if ((a.m & 1) == 0) {
      // 4 x 2 sizes per thread (16-byte loads of U^T, four independent row-sum chains so the
      // loads of one rank step are in flight together); each size's sum runs in rank order
      const int64_t np = a.m / 2;
      for (int64_t p0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p0 < np; p0 += 4 * stride) {
        double r[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
        if (rs) {
          for (int ra = 0; ra < a.r; ++ra) {
            const double w = __ldg(a.scalars + ra);
            const double* __restrict__ ur = a.ut + (int64_t)ra * a.m;
            double2 u[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int64_t p = p0 + k * stride < np ? p0 + k * stride : np - 1;  // clamped: unpredicated
              u[k] = __ldg(reinterpret_cast<const double2*>(ur + 2 * p));
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              r[k][0] += u[k].x * w;
              r[k][1] += u[k].y * w;
            }
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int64_t p = p0 + k * stride;
          if (p < np) {
            const int64_t s = 2 * p;
            a.dvec[s] = s == 0 ? epilogue0(b, n) : epilogue_rs(b, n, s, 0.0, r[k][0]);
            a.dvec[s + 1] = epilogue_rs(b, n, s + 1, 0.0, r[k][1]);
          }
        }
      }
    } else {
      for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < a.m; s += stride)
        a.dvec[s] = s == 0 ? epilogue0(b, n) : epilogue(b, n, s, 0.0);
    }
  }
  // launched as a programmatic dependent of the row kernel: do not complete before it does, so
  // the launches after this one see the row results (no-op for an ordinary launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Inverse column pass: two real columns per complex 1024-pt inverse FFT, then S = birth + D.
// The CTA's G tile (rows 0..N1/2, 2 kCW columns) is loaded row-coalesced into shared memory
// first (padded rows: conflict-free column reads), then each warp gathers its column pair.
template <int kCW>
__global__ void __launch_bounds__(kCW * 32, kCW == 8 ? 1 : 2) k_colinvw(RhsArgs a) {
  extern __shared__ double2 smem[];
  double2* X = smem;  // the G tile, then the FFT exchange regions, then the birth tile
  constexpr int GS = 2 * kCW + 1, GROWS = kW_N1 / 2 + 1;
  double2* tw = X + GROWS * GS;
  double* dv = reinterpret_cast<double*>(tw + 1024);  // [512][2 kCW] D values of the output tile
  if (a.skip && *a.skip) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i < 1024; i += blockDim.x) tw[i] = __ldg(a.tw32 + i);
  const double2* __restrict__ G = a.acc;
  const double scale = ldexp(0.5, -a.log2p);
  const bool birth = (a.flags & T_BIRTH) != 0;
  double* tile = reinterpret_cast<double*>(X);  // [512][2 kCW + 1] birth values, after the FFTs
  constexpr int TS = 2 * kCW + 1;
  for (int grp = blockIdx.x; grp < kW_N2 / (2 * kCW); grp += gridDim.x) {
    const int col0 = grp * kCW * 2;
    __syncthreads();  // previous group's tile reads done
    // G tile and the D values of this output tile, all in flight at once (cp.async)
    for (int idx = tid; idx < GROWS * 2 * kCW; idx += kCW * 32) {
      const int row = idx / (2 * kCW), c = idx % (2 * kCW);
      cp_async16(X + row * GS + c, G + (int64_t)row * kW_N2 + col0 + c);
    }
    for (int idx = tid; idx < kW_H * 2 * kCW; idx += kCW * 32) {
      const int nn1 = idx / (2 * kCW), c = idx % (2 * kCW);
      const int64_t jo = (int64_t)nn1 * kW_N2 + col0 + c + 1;
      cp_async8(dv + idx, a.dvec + (jo < a.m ? jo : 0), jo < a.m);
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    double2 v[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int k1 = lane + 32 * r;
      const bool refl = k1 > kW_N1 / 2;
      const int rowi = refl ? kW_N1 - k1 : k1;
      double2 ga = X[rowi * GS + 2 * w], gb = X[rowi * GS + 2 * w + 1];
      if (refl) {
        ga = cconj(ga);
        gb = cconj(gb);
      }
      v[r] = make_double2(ga.x - gb.y, ga.y + gb.x);
    }
    __syncthreads();  // tile consumed: the region becomes the exchange buffers
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
      if (jo < a.m) a.out[jo] = (birth ? tile[nn1 * TS + c] : 0.0) + dv[idx];
    }
    if (grp == 0 && tid == 0) a.out[0] = a.dvec[0];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
// Rank-pipelined persistent RHS core (one launch per RHS, one CTA of 8 warps per SM, co-resident
// by cooperative launch). Every CTA walks the same phase sequence
//     col(0) | col(1) row(0) | col(2) row(1) | ... | row(R-1) + D slice
// doing its static share of each phase: column groups [b*256/nb, (b+1)*256/nb) and row pairs
// [b*513/nb, (b+1)*513/nb). Cross-CTA order comes from per-rank counters instead of launches or
// grid barriers: row(g) waits until every CTA finished col(g); col(g) overwrites the buffer of
// rank g-2 only after every CTA finished row(g-2). The per-rank intermediate is therefore double-
// buffered (2 x 32 MiB) and stays in L2; the spectral accumulator (16 MiB) is read-modify-written
// in L2 per rank. A CTA that finishes a phase early runs ahead into the next one, which absorbs the
// 256/148 and 513/148 quantisation that per-rank launches pay.
struct PipeSync {
  unsigned* col_done;  // [R]
  unsigned* row_done;  // [R]
  unsigned* scal_ready;
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void wait_count(const unsigned* c, unsigned target) {
  if (threadIdx.x == 0) {
    unsigned v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
      if (v >= target) break;
      __nanosleep(200);
    }
    __threadfence();
  }
  __syncthreads();
}
__device__ __forceinline__ void signal_count(unsigned* c) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(c, 1u);
  }
}

__global__ void __launch_bounds__(256, 1) k_pipe(RhsArgs a, PipeSync ps) {
  extern __shared__ double2 smem[];
  double2* X = smem;               // 8 exchange / tile regions
  double2* S = X + 8 * kXR;        // 8 column staging regions (512 x (U,V))
  double2* tw = S + 8 * kW_H;      // W_1024^{l k1}, [k1][l]
  __shared__ double red[8][4];
  __shared__ double2 tk[8][32];
  if (a.skip && *a.skip) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int nb = gridDim.x, b = blockIdx.x;
  const int R = a.rf;
  const int64_t P = (int64_t)kW_N1 * kW_N2;
  const int ngroups = kW_N2 / 8, nrows = kW_N1 / 2 + 1;
  for (int i = tid; i < 1024; i += blockDim.x) tw[i] = __ldg(a.tw32 + i);
  const double2 wl = tw_p<-1>(a.twp, (uint32_t)(lane * 1024));  // W_2048^lane = W_P^{1024 lane}
  __syncthreads();
  const int gb0 = b * ngroups / nb, gb1 = (b + 1) * ngroups / nb;
  const int pb0 = b * nrows / nb, pb1 = (b + 1) * nrows / nb;
  double2* Xw = X + w * kXR;
  double2* Sw = S + w * kW_H;

  auto col_phase = [&](int g) {
    const int ub = g;
    double2* yg = a.y + (int64_t)(g & 1) * P;
    auto prefetch = [&](int grp) {
      const int n2 = grp * 8 + w;
      const double2* src = a.uvg + ((int64_t)ub * kW_N2 + n2) * kW_H;
#pragma unroll
      for (int r = 0; r < 16; ++r) cp_async16(Sw + lane + 32 * r, src + lane + 32 * r);
      cp_async_commit();
    };
    if (gb0 < gb1) prefetch(gb0);
    for (int grp = gb0; grp < gb1; ++grp) {
      const int n2 = grp * 8 + w;
      double nl[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) nl[r] = a.ng[(int64_t)n2 * kW_H + lane + 32 * r];
      const double2 base = tw_p<-1>(a.twp, (uint32_t)(n2 * lane));
      tk[w][lane] = tw_p<-1>(a.twp, (uint32_t)(32 * n2 * lane));
      cp_async_wait_all();
      __syncwarp();
      double2 v[32];
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const double2 uv = Sw[lane + 32 * r];
        const double x = uv.x * nl[r], y = uv.y * nl[r];
        v[r] = make_double2(x, y);
        const int64_t i = (int64_t)(lane + 32 * r) * kW_N2 + n2;
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
      if (grp + 1 < gb1) prefetch(grp + 1);
      warp_fft1024<-1, true>(v, Xw, tw, lane);
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
      double2* __restrict__ yt = yg + (int64_t)grp * 8;
      for (int idx = tid; idx < kW_N1 * 8; idx += blockDim.x) {
        const int k1c = idx >> 3, ww = idx & 7;
        yt[(int64_t)k1c * kW_N2 + ww] = X[ww * kXR + k1c];
      }
      if (tid < 4) {
        double t = 0.0;
        for (int q = 0; q < 8; ++q) t += red[q][tid];
        a.partials[((int64_t)ub * ngroups + grp) * 4 + tid] = t;
      }
      __syncthreads();
    }
  };

  // two row pairs at a time: warps 0-3 pair p, warps 4-7 pair p+1; each half syncs on its own
  // named barrier. acc (16 complex per thread) is read-modify-written in L2 per rank.
  auto row_phase = [&](int g) {
    const double wt = a.uniq_weight[g];
    const double2* yg = a.y + (int64_t)(g & 1) * P;
    const int half = w >> 2, hw = w & 3, rho = hw >> 1, h = hw & 1, ht = tid & 127;
    double2* Xh = X + half * 4 * kXR;
    for (int p0 = pb0; p0 < pb1; p0 += 2) {
      const int k1 = p0 + half;
      const bool active = k1 < pb1;
      if (active) {
        const int row = rho == 0 ? k1 : (kW_N1 - k1) & (kW_N1 - 1);
        const double2* __restrict__ src = yg + (int64_t)row * kW_N2;
        double2 v[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = src[lane + 32 * r];
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          const double2 hi = src[1024 + lane + 32 * r];
          v[r] = h == 0 ? cadd(v[r], hi) : cmul(csub(v[r], hi), cmul(wl, w64(r)));
        }
        warp_fft1024<-1, false>(v, X + w * kXR, tw, lane);
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 32; ++k) X[w * kXR + lane + 32 * k] = v[k];
      }
      asm volatile("bar.sync %0, 128;" ::"r"(1 + half) : "memory");
      if (active) {
        double2* accr = a.acc + (int64_t)k1 * kW_N2;
#pragma unroll 4
        for (int j = 0; j < 16; ++j) {
          const int q = ht + 128 * j;
          const int pq = (k1 == 0) ? ((kW_N2 - q) & (kW_N2 - 1)) : (kW_N2 - 1 - q);
          const double2 z = Xh[(q & 1) * kXR + (q >> 1)];
          const double2 zp = Xh[(2 + (pq & 1)) * kXR + (pq >> 1)];
          const double2 pr = split_product(z, zp);
          double2 acc = g == 0 ? czero() : accr[q];
          acc.x += wt * pr.x;
          acc.y += wt * pr.y;
          accr[q] = acc;
        }
      }
      asm volatile("bar.sync %0, 128;" ::"r"(1 + half) : "memory");
    }
  };

  const bool tm = (a.dbg & 128) != 0;
  unsigned long long tacc[4] = {0, 0, 0, 0}, t0 = tm ? gtime() : 0, tl = t0;
  auto lap = [&](int k) {
    if (tm) {
      const unsigned long long t = gtime();
      tacc[k] += t - tl;
      tl = t;
    }
  };
  for (int step = 0; step <= R; ++step) {
    if (step < R) {
      if (step >= 2) wait_count(ps.row_done + step - 2, nb);  // buffer (step & 1) free again
      lap(0);
      if (!(a.dbg & 256)) col_phase(step);
      signal_count(ps.col_done + step);
      lap(1);
    }
    if (step >= 1) {
      wait_count(ps.col_done + step - 1, nb);
      lap(2);
      if (!(a.dbg & 512)) row_phase(step - 1);
      signal_count(ps.row_done + step - 1);
      lap(3);
    }
  }
  if (tm && tid == 0 && (b % 16 == 0 || b == nb - 1))
    printf("pipe cta %d: total %.1f us  waitcol %.1f col %.1f waitrow %.1f row %.1f  (groups %d pairs %d)\n", b,
           1e-3 * (tl - t0), 1e-3 * tacc[0], 1e-3 * tacc[1], 1e-3 * tacc[2], 1e-3 * tacc[3], gb1 - gb0, pb1 - pb0);
  // scalars (one CTA) and this CTA's slice of the non-birth part D
  if (b == 0) {
    wait_count(ps.col_done + R - 1, nb);
    double* tot = a.scalars + a.r + 2;
    reduce_partials(a, a.nblk_colfwd, tot);
    __syncthreads();
    if (tid == 0) {
      finalize_scalars(a, tot, a.n.get()[0]);
      __threadfence();
      atomicAdd(ps.scal_ready, 1u);
    }
  }
  wait_count(ps.scal_ready, 1);
  const double* __restrict__ n = a.n.get();
  RhsArgs bb = a;
  bb.flags = a.flags & ~T_BIRTH;
  const int64_t s0 = (int64_t)b * a.m / nb, s1 = (int64_t)(b + 1) * a.m / nb;
  for (int64_t s = s0 + tid; s < s1; s += blockDim.x) a.dvec[s] = s == 0 ? epilogue0(bb, n) : epilogue(bb, n, s, 0.0);
}

static size_t smem_pipe() { return (size_t)(8 * kXR + 8 * kW_H + 1024) * sizeof(double2); }

template <int CW, bool STAGE>
static size_t smem_colw() { return (size_t)(CW * kXR + (STAGE ? CW * kW_H : 0) + 1024) * sizeof(double2); }
template <bool STAGE>
static size_t smem_roww() { return (size_t)(4 * kXR + 2048 + (STAGE ? 2 * kW_N2 : 0)) * sizeof(double2); }
static size_t smem_rown() { return (size_t)(8 * kXR + 1024) * sizeof(double2); }
static size_t smem_rowinvw() { return (size_t)(4 * kXR + 2048) * sizeof(double2); }
template <int CW>
static size_t smem_colinvw() {
  const size_t tile = (size_t)(kW_N1 / 2 + 1) * (2 * CW + 1);
  return ((tile > (size_t)CW * kXR ? tile : (size_t)CW * kXR) + 1024 + (size_t)kW_H * CW) * sizeof(double2);
}

// tuning knobs (AGK_WVAR): 8 (default) = interleaved E/O column tiles + direct-load row kernel
// with D beside it; 7 = natural layout, direct-load row kernel with in-register radix-2;
// 0/5 = natural layout, staged row CTAs; 1 = unstaged 4-warp CTAs; 2 = row unstaged;
// 6 = rank-pipelined persistent kernel (experimental)
static int wvar() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("AGK_WVAR");
    v = e ? atoi(e) : 8;
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
  SET(k_rown<false>, smem_rown());
  SET(k_rown<true>, smem_rown());
  SET((k_colw<8, true, true>), (smem_colw<8, true>()));
  SET(k_pipe, smem_pipe());
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
  if (v == 6 && p.pipe_counters) {
    // rank-pipelined persistent core (experimental): one cooperative launch for all ranks
    a.nblk_colfwd = kW_N2 / 8;
    k_transpose_n<<<(kW_H / 32) * (kW_N2 / 32), 256, 0, s>>>(a);
    if (mark) mark(mk, K_TRANSPOSE, s);
    cudaMemsetAsync(p.pipe_counters, 0, (2 * (size_t)a.rf + 1) * sizeof(unsigned), s);
    PipeSync ps{p.pipe_counters, p.pipe_counters + a.rf, p.pipe_counters + 2 * a.rf};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.nsm);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem_pipe();
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_pipe, a, ps);
    if (e != cudaSuccess) return e;
    if (mark) mark(mk, K_ROW, s);
    k_rowinvw<<<(kW_N1 / 2 + 2) / 2 < 2 * nsm ? (kW_N1 / 2 + 2) / 2 : 2 * nsm, 128, smem_rowinvw(), s>>>(a);
    if (mark) mark(mk, K_ROW, s);
    k_colinvw<8><<<kW_N2 / 16, 256, smem_colinvw<8>(), s>>>(a);
    if (mark) mark(mk, K_COL_INV, s);
    return cudaGetLastError();
  }
  const bool eoi = v == 8;
  const bool rn = v == 7 || eoi;
  const bool col8 = v != 1, rowstage = v == 0 || v == 5;
  const int cw = col8 ? 8 : 4;
  a.nblk_colfwd = kW_N2 / cw;
  k_transpose_n<<<(kW_H / 32) * (kW_N2 / 32), 256, 0, s>>>(a);
  if (mark) mark(mk, K_TRANSPOSE, s);
  for (int g0 = 0; g0 < a.rf; g0 += p.gsize) {
    const int gc = (a.rf - g0) < p.gsize ? (a.rf - g0) : p.gsize;
    const int items = (kW_N2 / cw) * gc;
    if (eoi) {
      k_colw<8, true, true><<<items < nsm ? items : nsm, 256, smem_colw<8, true>(), s>>>(a, g0, gc);
    } else if (col8) {
      k_colw<8, true><<<items < nsm ? items : nsm, 256, smem_colw<8, true>(), s>>>(a, g0, gc);
    } else {
      k_colw<4, false><<<items < 2 * nsm ? items : 2 * nsm, 128, smem_colw<4, false>(), s>>>(a, g0, gc);
    }
    if (mark) mark(mk, K_COL_FWD, s);
    if (rn && g0 + gc >= a.rf) {
      k_scalars_w<<<1, 256, 0, s>>>(a);  // D then runs beside the last row launch
    } else if (g0 + gc >= a.rf) {
      // fork: all column partials exist -> scalars and the non-birth part on the side stream
      cudaEventRecord(p.ev_fork, s);
      cudaStreamWaitEvent(p.side, p.ev_fork, 0);
      k_scalars_w<<<1, 256, 0, p.side>>>(a);
      k_dvec<<<4 * nsm, 256, 0, p.side>>>(a);
      cudaEventRecord(p.ev_join, p.side);
    }
    const int rows = kW_N1 / 2 + 1;
    if (rn) {
      // 2 row pairs per half; the SMs left over run D (programmatic dependent launch: k_dvec
      // starts once every row CTA is resident and waits for the row grid before it exits)
      const int per = (rows + 2 * nsm - 1) / (2 * nsm);
      const int grid = (rows + 2 * per - 1) / (2 * per);
      if (eoi) {
        k_rown<true><<<grid, 256, smem_rown(), s>>>(a, g0, gc, g0 == 0);
      } else {
        k_rown<false><<<grid, 256, smem_rown(), s>>>(a, g0, gc, g0 == 0);
      }
      if (g0 + gc >= a.rf) {
        if (mark) mark(mk, K_ROW, s);
        const int free = nsm - grid;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(8 * (free > 1 ? free : 1));
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = mark ? 0 : 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_dvec, a);
        if (e != cudaSuccess) return e;
      }
    } else if (rowstage) {
      k_roww<true><<<rows < nsm ? rows : nsm, 128, smem_roww<true>(), s>>>(a, g0, gc, g0 == 0);
    } else {
      k_roww<false><<<rows < 2 * nsm ? rows : 2 * nsm, 128, smem_roww<false>(), s>>>(a, g0, gc, g0 == 0);
    }
    if (mark) mark(mk, K_ROW, s);
  }
  k_rowinvw<<<(kW_N1 / 2 + 2) / 2 < 2 * nsm ? (kW_N1 / 2 + 2) / 2 : 2 * nsm, 128, smem_rowinvw(), s>>>(a);
  if (mark) mark(mk, K_ROW, s);
  // join the side stream (scalars + D) before the inverse column pass
  if (!rn) cudaStreamWaitEvent(s, p.ev_join, 0);
  static const bool civ4 = getenv("AGK_CIV") && atoi(getenv("AGK_CIV")) == 4;
  if (col8 && !civ4) {
    k_colinvw<8><<<kW_N2 / 16, 256, smem_colinvw<8>(), s>>>(a);
  } else {
    k_colinvw<4><<<kW_N2 / 8, 128, smem_colinvw<4>(), s>>>(a);
  }
  if (mark) mark(mk, K_COL_INV, s);
  return cudaGetLastError();
}

}  // namespace agk
