// rhs_w.cu — warp-synchronous fast path of the RHS for P = 2^21 (N1 = 1024 columns x N2 = 2048),
// the M = 2^20 shape of BASELINE configs 4 and 5.
//
// Same algebra as rhs.cu's four-step path (reference rhs.cpp:87-151 birth, 24-46 death,
// 170-210 shattering), restructured so every 1024-point transform is owned by ONE warp
// (warp_fft1024: two register radix-32 DFTs around one warp-private shared-memory exchange) —
// no block-wide barrier inside a transform:
//   k_transpose_n : n -> column-major grid layout ng (so each column's operands are contiguous)
//   k_colx        : per (column octet, rank): z = (U_a n, V_a n) from the column-major UV copy
//                   (cp.async prefetch of the next item), 1024-pt forward FFT (upper half zero)
//                   exchanging inside one swizzled shared tile with step B dealt by (column, k), so
//                   the four-step-twiddled results leave the registers as full 128-byte lines of
//                   the even/odd-permuted Y rows; moment partials.
//   k_rowd        : per row pair (k1, N1-k1) x rank: 1024-pt FFTs of the even and odd samples,
//                   the decimation-in-time radix-2 stage fused into the conjugate-pair split,
//                   w*A*B summed over ranks in registers. Two independent 4-warp halves per CTA.
//                   The last launch also runs the inverse row transform of the Hermitian rows and
//                   the inverse four-step twiddle -> G.
//   k_colinvw     : per column pair, 1024-pt inverse FFT of G_a + i G_b (two real outputs),
//                   epilogue birth + D, where D (death/sources/shattering) came from k_dvec.
#include "rhs_common.cuh"

namespace agk {

constexpr int kW_N1 = 1024, kW_N2 = 2048, kW_H = kW_N1 / 2;
// Y row stride (double2) and rank stride: rows padded by one 128-byte line, so the 1024 lines a
// column item writes (one per row) do not all share the low address bits of a 32 KB stride
constexpr int kW_YPAD = 8, kW_YS = kW_N2 + kW_YPAD;
constexpr int64_t kW_YP = (int64_t)kW_N1 * kW_YS;
// Region stride (double2) of the per-warp exchange / output regions: = 4 (mod 8) so that two
// regions read at the same offset by neighbouring lanes sit on different 16-byte bank groups
// (the tile store of k_colh and the split product of k_rowh both read region pairs that way).
constexpr int kXR = kXS + 4;

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
  return x;
}

// Timeline diagnostics (AGK_DBG & 512, tools/timeline.py): per kernel class, the first CTA's
// arrival, the first CTA's start of work (after its programmatic-dependency wait) and the last
// CTA's exit, as %globaltimer ns, so the overlap of the chained launches can be seen in graph mode.
__device__ unsigned long long g_timeline[8][3];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void tl_mark(const RhsArgs& a, int k, int what) {
  if (AGK_XDBG(a, 512) && threadIdx.x == 0) {
    const unsigned long long t = gtimer();
    if (what < 2) atomicMin(&g_timeline[k][what], t);
    else atomicMax(&g_timeline[k][what], t);
  }
}

// the same with a run-time test (see ROW_XDBG below)
__device__ __forceinline__ void tl_mark_rt(const RhsArgs& a, int k, int what) {
  if ((a.dbg & 512) && threadIdx.x == 0) {
    const unsigned long long t = gtimer();
    if (what < 2) atomicMin(&g_timeline[k][what], t);
    else atomicMax(&g_timeline[k][what], t);
  }
}

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// n (natural, m) -> ng[n2 * 512 + n1] = n[n1 * 2048 + n2] (0 past m). 64 x 64 tiles, 16 elements
// per thread in flight, 256-byte coalesced rows both ways.
__global__ void __launch_bounds__(256) k_transpose_n(RhsArgs a) {
  tl_mark(a, 0, 0);
  pdl_entry();  // then the column pass' prologue may start
  tl_mark(a, 0, 1);
  if (a.skip && *a.skip) return;
  __shared__ double t[64][65];
  const double* __restrict__ n = a.n.get();
  const int bx = blockIdx.x % (kW_N2 / 64), by = blockIdx.x / (kW_N2 / 64);  // n2 tile, n1 tile
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  double v[16];
  if (a.st.on) {
    // fused RK stage: n_i = x_i + tau sum_j a_j k_j[i], formed here and also stored in natural
    // layout (the D kernel reads it)
    const double t = a.st.tau_mul * *a.st.tau;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int64_t i = (int64_t)(by * 64 + ty + 4 * q) * kW_N2 + bx * 64 + tx;
      v[q] = i < a.m ? stage_at(a.st, t, n[i], i) : 0.0;
      if (i < a.m) a.stg_out[i] = v[q];
    }
  } else {
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int64_t i = (int64_t)(by * 64 + ty + 4 * q) * kW_N2 + bx * 64 + tx;
      v[q] = i < a.m ? n[i] : 0.0;
    }
  }
#pragma unroll
  for (int q = 0; q < 16; ++q) t[ty + 4 * q][tx] = v[q];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 16; ++q) a.ng[(int64_t)(bx * 64 + ty + 4 * q) * kW_H + by * 64 + tx] = t[tx][ty + 4 * q];
  tl_mark(a, 0, 2);
}

// Y layout (per rank, [k1][slot], 2048 slots per row): the row transform's first radix-2 stage
// is decimation in time, so each row is stored even/odd-permuted, slot(n2) = (n2 & 1) * 1024 +
// (n2 >> 1): a row-pass warp then loads its 1024 even or odd samples as contiguous full lines.
//
// Column pass: a CTA item is (column octet o, rank): the 8 columns n2 = 16 (o >> 1) + 2 c + (o & 1),
// whose outputs are the 8 consecutive slots (o & 1) * 1024 + 8 (o >> 1) + c of every row (one
// 128-byte line per row). Items are rank-minor, so n is reloaded only per octet. The operands
// (U,V) of the next item are staged by cp.async while the current item is transformed.
//
// The transposition is done by the transform's own exchange (no output tile): step A per warp
// (warp w = column w of the octet, lane = l: radix-32 DFT with the upper half zero as two radix-16
// DFTs, twiddles by recurrence), exchanged through the CTA's
// 1024 x 8 tile, but step B is dealt across the CTA by (column, k): lane (c = lane & 7,
// kk = lane >> 3) of warp w' runs the radix-32 DFT over l of column c at k = 4 w' + kk and so
// holds X_c[k + 32 q], q < 32. A warp store at fixed q is then 4 rows (k .. k+3... one per kk) of
// 8 consecutive slots = four full 128-byte Y lines straight from registers: the tile write-back
// (32 STS.128 + 32 LDS.128 per thread and item) and the wait for the tile to drain are gone.
__global__ void __launch_bounds__(256, 1) k_colx(RhsArgs a, int g0, int gcount) {
  tl_mark(a, 1, 0);
  extern __shared__ double2 smem[];
  double2* T = smem;               // 1024 x 8 exchange tile (tile_idx)
  double2* S = T + 8 * kW_N1;      // 8 staging regions (512 x (U,V))
  double2* tw = S + 8 * kW_H;      // W_1024^{l k1}, [k1][l]
  double2* tq = tw + 1024;         // [4][256]: four-step chain heads W_P^{n2 (k + 32 j)} of this thread's (column, k)
  __shared__ double red[2][8][4];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int cB = lane & 7, kB = 4 * w + (lane >> 3);  // step-B role
  const int items = (kW_N2 / 8) * gcount;
  const int it0 = (int)((int64_t)blockIdx.x * items / gridDim.x);
  const int it1 = (int)((int64_t)(blockIdx.x + 1) * items / gridDim.x);
  for (int i = tid; i < 1024; i += blockDim.x) tw[i] = __ldg(a.tw32 + i);
  double2* Sw = S + w * kW_H;
  auto col_of = [&](int o, int c) { return 16 * (o >> 1) + 2 * c + (o & 1); };
  auto prefetch = [&](int item) {
    const int o = item / gcount, ub = g0 + item % gcount;
    const double2* src = a.uvg + ((int64_t)ub * kW_N2 + col_of(o, w)) * kW_H;
#pragma unroll
    for (int r = 0; r < 16; ++r) cp_async16(Sw + lane + 32 * r, src + lane + 32 * r);
    cp_async_commit();
  };
  if (it0 < it1) prefetch(it0);
  __syncthreads();
  pdl_entry();  // programmatic dependent of the transpose of n (ng is read only from here on)
  tl_mark(a, 1, 1);
  if (a.skip && *a.skip) {
    cp_async_wait_all();
    return;
  }
  double nl[16];
  double2 stB = czero();
  int cur_o = -1;
  for (int item = it0; item < it1; ++item) {
    const int o = item / gcount, g = item % gcount, ub = g0 + g;
    const int n2 = col_of(o, w);
    if (o != cur_o) {
      cur_o = o;
#pragma unroll
      for (int r = 0; r < 16; ++r) nl[r] = a.ng[(int64_t)n2 * kW_H + lane + 32 * r];
      // four-step factors of the step-B role: W_P^{n2B k1}, k1 = kB + 32 q, as four chains
      // t_{j+4m} = (W_P^{n2B kB} W_P^{32 n2B j}) (W_P^{128 n2B})^m 
      const int n2B = col_of(o, cB);
      const double2 base = tw_p<-1>(a.twp, (uint32_t)(n2B * kB));
#pragma unroll
      for (int j = 0; j < 4; ++j) tq[j * 256 + tid] = cmul(base, tw_p<-1>(a.twp, (uint32_t)(32 * n2B * j)));
      stB = tw_p<-1>(a.twp, (uint32_t)(32 * n2B * 4));
    }
    cp_async_wait_all();
    __syncwarp();
    double2 v[32];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const double2 uv = Sw[lane + 32 * r];
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
    __syncwarp();
    if (item + 1 < it1) prefetch(item + 1);
    {
      // step A: radix-32 DFT over r with the upper half zero, as two radix-16 DFTs
      double2 ea[16], ob[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        ea[r] = v[r];
        ob[r] = mul_w32<-1>(v[r], r);
      }
      Dft<16, -1>::run(ea);
      Dft<16, -1>::run(ob);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        v[2 * k] = ea[k];
        v[2 * k + 1] = ob[k];
      }
      twiddle_a_rec<-1>(v, tw, lane);
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    s3 = warp_sum(s3);
    if (lane == 0) {
      double* rd = red[item & 1][w];
      rd[0] = s0;
      rd[1] = s1;
      rd[2] = s2;
      rd[3] = s3;
    }
    __syncthreads();  // every thread has read the previous item's exchange
#pragma unroll
    for (int k = 0; k < 32; ++k) T[tile_idx(32 * k + lane, w)] = v[k];
    __syncthreads();
    if (tid < 4) {
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) t += red[item & 1][q][tid];
      a.partials[((int64_t)ub * a.nblk_colfwd + o) * 4 + tid] = t;
    }
    // step B in the (column, k) role
#pragma unroll
    for (int l = 0; l < 32; ++l) v[l] = T[tile_idx(32 * kB + l, cB)];
    Dft<32, -1>::run(v);
    double2 t[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) t[j] = tq[j * 256 + tid];
    // rows kB + 32 q, slots (o & 1) * 1024 + 8 (o >> 1) + cB of rank g
    double2* __restrict__ yq = a.y + (int64_t)g * kW_YP + (int64_t)kB * kW_YS + (o & 1) * (kW_N2 / 2) + 8 * (o >> 1) + cB;
#pragma unroll
    for (int mm = 0; mm < 8; ++mm) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double2 yv = cmul(v[4 * mm + j], t[j]);
        double2* dst = yq + (int64_t)(4 * mm + j) * 32 * kW_YS;
        *dst = yv;
      }
      if (mm < 7) {
#pragma unroll
        for (int j = 0; j < 4; ++j) t[j] = cmul(t[j], stB);
      }
    }
  }
  tl_mark(a, 1, 2);
}

// Row pass: a CTA is two independent halves of 4 warps (named barriers 1 and 2), each owning one
// row pair (k1, N1-k1) at a time with warps (rho, h) = (row, even/odd samples). Per rank a warp
// loads its 1024 samples (contiguous: the permuted Y layout) and transforms them to E (h = 0) or
// O (h = 1); the half then forms X[q'] = E + W_2048^q' O, X[q' + 1024] = E - W_2048^q' O of both
// rows, the conjugate-pair split and w*A*B, accumulated over ranks in registers.
// LAST (the launch of the last rank group): the half then runs the inverse row transform of its
// accumulated Hermitian row k1 (2 warps, radix-2 DIF + 1024-point inverse FFTs) and the inverse
// four-step twiddle, writing G in place of the accumulator row.
// The shared-memory traffic of a transform is spread through its arithmetic instead of issued in
// bursts: the exchange stores follow each step-A twiddle product, and the results are parked where
// the thread itself read its step-B inputs (xs[lane * 33 + k] holds X[lane + 32 k]: no warp barrier
// between step B and the park; the product phase reads bin q at (q & 31) * 33 + (q >> 5),
// conflict-free since consecutive lanes are 33 entries apart); rank weights are staged in shared
// memory once per CTA (row pass 180 -> 174 us at config 4).
// Launched with 2 row pairs per half (grid = ceil(513 / 4) = 129 CTAs at N1 = 1024) so the SMs
// left over run the non-birth part D concurrently (k_dvec, programmatic dependent launch).
// The row kernel tests its experiment bits at run time (a.dbg is 0 unless an AGK_EXPERIMENTS
// build set it from AGK_DBG: the production library never reads the environment): folded away
// at compile time, ptxas allocates this 255-register kernel worse (36 instead of 8 bytes of
// spills, measured with -Xptxas -v).
#define ROW_XDBG(a, bits) ((((a).dbg) & (bits)) != 0)
template <bool LAST>
__global__ void __launch_bounds__(256, 1) k_rowd(RhsArgs a, int g0, int gcount, int first) {
  extern __shared__ double2 smem[];
  double2* X = smem;               // 8 regions: per half E1, O1 (row k1), E2, O2 (row N1-k1)
  double2* tw = X + 8 * kXR;       // W_1024^{l k1}, [k1][l]
  double2* twh = tw + 1024;        // W_2048^j, j < 1024
  __shared__ double2 tkk[8][32];
  __shared__ double wq_s[32];
  tl_mark_rt(a, 2, 0);
  pdl_entry();
  tl_mark_rt(a, 2, 1);
  if (a.skip && *a.skip) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, hf = w >> 2, hw = w & 3, rho = hw >> 1,
            h = hw & 1, ht = tid & 127, bar = 1 + hf;
  const int n1 = a.n1;
  const int64_t P = (int64_t)kW_N1 * kW_N2;
  const int nrows = n1 / 2 + 1;
  for (int i = tid; i < 1024; i += blockDim.x) {
    tw[i] = __ldg(a.tw32 + i);
    twh[i] = __ldg(a.tw2048h + i);
  }
  if (tid < 32 && tid < gcount) wq_s[tid] = 0.25 * a.uniq_weight[g0 + tid];
  __syncthreads();
  double2* Xh = X + hf * 4 * kXR;
  double2* Xw = X + w * kXR;
  for (int k1 = 2 * blockIdx.x + hf; k1 < nrows; k1 += 2 * gridDim.x) {
    const int row = rho == 0 ? k1 : (n1 - k1) & (n1 - 1);
    const double2* __restrict__ rsrc = a.y + (int64_t)row * kW_YS + h * (kW_N2 / 2);
    double2 acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = first ? czero() : a.acc[(int64_t)k1 * kW_N2 + ht + 128 * j];
    double2 v[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) v[r] = rsrc[lane + 32 * r];
    double2 tw1[8], tw2[8];
    const double2 wb1 = twh[ht];
    const double2 wb2 = k1 == 0 ? make_double2(wb1.x, -wb1.y) : make_double2(twh[ht + 1].x, -twh[ht + 1].y);
    auto tw_of = [&](int j, double2& t1w, double2& t2w) {
      t1w = mul_w16<-1>(wb1, j);
      t2w = (k1 == 0 && ht == 0 && j == 0) ? make_double2(1.0, 0.0) : mul_w16<+1>(wb2, j);
    };
    if constexpr (LAST) {
#pragma unroll
      for (int j = 0; j < 8; ++j) tw_of(j, tw1[j], tw2[j]);
    }
    // parked bin q of a region: (q & 31) * 33 + (q >> 5). This thread's bins q' = ht + 128 j and
    // their partners m = 1023 - q' (row 0: (1024 - q') & 1023) are 4 entries apart per j.
    const int pl = ht & 31, pc = ht >> 5;
    const double2* pq = Xh + pl * 33 + pc;
    const double2* pm = Xh + 2 * kXR + (k1 != 0 ? (31 - pl) * 33 + 31 - pc : (pl ? (32 - pl) * 33 + 31 - pc : 32 - pc));
    const double2* pm0 = (k1 == 0 && ht == 0) ? Xh + 2 * kXR : pm;
    for (int g = 0; g < gcount; ++g) {
      const double wq = wq_s[g];  // (the plan caps a group at 16 ranks)
      if (lane == 0 && !ROW_XDBG(a, 128)) {
        int gn = g + AGK_PFDIST(a), k1n = k1;
        if (gn >= gcount) {
          gn -= gcount;
          k1n += 2 * gridDim.x;
        }
        if (k1n < nrows) {
          const int rown = rho == 0 ? k1n : (n1 - k1n) & (n1 - 1);
          prefetch_l2(a.y + (int64_t)gn * kW_YP + (int64_t)rown * kW_YS + h * (kW_N2 / 2), 1024 * sizeof(double2));
        }
      }
      if (!ROW_XDBG(a, 16)) {
        Dft<32, -1>::run(v);
        twiddle_a_rec_store<-1>(v, tw, lane, [&](int k, double2 x) { Xw[k * 33 + lane] = x; });
        __syncwarp();
#pragma unroll
        for (int l = 0; l < 32; ++l) v[l] = Xw[lane * 33 + l];
        Dft<32, -1>::run(v);
#pragma unroll
        for (int k = 0; k < 32; ++k) Xw[lane * 33 + k] = v[k];
      }
      __syncwarp();  // keeps the next rank's loads (32 live registers) behind the transform
      if (g + 1 < gcount && !ROW_XDBG(a, 64)) {
        const double2* __restrict__ src = rsrc + (int64_t)(g + 1) * kW_YP;
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = src[lane + 32 * r];
      }
      bar_sync(bar, 128);
      if (!ROW_XDBG(a, 32))
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        // bin q' = ht + 128 j sits at pq[4 j]; its partner bin at pm[-4 j] (pm0: row 0's bin 0)
        const double2 e1 = pq[4 * j], o1 = pq[kXR + 4 * j];
        const double2* pmj = j == 0 ? pm0 : pm;
        const double2 e2 = pmj[-4 * j], o2 = pmj[kXR - 4 * j];
        double2 t1w, t2w;
        if constexpr (LAST) {
          t1w = tw1[j];
          t2w = tw2[j];
        } else {
          tw_of(j, t1w, t2w);
        }
        const double2 t1 = cmul(o1, t1w), t2 = cmul(o2, t2w);
        const double2 xa = cadd(e1, t1), xb = csub(e1, t1);
        const double2 pa = cadd(e2, t2), pb = csub(e2, t2);
        split_product_acc4(acc[j], wq, xa, pa);
        split_product_acc4(acc[j + 8], wq, xb, pb);
      }
      bar_sync(bar, 128);
    }
    if constexpr (!LAST) {
#pragma unroll
      for (int j = 0; j < 16; ++j) a.acc[(int64_t)k1 * kW_N2 + ht + 128 * j] = acc[j];
    } else {
      double2* Ar = Xh + 2 * kXR;  // 2120 >= 2048 contiguous entries
#pragma unroll
      for (int j = 0; j < 16; ++j) Ar[ht + 128 * j] = acc[j];
      bar_sync(bar, 128);
      if (rho == 0) {
        double2 v[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          const double2 lo = Ar[lane + 32 * r], hi = Ar[1024 + lane + 32 * r];
          v[r] = h == 0 ? cadd(lo, hi) : cmul(csub(lo, hi), cconj(twh[lane + 32 * r]));
        }
        warp_fft1024<+1, false>(v, Xw, tw, lane);
        const double2 base = tw_p<+1>(a.twp, (uint32_t)((2 * lane + h) * k1));
        tkk[w][lane] = tw_p<+1>(a.twp, (uint32_t)((64 * k1 * lane) & (P - 1)));
        __syncwarp();
        double2* __restrict__ gr = a.acc + (int64_t)k1 * kW_N2;
#pragma unroll
        for (int k = 0; k < 32; ++k) gr[2 * (lane + 32 * k) + h] = cmul(v[k], cmul(base, tkk[w][k]));
      }
      bar_sync(bar, 128);  // the regions are reused by the next row pair
    }
  }
  tl_mark_rt(a, 2, 2);
}

// The non-birth part of S for every size: -n_s sum_a U_sa w_a [+ shattering] [+ sources]
// (rhs.cpp:24-46, 162-168, 170-210, 227-229). A pure stream over U (R x M) at full occupancy;
// it runs on the SMs the last row launch leaves free, beside the row transforms.
__global__ void __launch_bounds__(256, 2) k_dvec(RhsArgs a) {
  extern __shared__ double dsm[];  // 4 rf moment totals, 2 r gains, r + 2 scalars
  tl_mark(a, 3, 0);
  tl_mark(a, 3, 1);
  if (!(a.skip && *a.skip) && !AGK_XDBG(a, 256)) {
    const double* __restrict__ n = a.n.get();
    const int fl = a.flags & ~T_BIRTH;
    const bool rs = (a.flags & (T_DEATH | T_DEATH_POS | T_SHATTER)) != 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const bool even = (a.m & 1) == 0;
    // Even m: KU x 2 sizes per thread per batch (16-byte loads); the U^T rows of the first RB
    // ranks and the n pairs of a batch are issued together (they do not depend on w), the first
    // batch before the scalars are final and each next batch before the current one is stored,
    // so a batch costs one round trip for r <= RB.
    constexpr int KU = 2, RB = 4;
    const int64_t np = a.m / 2;
    const int64_t pbeg = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double2 nv[KU], u[RB][KU];
    auto issue = [&](int64_t p0) {
#pragma unroll
      for (int k = 0; k < KU; ++k) {
        const int64_t pk = 2 * (p0 + k * stride < np ? p0 + k * stride : np - 1);  // clamped
        nv[k] = *reinterpret_cast<const double2*>(n + pk);
#pragma unroll
        for (int q = 0; q < RB; ++q)
          u[q][k] = (rs && q < a.r) ? __ldg(reinterpret_cast<const double2*>(a.ut + (int64_t)q * a.m + pk))
                                     : make_double2(0.0, 0.0);
      }
    };
    // w_a and the shattering gains from the column pass' moment partials, reduced by every CTA
    // in the same fixed order (bitwise identical copies); the first batch goes out between the
    // (register-heavy) partial sums and the (latency-bound) finalisation
    double* tot = dsm;
    double* sh = tot + 4 * a.rf;
    double* scal = sh + 2 * a.r;  // w_a, pair gain, monomer gain
    reduce_partials_wide(a, a.nblk_colfwd, tot);
    if (even && pbeg < np) issue(pbeg);
    __syncthreads();
    finalize_scalars_to(a, tot, n[0], sh, scal);
    __syncthreads();
    if (blockIdx.x == 0)
      for (int i = threadIdx.x; i < a.r + 2; i += blockDim.x) a.scalars[i] = scal[i];
    if (even) {
      for (int64_t p0 = pbeg; p0 < np; p0 += KU * stride) {
        double r[KU][2];
#pragma unroll
        for (int k = 0; k < KU; ++k) r[k][0] = r[k][1] = 0.0;
        if (rs) {
          // each size's row sum in rank order (rhs.cpp:24-46): ranks < RB from the batch
          // registers, the rest RB at a time
#pragma unroll
          for (int q = 0; q < RB; ++q) {
            if (q < a.r) {
              const double w = scal[q];
#pragma unroll
              for (int k = 0; k < KU; ++k) {
                r[k][0] += u[q][k].x * w;
                r[k][1] += u[q][k].y * w;
              }
            }
          }
          for (int ra = RB; ra < a.r; ra += RB) {  // (the batch registers are free again)
#pragma unroll
            for (int q = 0; q < RB; ++q)
#pragma unroll
              for (int k = 0; k < KU; ++k) {
                const int64_t pk = 2 * (p0 + k * stride < np ? p0 + k * stride : np - 1);
                u[q][k] = ra + q < a.r ? __ldg(reinterpret_cast<const double2*>(a.ut + (int64_t)(ra + q) * a.m + pk))
                                       : make_double2(0.0, 0.0);
              }
#pragma unroll
            for (int q = 0; q < RB; ++q) {
              if (ra + q < a.r) {
                const double w = scal[ra + q];
#pragma unroll
                for (int k = 0; k < KU; ++k) {
                  r[k][0] += u[q][k].x * w;
                  r[k][1] += u[q][k].y * w;
                }
              }
            }
          }
        }
        double2 nk[KU];
#pragma unroll
        for (int k = 0; k < KU; ++k) nk[k] = nv[k];
        if (p0 + KU * stride < np) issue(p0 + KU * stride);  // the next batch's loads go out now
#pragma unroll
        for (int k = 0; k < KU; ++k) {
          const int64_t p = p0 + k * stride;
          if (p < np) {
            const int64_t s = 2 * p;
            a.dvec[s] = s == 0 ? dvalue0(a, fl, scal, nk[k].x) : dvalue(a, fl, nk[k].x, s, r[k][0]);
            a.dvec[s + 1] = dvalue(a, fl, nk[k].y, s + 1, r[k][1]);
          }
        }
      }
    } else {
      for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < a.m; s += stride) {
        double rowsum = 0.0;
        if (rs)
          for (int ra = 0; ra < a.r; ++ra) rowsum += __ldg(a.ut + (int64_t)ra * a.m + s) * scal[ra];
        a.dvec[s] = s == 0 ? dvalue0(a, fl, scal, n[0]) : dvalue(a, fl, n[s], s, rowsum);
      }
    }
  }
  tl_mark(a, 5, 2);  // D done (before the wait for the row grid)
  // launched as a programmatic dependent of the row kernel: do not complete before it does, so
  // the launches after this one see the row results (no-op for an ordinary launch)
  pdl_entry();
  tl_mark(a, 3, 2);
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
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // constant twiddle table: staged while the previous kernel drains (programmatic dependent launch)
  tl_mark(a, 4, 0);
  for (int i = tid; i < 1024; i += blockDim.x) tw[i] = __ldg(a.tw32 + i);
  pdl_entry();
  tl_mark(a, 4, 1);
  if (a.skip && *a.skip) return;
  const double2* __restrict__ G = a.acc;
  const double scale = ldexp(0.5, -a.log2p);
  const bool birth = (a.flags & T_BIRTH) != 0;
  double* tile = reinterpret_cast<double*>(X);  // [512][2 kCW + 1] birth values, after the FFTs
  constexpr int TS = 2 * kCW + 1;
  for (int grp = blockIdx.x; grp < kW_N2 / (2 * kCW); grp += gridDim.x) {
    const int col0 = grp * kCW * 2;
    __syncthreads();  // previous group's tile reads done
    // G tile and the D values of this output tile, all in flight at once (cp.async, two groups:
    // the transforms wait for G only, the D values land while they run)
    for (int idx = tid; idx < GROWS * 2 * kCW; idx += kCW * 32) {
      const int row = idx / (2 * kCW), c = idx % (2 * kCW);
      cp_async16(X + row * GS + c, G + (int64_t)row * kW_N2 + col0 + c);
    }
    cp_async_commit();
    for (int idx = tid; idx < kW_H * 2 * kCW; idx += kCW * 32) {
      const int nn1 = idx / (2 * kCW), c = idx % (2 * kCW);
      const int64_t jo = (int64_t)nn1 * kW_N2 + col0 + c + 1;
      cp_async8(dv + idx, a.dvec + (jo < a.m ? jo : 0), jo < a.m);
    }
    cp_async_commit();
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
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
    cp_async_wait_all();  // this thread's D values
    __syncthreads();  // all exchanges done: the regions become the birth tile; every D value landed
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
  tl_mark(a, 4, 2);
}

static size_t smem_colx() { return (size_t)(8 * kW_N1 + 8 * kW_H + 1024 + 4 * 256) * sizeof(double2); }
static size_t smem_rowd() { return (size_t)(8 * kXR + 2048) * sizeof(double2); }
template <int CW>
static size_t smem_colinvw_t() {
  const size_t tile = (size_t)(kW_N1 / 2 + 1) * (2 * CW + 1);
  return ((tile > (size_t)CW * kXR ? tile : (size_t)CW * kXR) + 1024 + (size_t)kW_H * CW) * sizeof(double2);
}
static size_t smem_colinvw4() { return smem_colinvw_t<4>(); }
static size_t smem_colinvw() {
  constexpr int CW = 8;
  const size_t tile = (size_t)(kW_N1 / 2 + 1) * (2 * CW + 1);
  return ((tile > (size_t)CW * kXR ? tile : (size_t)CW * kXR) + 1024 + (size_t)kW_H * CW) * sizeof(double2);
}

cudaError_t rhs_w_set_smem_limits() {
  cudaError_t e;
#define SET(fn, bytes) \
  if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(bytes))) != cudaSuccess) return e;
  SET(k_colx, smem_colx());
  SET(k_rowd<false>, smem_rowd());
  SET(k_rowd<true>, smem_rowd());
  SET(k_colinvw<8>, smem_colinvw());
  SET(k_colinvw<4>, smem_colinvw4());
#undef SET
  return cudaSuccess;
}

// One RHS: transpose of n | per rank group, column pass | row pass (the last one also runs the
// inverse row transform, with D computed beside it on the SMs the row grid leaves free) | inverse
// column pass with the epilogue. 5 launches for <= 16 unique ranks (the plan's `launches`), each a
// programmatic dependent of the one before (pdl_entry in every kernel; off under timing marks).
cudaError_t rhs_w_launch(const RhsPlan& p, const RhsArgs& a0, cudaStream_t s, void (*mark)(void*, int, cudaStream_t),
                         void* mk) {
  RhsArgs first = a0;
  first.dbg = knob("AGK_DBG", 0);  // experiment switches (tools/ab.sh): AGK_EXPERIMENTS builds only
  first.pfd = knob("AGK_PFD", 1);  // L2 prefetch distance (items)
  // a fused RK stage is formed by the transpose; the later kernels read the stored stage vector
  RhsArgs a = first;
  if (a.st.on) {
    a.st.on = 0;
    a.n = VecRef{a.stg_out, nullptr, 0};
  }
  const int nsm = p.nsm > 0 ? p.nsm : 148;
  const bool pdl = !mark && pdl_enabled();
  AGK_CK(launch_k(k_transpose_n, (kW_H / 64) * (kW_N2 / 64), 256, 0, s, pdl && (pdl_mask() & 1), first));
  if (mark) mark(mk, K_TRANSPOSE, s);
  a.nblk_colfwd = kW_N2 / 8;
  const int rows = kW_N1 / 2 + 1;
  // 2 row pairs per half; the SMs left over run D
  const int per = (rows + 2 * nsm - 1) / (2 * nsm);
  const int rgrid = (rows + 2 * per - 1) / (2 * per);
  for (int g0 = 0; g0 < a.rf; g0 += p.gsize) {
    const int gc = (a.rf - g0) < p.gsize ? (a.rf - g0) : p.gsize;
    const bool last = g0 + gc >= a.rf;
    const int items = (kW_N2 / 8) * gc;
    const int cgrid = items < nsm ? items : nsm;
    AGK_CK(launch_k(k_colx, cgrid, 256, smem_colx(), s, pdl && (pdl_mask() & 2), a, g0, gc));
    if (mark) mark(mk, K_COL_FWD, s);
    if (!last) {
      AGK_CK(launch_k(k_rowd<false>, rgrid, 256, smem_rowd(), s, pdl, a, g0, gc, (int)(g0 == 0)));
      if (mark) mark(mk, K_ROW, s);
      continue;
    }
    AGK_CK(launch_k(k_rowd<true>, rgrid, 256, smem_rowd(), s, pdl && (pdl_mask() & 4), a, g0, gc, (int)(g0 == 0)));
    if (mark) mark(mk, K_ROW, s);
    // D (k_dvec) either beside the row pass, on the SMs its grid leaves free (it starts once every
    // row CTA passed its wait, i.e. the column pass is complete, and waits for the row grid before
    // it exits), or after it on every SM. Beside wins when the row pass outlasts D on the free SMs:
    // measured at M = 2^20 (tools/timeline.py), row ~ 20 + 9.6 rf us and D on 19 SMs ~ 65 + 4 r us.
    const int free = nsm - rgrid;
    const size_t dsm = (size_t)(4 * a.rf + 3 * a.r + 2) * sizeof(double);
    const int dmode = knob("AGK_DVEC_MODE", 0);  // experiments: 1 beside, 2 after (0: the measured rule)
    if ((dmode == 1 || (dmode == 0 && 9.6 * a.rf >= 45.0 + 4.0 * a.r)) && free >= 8) {
      // every k_dvec CTA must be resident from the start: a CTA that finished early would otherwise
      // hold its SM slot in the final wait for the row grid, and the rest of D would run after it
      AGK_CK(launch_k(k_dvec, 2 * free, 256, dsm, s, !mark, a));
    } else {
      AGK_CK(launch_k(k_dvec, 2 * nsm, 256, dsm, s, false, a));
    }
    if (mark) mark(mk, K_DVEC, s);
  }
  static const bool civ4 = knob("AGK_CIV", 8) == 4;
  if (civ4) {
    AGK_CK(launch_k(k_colinvw<4>, kW_N2 / 8, 128, smem_colinvw4(), s, pdl, a));
  } else {
    AGK_CK(launch_k(k_colinvw<8>, kW_N2 / 16, 256, smem_colinvw(), s, pdl && (pdl_mask() & 8), a));
  }
  if (mark) mark(mk, K_COL_INV, s);
  return cudaGetLastError();
}

unsigned long long* timeline_ptr() {
  static unsigned long long* p = nullptr;
  if (!p) cudaGetSymbolAddress(reinterpret_cast<void**>(&p), g_timeline);
  return p;
}

}  // namespace agk

// diagnostics only (tools/timeline.py): reset (reset != 0) or read the AGK_DBG & 512 timeline
extern "C" int agk_dbg_timeline(unsigned long long* out, int reset) {
  unsigned long long h[8][3];
  if (reset) {
    for (int k = 0; k < 8; ++k) h[k][0] = h[k][1] = ~0ull, h[k][2] = 0;
    return (int)cudaMemcpyToSymbol(agk::g_timeline, h, sizeof(h));
  }
  const cudaError_t e = cudaMemcpyFromSymbol(h, agk::g_timeline, sizeof(h));
  for (int k = 0; k < 24; ++k) out[k] = (&h[0][0])[k];
  return (int)e;
}
