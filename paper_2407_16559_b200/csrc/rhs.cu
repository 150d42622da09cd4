// rhs.cu — B200 kernels for the low-rank Smoluchowski right-hand side (fp64, sm_100a).
//
// Replaces eval_rhs / birth_term / death_term / shattering_terms (reference src/rhs.cpp:24-235).
// The reference does, per unique rank, one packed length-P complex FFT of z = U_a n + i V_a n,
// splits the two real spectra, accumulates w * A_k B_k, then one inverse FFT (rhs.cpp:126-149),
// and separately R dot products + an M x R pass for the death term (rhs.cpp:24-36).
//
// Here the same algebra runs as
//   small path (P = next_pow2(2m) <= 8192): ONE CTA does everything on-chip (k_small);
//   four-step path (P = N1 * N2 >= 2^14), per group of unique ranks:
//     k_col_fwd : fused load of U_a∘n and V_a∘n (zero padding never materialised), N1-point
//                 column FFTs in registers/smem, four-step twiddle, moment partials
//                 (w_a and the shattering sums) -> intermediate Y (L2 resident per group)
//     k_row     : row FFTs of rows k1 and N1-k1 together, conjugate-pair split, w*A*B summed
//                 over the group's ranks in registers; the last group also does the inverse
//                 row FFT of the Hermitian half (rows 0..N1/2) and the inverse twiddle -> G
//   then k_col_inv : two real columns per complex inverse FFT (G is Hermitian in k1), 1/P and
//                 the 1/2 of the birth term, death (n_s * sum_a U_sa w_a), sources and
//                 shattering fused into the epilogue -> out.
// All reductions are fixed-order (no floating-point atomics): results are bitwise
// reproducible run to run.
#include <cstdio>

#include "internal.h"
#include "rhs_common.cuh"

namespace agk {


// ------------------------------------------------------------------ shared device helpers

// ------------------------------------------------------------------ small path: one CTA

template <int P>
struct SmallCfg {
  static constexpr int E = P >= 16 ? 16 : P;
  static constexpr int T = P / E;
  static constexpr int NT = T < 128 ? 128 : T;
  using PL = FftPlan<P, E>;
  static constexpr size_t SMEM_BYTES = (size_t)(PL::SMEM + PL::TWS) * sizeof(double2);
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
};

template <int P>
__global__ void __launch_bounds__(SmallCfg<P>::NT) k_small(RhsArgs a) {
  pdl_entry();
  using CF = SmallCfg<P>;
  constexpr int E = CF::E, T = CF::T, NT = CF::NT;
  using PL = typename CF::PL;
  constexpr int H = P / 2 + 1;
  constexpr int QA = (H + NT - 1) / NT;
  extern __shared__ double2 zs[];
  double2* smtw = zs + PL::SMEM;
  __shared__ double red[(NT / 32) * 4];
  if (a.skip && *a.skip) return;
  load_twiddles<P, E>(smtw, a.tw_small);
  const int tid = threadIdx.x;
  const int64_t m = a.m;
  if (a.st.on) {  // fused RK stage: form the stage vector once (visible to the CTA after the barrier)
    const double* x = a.n.get();
    const double t = a.st.tau_mul * *a.st.tau;
    for (int64_t i = tid; i < m; i += NT) a.stg_out[i] = stage_at(a.st, t, x[i], i);
    __syncthreads();
  }
  const double* __restrict__ n = a.st.on ? a.stg_out : a.n.get();
  const bool act = tid < T;
  double2 acc[QA];
#pragma unroll
  for (int q = 0; q < QA; ++q) acc[q] = czero();

  for (int ub = 0; ub < a.rf; ++ub) {
    const int ra = a.uniq_rank[ub];
    const double* __restrict__ ut = a.ut + (int64_t)ra * m;
    const double* __restrict__ vv = a.v + (int64_t)ra * m;
    const double wt = a.uniq_weight[ub];
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = tid; i < P; i += NT) {
      double2 z = czero();
      if (i < m) {
        const double ni = n[i];
        z = make_double2(ut[i] * ni, vv[i] * ni);
        if (i >= 1) {
          const double sz = (double)(i + 1);
          s[0] += z.x;
          s[1] += sz * z.x;
          s[2] += z.y;
          s[3] += sz * z.y;
        }
      }
      zs[pad_idx<PL::PADS>(i)] = z;
    }
    block_sum<4>(s, red);
    if (tid == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) a.partials[ub * 4 + q] = s[q];
    }
    double2 v[E];
    if (act) {
#pragma unroll
      for (int r = 0; r < E; ++r) v[r] = zs[pad_idx<PL::PADS>(tid + r * T)];
    }
    __syncthreads();
    block_fft<P, E, -1, false>(v, zs, tid, smtw, act);
    if (act) {
#pragma unroll
      for (int r = 0; r < E; ++r) zs[pad_idx<PL::PADS>(tid + r * T)] = v[r];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < QA; ++q) {
      const int k = tid + q * NT;
      if (k < H) {
        const double2 pr = split_product(zs[pad_idx<PL::PADS>(k)], zs[pad_idx<PL::PADS>((P - k) & (P - 1))]);
        acc[q].x += wt * pr.x;
        acc[q].y += wt * pr.y;
      }
    }
    __syncthreads();
  }
  // Hermitian spectrum of the real convolution, then one inverse transform
#pragma unroll
  for (int q = 0; q < QA; ++q) {
    const int k = tid + q * NT;
    if (k < H) {
      zs[pad_idx<PL::PADS>(k)] = acc[q];
      if (k > 0 && k < P / 2) zs[pad_idx<PL::PADS>(P - k)] = cconj(acc[q]);
    }
  }
  __syncthreads();
  double2 v[E];
  if (act) {
#pragma unroll
    for (int r = 0; r < E; ++r) v[r] = zs[pad_idx<PL::PADS>(tid + r * T)];
  }
  __syncthreads();
  block_fft<P, E, +1, false>(v, zs, tid, smtw, act);
  if (act) {
#pragma unroll
    for (int r = 0; r < E; ++r) zs[pad_idx<PL::PADS>(tid + r * T)] = v[r];
  }
  if (tid == 0) finalize_scalars(a, a.partials, n[0]);
  __syncthreads();
  const double scale = ldexp(0.5, -a.log2p);  // (1/P) of the inverse times the 1/2 of birth
  for (int64_t jo = tid; jo < m; jo += NT) {
    if (jo == 0) {
      a.out[0] = epilogue0(a, n);
    } else {
      a.out[jo] = epilogue(a, n, jo, scale * zs[pad_idx<PL::PADS>((int)jo - 1)].x);
    }
  }
}

// ------------------------------------------------------------------ four-step path

// Defaults (points per thread of the forward column, row and inverse column passes), measured per
// size (tools/gpu/mvar.sh, profiles/mvar_r02u.txt): 4 up to P = 2^16 (the latency-bound small sizes
// want more warps); 8 for the forward column and row passes at 2^17 <= P <= 2^20, whose 4-point
// transforms were bound by shared-memory traffic (five exchange passes per 512-point transform:
// 2.8 us of a 5 us phase, tools/timeline.py), with the inverse column pass at 2 (P = 2^17) or 4
// points (its epilogue wants the threads); 16 above.
template <int L, int E1_ = (L <= 16 ? 4 : (L <= 20 ? 8 : 16)), int E2_ = (L <= 16 ? 4 : (L <= 20 ? 8 : 16)),
          int C_ = (L <= 20 ? 4 : (L <= 21 ? 8 : 2)), int ROWMODE_ = 0,
          int E1I_ = (L <= 16 ? 4 : (L == 17 ? 2 : (L <= 20 ? 4 : E1_)))>
struct Cfg {
  static constexpr int E1I = E1I_;  // points per thread of the inverse column pass (its own choice)
  static constexpr int ROWMODE = ROWMODE_;  // 1: no staging, 2 CTAs/SM register budget
  static constexpr int N1 = 1 << (L / 2), N2 = 1 << (L - L / 2);
  static constexpr int E1 = E1_;
  static constexpr int E2 = E2_;
  static constexpr int C = C_;
  static constexpr int CP = C / 2 > 0 ? C / 2 : 1;
  static constexpr int T1 = N1 / E1, T2 = N2 / E2;
  using PL1 = FftPlan<N1, E1>;
  using PL2 = FftPlan<N2, E2>;
  using PL1I = FftPlan<N1, E1I>;
  static constexpr int R1 = PL1::template smem<kNoPad>();  // column team region (no padding)
  static constexpr int R1I = PL1I::template smem<kNoPad>();
  // + staging of the next rank's U, V (column kernel) / Y rows (row kernel)
  static constexpr size_t SM_COLFWD = (size_t)(C * R1 + PL1::TWS) * sizeof(double2) + (size_t)C * N1 * sizeof(double);
  static constexpr bool ROW_STAGE = ROWMODE == 0 && (2 * PL2::SMEM + PL2::TWS + 2 * N2) * 16 <= 232448;
  static constexpr int ROW_MINB = ROWMODE == 1 ? 2 : 1;
  static constexpr size_t SM_ROW = (size_t)(2 * PL2::SMEM + PL2::TWS + (ROW_STAGE ? 2 * N2 : 0)) * sizeof(double2);
  static constexpr size_t SM_COLINV = (size_t)(CP * R1I + PL1I::TWS) * sizeof(double2);
  static_assert(SM_COLFWD <= 232448 && SM_ROW <= 232448 && SM_COLINV <= 232448, "shared memory budget");
  static_assert(C * T1 >= 32 && 2 * T2 >= 32, "column-forward and row CTAs need full warps");
};

template <int N1, int E1, int C>
__global__ void __launch_bounds__(C*(N1 / E1)) k_col_fwd(RhsArgs a, int g0, int gcount) {
  using PL = FftPlan<N1, E1>;
  constexpr int T1 = N1 / E1, NT = C * T1, H = E1 / 2;
  constexpr int RG = PL::template smem<kNoPad>();
  extern __shared__ double2 smem[];
  double2* smtw = smem + C * RG;
  double* stage = reinterpret_cast<double*>(smtw + PL::TWS);  // [2][H][NT]: own elements only
  __shared__ double red[((NT + 31) / 32) * 4];
  const int tid = threadIdx.x, c = tid % C, j = tid / C;
  const int64_t n2 = (int64_t)blockIdx.x * C + c;
  const int64_t N2 = a.n2, m = a.m, P = (int64_t)N1 * N2;
  AGK_TL(a, 1, 0);
  // stage this thread's U_a, V_a elements of unique rank ub (zero-filled past m)
  auto prefetch = [&](int ub) {
    const int ra = a.uniq_rank[ub];
    const double* ut = a.ut + (int64_t)ra * m;
    const double* vv = a.v + (int64_t)ra * m;
#pragma unroll
    for (int r = 0; r < H; ++r) {
      const int64_t i = (int64_t)(j + r * T1) * N2 + n2;
      const bool ok = i < m;
      cp_async8(stage + r * NT + tid, ut + (ok ? i : 0), ok);
      cp_async8(stage + (H + r) * NT + tid, vv + (ok ? i : 0), ok);
    }
    cp_async_commit();
  };
  // immutable operands (U, V, tables) first: they overlap the predecessor's tail
  if (gcount > 0) prefetch(g0);
  load_twiddles<N1, E1>(smtw, a.tw_n1);
  const TwSeries<-1> tw0(a.twp, (uint32_t)(n2 * j), (uint32_t)(n2 * T1));  // four-step twiddles
  pdl_wait();  // dependents are triggered at the end (mid-size path: trigger late)
  AGK_TL(a, 1, 1);
  if (a.skip && *a.skip) {
    cp_async_wait_all();
    return;
  }
  const double* __restrict__ n = a.n.get();
  double nl[H];
  if (a.st.on) {
    // fused RK stage: n_i = x_i + tau sum_j a_j k_j[i] formed here (each i by one thread) and
    // stored for the row and inverse-column kernels
    const double t = a.st.tau_mul * *a.st.tau;
#pragma unroll
    for (int r = 0; r < H; ++r) {
      const int64_t i = (int64_t)(j + r * T1) * N2 + n2;
      nl[r] = i < m ? stage_at(a.st, t, n[i], i) : 0.0;
      if (i < m) a.stg_out[i] = nl[r];
    }
  } else {
#pragma unroll
    for (int r = 0; r < H; ++r) {
      const int64_t i = (int64_t)(j + r * T1) * N2 + n2;
      nl[r] = i < m ? n[i] : 0.0;
    }
  }
  double2* sm = smem + c * RG;
  for (int g = 0; g < gcount; ++g) {
    const int ub = g0 + g;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    double2 v[E1];
    cp_async_wait_all();
#pragma unroll
    for (int r = 0; r < H; ++r) {
      const int64_t i = (int64_t)(j + r * T1) * N2 + n2;
      const double x = stage[r * NT + tid] * nl[r], y = stage[(H + r) * NT + tid] * nl[r];
      v[r] = make_double2(x, y);
      if (i >= 1) {  // zero-filled past m: contributes nothing
        const double sz = (double)(i + 1);
        s[0] += x;
        s[1] += sz * x;
        s[2] += y;
        s[3] += sz * y;
      }
    }
    if (g + 1 < gcount) prefetch(ub + 1);  // overlaps this rank's transforms
#pragma unroll
    for (int r = H; r < E1; ++r) v[r] = czero();
    AGK_TL(a, 5, 0);
    AGK_TL(a, 5, 2);
    __syncthreads();  // twiddle tables ready / previous rank's smem reads done
    block_fft<N1, E1, -1, true, kNoPad>(v, sm, j, smtw);
    AGK_TL(a, 5, 1);
    AGK_TL(a, 6, 2);
    double2* __restrict__ yg = a.y + (int64_t)g * P;
    TwSeries<-1> tw = tw0;
#pragma unroll
    for (int r = 0; r < E1; ++r) {
      const int64_t k1 = j + r * T1;
      yg[k1 * N2 + n2] = cmul(v[r], tw.next());
    }
    block_sum<4>(s, red);
    if (tid == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) a.partials[((int64_t)ub * a.nblk_colfwd + blockIdx.x) * 4 + q] = s[q];
    }
  }
  AGK_TL(a, 1, 2);
  pdl_trigger();
}

template <int N2, int E2, bool STAGE, int MINB>
__global__ void __launch_bounds__(2 * (N2 / E2), MINB) k_row(RhsArgs a, int g0, int gcount, int first, int last) {
  using PL = FftPlan<N2, E2>;
  constexpr int T2 = N2 / E2, NT = 2 * T2, Q = E2 / 2;
  extern __shared__ double2 smem[];
  double2* smtw = smem + 2 * PL::SMEM;
  double2* stage = smtw + PL::TWS;  // [E2][NT]: this thread's elements of the next rank's row
  AGK_TL(a, 2, 0);
  load_twiddles<N2, E2>(smtw, a.tw_n2);  // immutable table: overlaps the predecessor's tail
  const int tid = threadIdx.x, team = tid / T2, j = tid % T2;
  const int n1 = a.n1;
  const int k1 = blockIdx.x;
  const TwSeries<+1> itw0(a.twp, (uint32_t)(j * k1), (uint32_t)(T2 * k1));  // inverse four-step twiddles
  pdl_wait();  // dependents are triggered at the end (mid-size path: trigger late)
  AGK_TL(a, 2, 1);
  if (a.skip && *a.skip) return;
  const int row = team == 0 ? k1 : (n1 - k1) & (n1 - 1);
  const int64_t P = (int64_t)n1 * N2;
  auto prefetch = [&](int g) {
    if constexpr (STAGE) {
      const double2* yr = a.y + (int64_t)g * P + (int64_t)row * N2;
#pragma unroll
      for (int r = 0; r < E2; ++r) cp_async16(stage + r * NT + tid, yr + j + r * T2);
      cp_async_commit();
    }
  };
  if (last && k1 == n1 / 2 + 1) {
    // the extra CTA of the last launch: w_a and the shattering gains from the column pass'
    // moment partials, beside the row transforms instead of ahead of one of them
    double* tot = a.scalars + a.r + 2;
    reduce_partials(a, a.nblk_colfwd, tot);  // (register-light: the row kernel's budget is tight)
    __syncthreads();
    if (tid == 0) finalize_scalars(a, tot, a.n.get()[0]);
    return;
  }
  if (gcount > 0) prefetch(0);

  double2 acc[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = first ? czero() : a.acc[(int64_t)k1 * N2 + tid + q * NT];

  double2* smt = smem + team * PL::SMEM;
  for (int g = 0; g < gcount; ++g) {
    const double wt = a.uniq_weight[g0 + g];
    double2 v[E2];
    if constexpr (STAGE) {
      cp_async_wait_all();
#pragma unroll
      for (int r = 0; r < E2; ++r) v[r] = stage[r * NT + tid];
      AGK_TL(a, 7, 0);
      if (g + 1 < gcount) prefetch(g + 1);
    } else {
      const double2* __restrict__ yr = a.y + (int64_t)g * P + (int64_t)row * N2;
#pragma unroll
      for (int r = 0; r < E2; ++r) v[r] = yr[j + r * T2];
    }
    __syncthreads();  // twiddle tables ready / previous rank's split reads done
    block_fft<N2, E2, -1, false>(v, smt, j, smtw);
#pragma unroll
    for (int r = 0; r < E2; ++r) smt[pad_idx<PL::PADS>(j + r * T2)] = v[r];
    __syncthreads();
    const double2* s0 = smem;
    const double2* s1 = (k1 == 0) ? smem : smem + PL::SMEM;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int k2 = tid + q * NT;
      const int pk = (k1 == 0) ? ((N2 - k2) & (N2 - 1)) : (N2 - 1 - k2);
      const double2 pr = split_product(s0[pad_idx<PL::PADS>(k2)], s1[pad_idx<PL::PADS>(pk)]);
      acc[q].x += wt * pr.x;
      acc[q].y += wt * pr.y;
    }
  }
  AGK_TL(a, 7, 1);
  AGK_TL(a, 7, 2);
  if (!last) {
#pragma unroll
    for (int q = 0; q < Q; ++q) a.acc[(int64_t)k1 * N2 + tid + q * NT] = acc[q];
    return;
  }
  // inverse row transform of the Hermitian half-row k1 (team 0), then the inverse twiddle
  __syncthreads();
#pragma unroll
  for (int q = 0; q < Q; ++q) smem[pad_idx<PL::PADS>(tid + q * NT)] = acc[q];
  __syncthreads();
  double2 u[E2];
  const bool act = team == 0;
  if (act) {
#pragma unroll
    for (int r = 0; r < E2; ++r) u[r] = smem[pad_idx<PL::PADS>(j + r * T2)];
  }
  __syncthreads();
  block_fft<N2, E2, +1, false>(u, smem, j, smtw, act);
  AGK_TL(a, 6, 0);
  if (act) {
    TwSeries<+1> tw = itw0;
#pragma unroll
    for (int r = 0; r < E2; ++r) {
      const int64_t c2 = j + r * T2;
      a.acc[(int64_t)k1 * N2 + c2] = cmul(u[r], tw.next());
    }
  }
  AGK_TL(a, 2, 2);
  pdl_trigger();
}

template <int N1, int E1, int CP>
__global__ void __launch_bounds__(CP*(N1 / E1)) k_col_inv(RhsArgs a) {
  using PL = FftPlan<N1, E1>;
  constexpr int T1 = N1 / E1;
  constexpr int RG = PL::template smem<kNoPad>();
  extern __shared__ double2 smem[];
  double2* smtw = smem + CP * RG;
  AGK_TL(a, 4, 0);
  load_twiddles<N1, E1>(smtw, a.tw_n1);  // immutable table: overlaps the predecessor's tail
  pdl_wait();  // dependents are triggered at the end (mid-size path: trigger late)
  AGK_TL(a, 4, 1);
  if (a.skip && *a.skip) return;
  const int tid = threadIdx.x, c = tid % CP, j = tid / CP;
  const int64_t N2 = a.n2, m = a.m;
  const int64_t col = (int64_t)blockIdx.x * 2 * CP + 2 * c;
  const double2* __restrict__ G = a.acc;
  double2 v[E1];
#pragma unroll
  for (int r = 0; r < E1; ++r) {
    const int k1 = j + r * T1;
    const bool refl = k1 > N1 / 2;
    const int64_t rowi = refl ? N1 - k1 : k1;
    double2 ga = G[rowi * N2 + col], gb = G[rowi * N2 + col + 1];
    if (refl) {
      ga = cconj(ga);
      gb = cconj(gb);
    }
    v[r] = make_double2(ga.x - gb.y, ga.y + gb.x);  // G_a + i G_b: two real outputs at once
  }
  // the epilogue's other inputs (n, the U rows of up to 4 ranks, w_a) do not depend on the
  // transform: their loads go out with G's and land while the FFT runs
  const double* __restrict__ n = a.n.get();
  const bool rs = (a.flags & (T_DEATH | T_DEATH_POS | T_SHATTER)) != 0;
  constexpr int NO = E1;  // outputs per thread: 2 per transform row n1 < N1/2
  constexpr int RK = E1 <= 4 ? 4 : (E1 <= 8 ? 2 : 0);  // ranks preloaded (register budget)
  double nn[NO], u[RK > 0 ? RK : 1][NO], w[RK > 0 ? RK : 1];
#pragma unroll
  for (int q = 0; q < NO; ++q) {
    const int64_t jo = (int64_t)(j + (q >> 1) * T1) * N2 + col + 1 + (q & 1);  // out index = conv index + 1
    const bool ok = rs && jo < m;
    nn[q] = ok ? n[jo] : 0.0;
#pragma unroll
    for (int k = 0; k < RK; ++k) u[k][q] = (ok && k < a.r) ? __ldg(a.ut + (int64_t)k * m + jo) : 0.0;
  }
#pragma unroll
  for (int k = 0; k < RK; ++k) w[k] = (rs && k < a.r) ? a.scalars[k] : 0.0;
  (void)w;
  __syncthreads();
  block_fft<N1, E1, +1, false, kNoPad>(v, smem + c * RG, j, smtw);
  const double scale = ldexp(0.5, -a.log2p);
#pragma unroll
  for (int q = 0; q < NO; ++q) {
    const int64_t jo = (int64_t)(j + (q >> 1) * T1) * N2 + col + 1 + (q & 1);
    if (jo < m) {
      double rowsum = 0.0;  // rank order, as rhs.cpp:24-46
      if (rs) {
#pragma unroll
        for (int k = 0; k < RK; ++k)
          if (k < a.r) rowsum += u[k][q] * w[k];
        for (int ra = RK; ra < a.r; ++ra) rowsum += __ldg(a.ut + (int64_t)ra * m + jo) * a.scalars[ra];
      }
      a.out[jo] = epilogue_rsn(a, nn[q], jo, scale * ((q & 1) ? v[q >> 1].y : v[q >> 1].x), rowsum);
    }
  }
  if (blockIdx.x == 0 && tid == 0) a.out[0] = epilogue0(a, n);
  AGK_TL(a, 4, 2);
  pdl_trigger();
}

// ------------------------------------------------------------------ injected fakes

__global__ void k_fake(int kind, double param, VecRef nref, double* out, int64_t m, const int* skip) {
  pdl_entry();
  if (skip && *skip) return;
  const double* n = nref.get();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    double o;
    switch (kind) {
      case AGK_RHS_DECAY: o = -n[i]; break;
      case AGK_RHS_STILL: o = 0.0; break;
      case AGK_RHS_DRAIN: o = i == 0 ? -param : 0.0; break;
      case AGK_RHS_BURST_INF: o = __longlong_as_double(0x7ff0000000000000LL); break;
      default: o = __longlong_as_double(0x7ff8000000000000LL); break;
    }
    out[i] = o;
  }
}

cudaError_t fake_rhs_launch(int kind, double param, VecRef n, double* out, int64_t m, const int* skip,
                            cudaStream_t s) {
  const int threads = 256;
  int blocks = (int)((m + threads - 1) / threads);
  if (blocks > 4 * 148) blocks = 4 * 148;
  AGK_CK(launch_k(k_fake, blocks, threads, 0, s, pdl_enabled(), kind, param, n, out, m, skip));
  return cudaGetLastError();
}

// ------------------------------------------------------------------ host-side dispatch

static int ilog2_host(int64_t x) {
  int l = 0;
  while (((int64_t)1 << l) < x) ++l;
  return l;
}

void rhs_make_plan(int64_t m, int rf, RhsPlan* p) {
  int64_t P = 1;
  while (P < 2 * m) P <<= 1;
  p->log2p = ilog2_host(P);
  p->small = P <= 4096;
  p->n1 = 1 << (p->log2p / 2);
  p->n2 = 1 << (p->log2p - p->log2p / 2);
  const int L = p->log2p;
  p->c = L <= 20 ? 4 : (L <= 21 ? 8 : 2);
  p->cp = p->c / 2 > 0 ? p->c / 2 : 1;
  // Ranks per group: all unique ranks in one column/row launch pair (measured fastest at
  // M = 2^20, R = 16: the per-group intermediate then streams through HBM, but the launches and
  // the accumulator round trips of smaller groups cost more), capped at 1 GiB of intermediate.
  int g = (int)((1ll << 30) / (16 * P));
  g = knob("AGK_RANK_GROUP", g);
  if (g < 1) g = 1;
  if (g > rf) g = rf;
  const bool fast = L == 21 && knob("AGK_FAST", 1) != 0;
  if (fast && g > 16) g = 16;  // warp path: <= 16 rank slots
  p->gsize = g;
  const int ngroups = (rf + g - 1) / g;
  p->fast = fast;
  p->launches = p->small ? 1 : 2 * ngroups + 1 + (p->fast ? 2 : 0);  // fast: + transpose, dvec
  p->nsm = 148;
  p->dense = 0;
}

size_t rhs_y_elems(const RhsPlan& p) {
  // rows padded by 8 entries (rhs_w.cu kW_YPAD; the other paths use the unpadded prefix)
  return p.small ? 1 : (size_t)p.gsize * p.n1 * (p.n2 + 8);
}
size_t rhs_acc_elems(const RhsPlan& p) { return p.small ? 1 : (size_t)(p.n1 / 2 + 1) * p.n2; }
size_t rhs_partial_elems(const RhsPlan& p, int rf) {
  const size_t nblk = p.small ? 1 : (size_t)p.n2;  // any column-block width >= 2, or one block per column
  return (size_t)rf * nblk * 4;
}

// Optional per-launch event markers (bench.py's per-kernel roofline): after each kernel the
// launcher records marks->ev[marks->n++] and tags it with the kernel class.
struct Marks {
  cudaEvent_t* ev;
  int* cls;
  int cap, n;
};
static void mark(Marks* mk, int cls, cudaStream_t s) {
  if (mk && mk->n < mk->cap) {
    cudaEventRecord(mk->ev[mk->n], s);
    mk->cls[mk->n++] = cls;
  }
}
static void mark_cb(void* mk, int cls, cudaStream_t s) { mark(static_cast<Marks*>(mk), cls, s); }

#ifdef AGK_EXPERIMENTS
int knob(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
#endif

bool pdl_enabled() {
  static const bool on = knob("AGK_PDL", 1) != 0;
  return on;
}
int pdl_mask() {
  // measured per edge (tools/gpu/pdl.sh, profiles/pdl_r02i.txt): on for the inverse column pass (8),
  // the RK-trial chain (16) and the four-step path (32: P = 2^13; 64: the mid sizes, whose kernels
  // trigger their dependents at their end: -0.5 us at configs 2 and 3; triggered at entry the
  // early-placed dependent grid was slower); off for the transpose (1), for the column pass as the
  // transpose's dependent (2: with k_colx its early-placed CTAs cost 3.7 us per RHS at config 4 and
  // 6 us at config 5) and for the column -> row edge (4)
  static const int m = knob("AGK_PDLMASK", 8 | 16 | 32 | 64);
  return m;
}

// A fused RK stage (a.st.on): only the first kernel of an RHS forms the stage (and stores it to
// a.stg_out); the others read the stored vector.
static RhsArgs rest_args(const RhsArgs& a) {
  RhsArgs r = a;
  if (a.st.on) {
    r.st.on = 0;
    r.n = VecRef{a.stg_out, nullptr, 0};
  }
  return r;
}

template <int P>
static cudaError_t launch_small(const RhsArgs& a, cudaStream_t s, Marks* mk) {
  AGK_CK(launch_k(k_small<P>, 1, SmallCfg<P>::NT, SmallCfg<P>::SMEM_BYTES, s, !mk && pdl_enabled() && (pdl_mask() & 32), a));
  mark(mk, K_SMALL, s);
  return cudaGetLastError();
}

template <typename CF>
static cudaError_t launch_four_step_cf(const RhsPlan& p, const RhsArgs& a0, cudaStream_t s, Marks* mk) {
  RhsArgs first = a0;
  first.nblk_colfwd = CF::N2 / CF::C;
  if (knob("AGK_DBG", 0) & 512) first.tl = timeline_ptr();  // experiments build only
  const RhsArgs a = rest_args(first);
  const size_t sm1 = CF::SM_COLFWD, sm2 = CF::SM_ROW, sm3 = CF::SM_COLINV;
  const bool pdl = !mk && pdl_enabled() && (pdl_mask() & (CF::N1 * CF::N2 <= 8192 ? 64 : 32));
  for (int g0 = 0; g0 < a.rf; g0 += p.gsize) {
    const int gc = (a.rf - g0) < p.gsize ? (a.rf - g0) : p.gsize;
    AGK_CK(launch_k(k_col_fwd<CF::N1, CF::E1, CF::C>, CF::N2 / CF::C, CF::C * CF::T1, sm1, s, pdl,
                    g0 == 0 ? first : a, g0, gc));
    mark(mk, K_COL_FWD, s);
    AGK_CK(launch_k(k_row<CF::N2, CF::E2, CF::ROW_STAGE, CF::ROW_MINB>, CF::N1 / 2 + 1 + (g0 + gc >= a.rf ? 1 : 0),
                    2 * CF::T2, sm2, s, pdl, a, g0,
                    gc, (int)(g0 == 0), (int)(g0 + gc >= a.rf)));
    mark(mk, K_ROW, s);
  }
  AGK_CK(launch_k(k_col_inv<CF::N1, CF::E1I, CF::CP>, CF::N2 / (2 * CF::CP), CF::CP * (CF::N1 / CF::E1I), sm3, s, pdl, a));
  mark(mk, K_COL_INV, s);
  return cudaGetLastError();
}

// Tuning variants of the M = 2^20 shape (AGK_VARIANT), default 0.
#define AGK_L21_VARIANTS(X) \
  X(0, 16, 16, 8, 0) X(1, 16, 16, 4, 0) X(2, 8, 16, 8, 0) X(6, 16, 16, 8, 1) X(7, 16, 16, 4, 1)

#ifdef AGK_EXPERIMENTS
static int l21_variant() {
  static int v = -1;
  if (v < 0) {
    v = knob("AGK_VARIANT", 0);
  }
  return v;
}

// Mid-size variants (AGK_MVAR) for 2^14 <= P <= 2^20: fewer points per thread = more warps.
#define AGK_MID_VARIANTS(X, L) \
  X(1, L, 8, 8, 4, 8) X(2, L, 4, 4, 4, 4) X(3, L, 4, 8, 8, 4) X(4, L, 8, 8, 8, 8) X(5, L, 8, 8, 4, 4) X(6, L, 8, 4, 4, 4) \
  X(7, L, 4, 8, 4, 4) X(8, L, 8, 8, 8, 4) X(9, L, 8, 8, 2, 4) X(10, L, 8, 8, 4, 2) X(11, L, 8, 8, 4, 8)

static int mid_variant() {
  static int v = -1;
  if (v < 0) {
    v = knob("AGK_MVAR", 0);
  }
  return v;
}

#endif

template <int L>
static cudaError_t launch_four_step(const RhsPlan& p, const RhsArgs& a, cudaStream_t s, Marks* mk) {
#ifdef AGK_EXPERIMENTS
  if constexpr (L >= 14 && L <= 20) {
    switch (mid_variant()) {
#define AGK_M(id, LL, e1, e2, c, e1i) \
  case id: return launch_four_step_cf<Cfg<LL, e1, e2, c, 0, e1i>>(p, a, s, mk);
      AGK_MID_VARIANTS(AGK_M, L)
#undef AGK_M
      default: break;
    }
  }
  if constexpr (L == 21) {
    switch (l21_variant()) {
#define AGK_X(id, e1, e2, c, rm) \
  case id: return launch_four_step_cf<Cfg<21, e1, e2, c, rm>>(p, a, s, mk);
      AGK_L21_VARIANTS(AGK_X)
#undef AGK_X
      default: break;
    }
  }
#endif
  return launch_four_step_cf<Cfg<L>>(p, a, s, mk);
}

static cudaError_t rhs_launch_impl(const RhsPlan& p, const RhsArgs& a, cudaStream_t s, Marks* mk) {
  if (p.dense) {
    if (a.st.on) return cudaErrorInvalidValue;  // no fused stages on the dense path (rhs_stage_fusable)
    return rhs_dense_launch(p, a, s, mk ? mark_cb : nullptr, mk);
  }
  if (p.fast) return rhs_w_launch(p, a, s, mk ? mark_cb : nullptr, mk);
  switch (p.log2p) {
    case 2: return launch_small<4>(a, s, mk);
    case 3: return launch_small<8>(a, s, mk);
    case 4: return launch_small<16>(a, s, mk);
    case 5: return launch_small<32>(a, s, mk);
    case 6: return launch_small<64>(a, s, mk);
    case 7: return launch_small<128>(a, s, mk);
    case 8: return launch_small<256>(a, s, mk);
    case 9: return launch_small<512>(a, s, mk);
    case 10: return launch_small<1024>(a, s, mk);
    case 11: return launch_small<2048>(a, s, mk);
    case 12: return launch_small<4096>(a, s, mk);
    case 13: return launch_four_step<13>(p, a, s, mk);
    case 14: return launch_four_step<14>(p, a, s, mk);
    case 15: return launch_four_step<15>(p, a, s, mk);
    case 16: return launch_four_step<16>(p, a, s, mk);
    case 17: return launch_four_step<17>(p, a, s, mk);
    case 18: return launch_four_step<18>(p, a, s, mk);
    case 19: return launch_four_step<19>(p, a, s, mk);
    case 20: return launch_four_step<20>(p, a, s, mk);
    case 21: return launch_four_step<21>(p, a, s, mk);
    case 22: return launch_four_step<22>(p, a, s, mk);
    case 23: return launch_four_step<23>(p, a, s, mk);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t rhs_launch(const RhsPlan& p, const RhsArgs& a, cudaStream_t s) { return rhs_launch_impl(p, a, s, nullptr); }

cudaError_t rhs_launch_marked(const RhsPlan& p, const RhsArgs& a, cudaStream_t s, cudaEvent_t* ev, int* cls, int cap,
                              int* n) {
  Marks mk{ev, cls, cap, 0};
  cudaError_t e = rhs_launch_impl(p, a, s, &mk);
  *n = mk.n;
  return e;
}

template <int P>
static cudaError_t smem_small() {
  return cudaFuncSetAttribute(k_small<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SmallCfg<P>::SMEM_BYTES);
}

template <typename CF>
static cudaError_t smem_four_step_cf() {
  cudaError_t e;
  e = cudaFuncSetAttribute(k_col_fwd<CF::N1, CF::E1, CF::C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)CF::SM_COLFWD);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_row<CF::N2, CF::E2, CF::ROW_STAGE, CF::ROW_MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SM_ROW);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_col_inv<CF::N1, CF::E1I, CF::CP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)CF::SM_COLINV);
}

template <int L>
static cudaError_t smem_four_step() {
  cudaError_t e = smem_four_step_cf<Cfg<L>>();
  if (e != cudaSuccess) return e;
#ifdef AGK_EXPERIMENTS
  if constexpr (L == 21) {
#define AGK_X(id, e1, e2, c, rm) \
  if ((e = smem_four_step_cf<Cfg<21, e1, e2, c, rm>>()) != cudaSuccess) return e;
    AGK_L21_VARIANTS(AGK_X)
#undef AGK_X
  }
  if constexpr (L >= 14 && L <= 20) {
#define AGK_M(id, LL, e1, e2, c, e1i) \
  if ((e = smem_four_step_cf<Cfg<LL, e1, e2, c, 0, e1i>>()) != cudaSuccess) return e;
    AGK_MID_VARIANTS(AGK_M, L)
#undef AGK_M
  }
#endif
  return e;
}

cudaError_t rhs_set_smem_limits() {
  cudaError_t e = cudaSuccess;
#define AGK_TRY(x) \
  if ((e = (x)) != cudaSuccess) return e;
  AGK_TRY(smem_small<1024>());
  AGK_TRY(smem_small<2048>());
  AGK_TRY(smem_small<4096>());
  AGK_TRY(smem_four_step<13>());
  AGK_TRY(smem_four_step<14>());
  AGK_TRY(smem_four_step<15>());
  AGK_TRY(smem_four_step<16>());
  AGK_TRY(smem_four_step<17>());
  AGK_TRY(smem_four_step<18>());
  AGK_TRY(smem_four_step<19>());
  AGK_TRY(smem_four_step<20>());
  AGK_TRY(smem_four_step<21>());
  AGK_TRY(smem_four_step<22>());
  AGK_TRY(smem_four_step<23>());
  AGK_TRY(rhs_w_set_smem_limits());
#undef AGK_TRY
  return e;
}

}  // namespace agk
