// fft.cuh — fp64 complex FFT building blocks for sm_100a (SIMT DFMA pipe; no tensor cores).
//
// Replaces the reference's radix-2 plan (fft.cpp:64-137): instead of one length-P transform
// with a bit-reversal permutation, transforms are done by teams of threads on-chip:
//   * each thread holds E points in registers, E in {2,4,8,16};
//   * Stockham autosort passes (radix <= E) exchange through shared memory, so no
//     bit-reversal pass and every pass' global/shared traffic is unit-stride;
//   * radix-16/8/4/2 butterflies are straight-line code with compile-time twiddles; inter-pass
//     twiddles come from an accurate table (host long-double sincos) in global memory (L1).
// Layout contract of block_fft: thread j of a team of T = N/E threads holds x[j + r*T] in
// v[r] on entry and X[j + r*T] on exit (natural order, same distribution).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace agk {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 czero() { return make_double2(0.0, 0.0); }

// multiply by exp(SIGN * i*pi/2): SIGN=-1 -> -i (forward), SIGN=+1 -> +i (inverse)
template <int SIGN>
__device__ __forceinline__ double2 mul_q(double2 a) {
  return SIGN < 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}

// exp(SIGN * 2*pi*i*m/16), m in [0,16): compile-time constants after unrolling.
template <int SIGN>
__device__ __forceinline__ double2 w16(int m) {
  constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
  constexpr double h = 0.70710678118654752440;
  const double cs[16] = {1.0, c1, h, s1, 0.0, -s1, -h, -c1, -1.0, -c1, -h, -s1, 0.0, s1, h, c1};
  const double sn[16] = {0.0, s1, h, c1, 1.0, c1, h, s1, 0.0, -s1, -h, -c1, -1.0, -c1, -h, -s1};
  return make_double2(cs[m & 15], SIGN * sn[m & 15]);
}

// multiply by a compile-time 16th root of unity, using the cheap forms where they exist
template <int SIGN>
__device__ __forceinline__ double2 mul_w16(double2 a, int m) {
  m &= 15;
  if (m == 0) return a;
  if (m == 4) return mul_q<SIGN>(a);
  if (m == 8) return make_double2(-a.x, -a.y);
  if (m == 12) return mul_q<-SIGN>(a);
  if (m == 2 || m == 6 || m == 10 || m == 14) {  // (+-1 +- i)/sqrt2
    constexpr double h = 0.70710678118654752440;
    const double2 w = w16<SIGN>(m);
    // (x+iy)(wr+i wi) with |wr|=|wi|=h
    return make_double2(h * ((w.x > 0 ? a.x : -a.x) - (w.y > 0 ? a.y : -a.y)),
                        h * ((w.y > 0 ? a.x : -a.x) + (w.x > 0 ? a.y : -a.y)));
  }
  return cmul(a, w16<SIGN>(m));
}

// ---- in-register DFTs, natural order in and out
template <int R, int SIGN>
struct Dft;

template <int SIGN>
struct Dft<1, SIGN> {
  __device__ __forceinline__ static void run(double2*) {}
};

template <int SIGN>
struct Dft<2, SIGN> {
  __device__ __forceinline__ static void run(double2* x) {
    const double2 a = x[0];
    x[0] = cadd(a, x[1]);
    x[1] = csub(a, x[1]);
  }
};

template <int SIGN>
struct Dft<4, SIGN> {
  __device__ __forceinline__ static void run(double2* x) {
    const double2 s02 = cadd(x[0], x[2]), d02 = csub(x[0], x[2]);
    const double2 s13 = cadd(x[1], x[3]), d13 = mul_q<SIGN>(csub(x[1], x[3]));
    x[0] = cadd(s02, s13);
    x[2] = csub(s02, s13);
    x[1] = cadd(d02, d13);
    x[3] = csub(d02, d13);
  }
};

// multiply by exp(SIGN * 2*pi*i*m/32), m a compile-time constant after unrolling
template <int SIGN>
__device__ __forceinline__ double2 mul_w32(double2 a, int m) {
  m &= 31;
  if ((m & 1) == 0) return mul_w16<SIGN>(a, m >> 1);
  // odd m: cos/sin of pi*m/16
  constexpr double c1 = 0.98078528040323044913, s1 = 0.19509032201612826785;  // pi/16
  constexpr double c3 = 0.83146961230254523708, s3 = 0.55557023301960222474;  // 3pi/16
  const double cs[8] = {c1, c3, s3, s1, -s1, -s3, -c3, -c1};  // m = 1,3,...,15
  const double sn[8] = {s1, s3, c3, c1, c1, c3, s3, s1};
  const int q = (m & 15) >> 1;
  const double sg = (m & 16) ? -1.0 : 1.0;  // exp(i*pi*(m+16)/16) = -exp(i*pi*m/16)
  return cmul(a, make_double2(sg * cs[q], sg * SIGN * sn[q]));
}

// Twiddled radix-2 butterfly x0 = e + W_32^m o, x1 = e - W_32^m o (W = exp(SIGN 2 pi i m/32),
// m a compile-time constant after unrolling) in 6 DFMA instead of 4 (complex product) + 4 (adds):
// W_32^m = (SIGN i)^q W_32^r, m = 8q + r, and W_32^r = c (1 + i SIGN tan) for r <= 4,
// = s (cot + i SIGN) for r > 4 (s = sin = cos of the complement, cot = tan of the complement), so
// W o = K * u with u from two DFMA and the scale K folded into the two output DFMA pairs.
template <int SIGN>
__device__ __forceinline__ void bfly_w32(double2& x0, double2& x1, double2 e, double2 o, int m) {
  m &= 31;
  const int q = m >> 3, r = m & 7;
  if (r == 0) {
    double2 p = o;
    if (q == 1) p = mul_q<SIGN>(o);
    if (q == 2) p = make_double2(-o.x, -o.y);
    if (q == 3) p = mul_q<-SIGN>(o);
    x0 = cadd(e, p);
    x1 = csub(e, p);
    return;
  }
  constexpr double C[5] = {1.0, 0.9807852804032304491262, 0.9238795325112867561282, 0.8314696123025452370788,
                           0.7071067811865475244008};
  constexpr double T[5] = {0.0, 0.1989123673796580069116, 0.4142135623730950488017, 0.6681786379192989199978, 1.0};
  double2 u;
  double k;
  if (r <= 4) {  // c (1 + i SIGN t): u = o (1 + i SIGN t)
    const double t = SIGN * T[r];
    u = make_double2(fma(-t, o.y, o.x), fma(t, o.x, o.y));
    k = C[r];
  } else {  // s (ct + i SIGN): u = o (ct + i SIGN), ct = cot(pi r/16) = tan(pi (8-r)/16)
    const double ct = T[8 - r];
    u = make_double2(fma(ct, o.x, -SIGN * o.y), fma(ct, o.y, SIGN * o.x));
    k = C[8 - r];
  }
  if (q == 1) u = mul_q<SIGN>(u);
  if (q == 2) u = make_double2(-u.x, -u.y);
  if (q == 3) u = mul_q<-SIGN>(u);
  x0 = make_double2(fma(k, u.x, e.x), fma(k, u.y, e.y));
  x1 = make_double2(fma(-k, u.x, e.x), fma(-k, u.y, e.y));
}

// radix-2 decimation in time on top of the half-size DFT: X[k] = E[k] + W^k O[k]
template <int R, int SIGN>
struct Dft {
  __device__ __forceinline__ static void run(double2* x) {
    static_assert(R <= 32, "compile-time twiddles cover radix <= 32");
    double2 e[R / 2], o[R / 2];
#pragma unroll
    for (int r = 0; r < R / 2; ++r) {
      e[r] = x[2 * r];
      o[r] = x[2 * r + 1];
    }
    Dft<R / 2, SIGN>::run(e);
    Dft<R / 2, SIGN>::run(o);
#pragma unroll
    for (int k = 0; k < R / 2; ++k) bfly_w32<SIGN>(x[k], x[k + R / 2], e[k], o[k], k * (32 / R));
  }
};

// DFT of R points whose upper half is zero (zero-padded convolution input):
// X[2k] = DFT_{R/2}(x)[k], X[2k+1] = DFT_{R/2}(x_r W_R^r)[k].
template <int R, int SIGN>
__device__ __forceinline__ void dft_halfzero(double2* x) {
  if constexpr (R == 1) {
    return;
  } else {
    double2 a[R / 2], b[R / 2];
#pragma unroll
    for (int r = 0; r < R / 2; ++r) {
      a[r] = x[r];
      b[r] = mul_w32<SIGN>(x[r], r * (32 / R));
    }
    Dft<R / 2, SIGN>::run(a);
    Dft<R / 2, SIGN>::run(b);
#pragma unroll
    for (int k = 0; k < R / 2; ++k) {
      x[2 * k] = a[k];
      x[2 * k + 1] = b[k];
    }
  }
}

__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }

// ---- asynchronous global -> shared copies (LDGSTS): next work item's operands are staged
// while the current item's transforms run. src_bytes = 0 zero-fills (out-of-range elements).
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}
// Bulk L2 prefetch of a contiguous range (one instruction, no registers, no completion to wait
// on): pulls the next work item's operands from HBM into L2 a whole transform ahead, so the
// later register/shared loads of them hit L2.
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Shared-memory index padding: one spare slot every 2^S entries breaks the bank conflicts of
// the radix-2^S first pass (stride 2^S x 16 B). S >= 30 means no padding (the column kernels
// interleave teams across lanes, which already spreads the banks).
template <int S>
__device__ __forceinline__ int pad_idx(int i) {
  if constexpr (S >= 30) {
    return i;
  } else {
    return i + (i >> S);
  }
}
template <int N, int S>
struct Padded {
  // +1: successive team regions start on different banks
  static constexpr int value = (S >= 30 ? N : N + (N >> S)) + 1;
};
constexpr int kNoPad = 30;

// Accurate table of W_N^k = exp(-2*pi*i*k/N), k < N, in global memory (host long double).
struct TwTable {
  const double2* w;
  int log2n;
};

// Pass schedule: first pass radix R0 = 2^(log2N mod log2E) if nonzero (so that the Ns=1 pass,
// which carries the zero-padding, can be the small one), then NFULL passes of radix E.
// Inter-pass twiddles live in shared memory, one table per full pass laid out [r-1][k]
// (k = b mod Ns fastest) so that consecutive lanes read consecutive entries.
template <int N, int E>
struct FftPlan {
  static constexpr int L = ilog2(N), LE = ilog2(E);
  static constexpr int REM = L % LE;
  static constexpr int R0 = REM ? (1 << REM) : E;
  static constexpr int NFULL = REM ? L / LE : L / LE - 1;
  static constexpr int PADS = ilog2(R0) > 0 ? ilog2(R0) : 1;
  template <int PS>
  static constexpr int smem() { return Padded<N, PS>::value; }  // double2 entries per team
  static constexpr int SMEM = Padded<N, PADS>::value;
  static constexpr int tw_off(int i) {
    int off = 0, ns = R0;
    for (int q = 0; q < i; ++q) {
      off += (E - 1) * ns;
      ns *= E;
    }
    return off;
  }
  static constexpr int TWS = tw_off(NFULL);  // double2 entries of the twiddle tables
};

// Fill the plan's shared twiddle tables from the global W_N table (cooperative, all threads).
template <int N, int E>
__device__ __forceinline__ void load_twiddles(double2* smtw, const TwTable& g) {
  using P = FftPlan<N, E>;
  for (int idx = threadIdx.x; idx < P::TWS; idx += blockDim.x) {
    int off = 0, ns = P::R0, pass = 0;
    while (idx >= off + (E - 1) * ns) {
      off += (E - 1) * ns;
      ns *= E;
      ++pass;
    }
    const int rel = idx - off, r = rel / ns + 1, k = rel % ns;
    // W_{ns E}^{k r} = W_N^{k r N / (ns E)}
    smtw[idx] = __ldg(g.w + (int64_t)k * r * (N / (ns * E)));
  }
}

// One Stockham pass of radix R over a team's data (see file header for the layout).
template <int N, int E, int R, int SIGN, int PADS, bool LAST, bool HALFZERO>
__device__ __forceinline__ void stockham_pass(double2 (&v)[E], double2* sm, int j, int ns,
                                              const double2* twp, bool active) {
  constexpr int T = N / E;
  constexpr int Q = E / R;
  if (active) {
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int b = j + q * T;
      const int k = b & (ns - 1);
      double2 u[R];
#pragma unroll
      for (int r = 0; r < R; ++r) u[r] = v[q + r * Q];
      if (ns > 1) {
#pragma unroll
        for (int r = 1; r < R; ++r) {
          const double2 w = twp[(r - 1) * ns + k];
          u[r] = cmul(u[r], SIGN < 0 ? w : cconj(w));
        }
      }
      if constexpr (HALFZERO) {
        dft_halfzero<R, SIGN>(u);
      } else {
        Dft<R, SIGN>::run(u);
      }
      if constexpr (LAST) {
#pragma unroll
        for (int r = 0; r < R; ++r) v[q + r * Q] = u[r];
      } else {
        const int base = (b - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) sm[pad_idx<PADS>(base + r * ns)] = u[r];
      }
    }
  }
  if constexpr (!LAST) {
    __syncthreads();
    if (active) {
#pragma unroll
      for (int r = 0; r < E; ++r) v[r] = sm[pad_idx<PADS>(j + r * T)];
    }
    __syncthreads();
  }
}

template <int N, int E, int SIGN, int PADS, int IDX, int NPASS>
struct FullPasses {
  __device__ __forceinline__ static void run(double2 (&v)[E], double2* sm, int j, int ns,
                                             const double2* smtw, bool active) {
    if constexpr (IDX < NPASS) {
      stockham_pass<N, E, E, SIGN, PADS, IDX == NPASS - 1, false>(
          v, sm, j, ns, smtw + FftPlan<N, E>::tw_off(IDX), active);
      FullPasses<N, E, SIGN, PADS, IDX + 1, NPASS>::run(v, sm, j, ns * E, smtw, active);
    }
  }
};

// N-point FFT by a team of N/E threads (team-local smem region `sm`, FftPlan::smem<PADS>()
// entries; shared twiddle tables `smtw` filled by load_twiddles<N,E>). Every thread of the CTA
// must call it (barriers); inactive threads pass active=false.
// HALFZERO: entries x[N/2..N) are zero on entry (v[r] for r >= E/2 are ignored).
template <int N, int E, int SIGN, bool HALFZERO, int PADS = FftPlan<N, E>::PADS>
__device__ __forceinline__ void block_fft(double2 (&v)[E], double2* sm, int j, const double2* smtw,
                                          bool active = true) {
  using P = FftPlan<N, E>;
  static_assert(E <= N, "E must not exceed N");
  if constexpr (N == 1) {
    return;
  } else {
    constexpr bool only = (P::NFULL == 0);
    stockham_pass<N, E, P::R0, SIGN, PADS, only, HALFZERO>(v, sm, j, 1, nullptr, active);
    FullPasses<N, E, SIGN, PADS, 0, P::NFULL>::run(v, sm, j, P::R0, smtw, active);
  }
}

// ---- warp-synchronous 1024-point FFT (32 x 32): no block barriers, one shared-memory exchange.
// On entry lane l holds x[l + 32 r] in v[r]; on exit X[l + 32 k] in v[k] (same distribution).
//   step A: DFT_32 over r in registers -> Y_l[k1]; twiddle W_1024^{l k1} (table tw[k1*32 + l]);
//   exchange through the warp's region xs (32 rows x 33, conflict-free both ways);
//   step B: DFT_32 over l in registers.
constexpr int kXS = 32 * 33;  // double2 entries of a warp exchange region
// Step-A twiddles v[k] *= W_1024^{SIGN lane k}, k = 1..31, from 4 table entries: four chains
// t_{j+4m} = t_j (W^{4 lane})^m, at most 7 roundings each (~1e-15 relative), in place of 31
// shared-memory loads on the transform's critical path.
template <int SIGN>
__device__ __forceinline__ void twiddle_a_rec(double2 (&v)[32], const double2* tw, int lane) {
  double2 t[4], w4;
  t[0] = make_double2(1.0, 0.0);
#pragma unroll
  for (int j = 1; j < 4; ++j) t[j] = tw[j * 32 + lane];
  w4 = tw[4 * 32 + lane];
  if (SIGN > 0) {
#pragma unroll
    for (int j = 1; j < 4; ++j) t[j] = cconj(t[j]);
    w4 = cconj(w4);
  }
#pragma unroll
  for (int m = 0; m < 8; ++m) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = 4 * m + j;
      if (m == 0 && j == 0) continue;
      if (m == 1 && j == 0) {
        v[k] = cmul(v[k], w4);
        continue;
      }
      v[k] = cmul(v[k], t[j]);
    }
    if (m < 7) {
#pragma unroll
      for (int j = 0; j < 4; ++j) t[j] = (m == 0 && j == 0) ? w4 : cmul(t[j], w4);
    }
  }
}
// the same, handing each twiddled value to store(k, v[k]) as soon as it is formed (the caller's
// exchange stores then interleave with the twiddle arithmetic)
template <int SIGN, class Store>
__device__ __forceinline__ void twiddle_a_rec_store(double2 (&v)[32], const double2* tw, int lane, Store&& store) {
  double2 t[4], w4;
  t[0] = make_double2(1.0, 0.0);
#pragma unroll
  for (int j = 1; j < 4; ++j) t[j] = tw[j * 32 + lane];
  w4 = tw[4 * 32 + lane];
  if (SIGN > 0) {
#pragma unroll
    for (int j = 1; j < 4; ++j) t[j] = cconj(t[j]);
    w4 = cconj(w4);
  }
#pragma unroll
  for (int m = 0; m < 8; ++m) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = 4 * m + j;
      if (m == 0 && j == 0) {
      } else if (m == 1 && j == 0) {
        v[k] = cmul(v[k], w4);
      } else {
        v[k] = cmul(v[k], t[j]);
      }
      store(k, v[k]);
    }
    if (m < 7) {
#pragma unroll
      for (int j = 0; j < 4; ++j) t[j] = (m == 0 && j == 0) ? w4 : cmul(t[j], w4);
    }
  }
}
template <int SIGN, bool HALFZERO, bool REC = false>
__device__ __forceinline__ void warp_fft1024(double2 (&v)[32], double2* xs, const double2* tw, int lane) {
  if constexpr (HALFZERO) {
    dft_halfzero<32, SIGN>(v);
  } else {
    Dft<32, SIGN>::run(v);
  }
  if constexpr (REC) {
    twiddle_a_rec<SIGN>(v, tw, lane);
  } else {
#pragma unroll
    for (int k = 1; k < 32; ++k) {
      const double2 w = tw[k * 32 + lane];
      v[k] = cmul(v[k], SIGN < 0 ? w : cconj(w));
    }
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 32; ++k) xs[k * 33 + lane] = v[k];
  __syncwarp();
#pragma unroll
  for (int l = 0; l < 32; ++l) v[l] = xs[lane * 33 + l];
  Dft<32, SIGN>::run(v);
}

// The same transform with the exchange inside an interleaved tile of 1024 rows x 8 chunks (16 B):
// warp w's entry i lives at chunk w ^ ((i ^ (i >> 5)) & 7) of row i. The XOR swizzle keeps both
// exchange patterns (i = 32k + lane and i = 32 lane + l) conflict-free, and since each warp owns
// one chunk per row, eight warps can share one tile without synchronising.
__device__ __forceinline__ int tile_idx(int i, int w) { return i * 8 + (w ^ ((i ^ (i >> 5)) & 7)); }
// step A alone (registers + twiddle table): the caller may interleave other work before step B
template <int SIGN, bool HALFZERO, bool REC = false>
__device__ __forceinline__ void warp_fft1024_a(double2 (&v)[32], const double2* tw, int lane) {
  if constexpr (HALFZERO) {
    dft_halfzero<32, SIGN>(v);
  } else {
    Dft<32, SIGN>::run(v);
  }
  if constexpr (REC) {
    twiddle_a_rec<SIGN>(v, tw, lane);
  } else {
#pragma unroll
    for (int k = 1; k < 32; ++k) {
      const double2 t = tw[k * 32 + lane];
      v[k] = cmul(v[k], SIGN < 0 ? t : cconj(t));
    }
  }
}
// L1-resident read-only loads (twiddle tables read from global memory) and L1-bypassing
// streaming loads, so a small L1 (most of the SRAM given to shared memory) keeps the tables.
__device__ __forceinline__ double2 ldg_keep(const double2* p) {
  double2 r;
  asm("ld.global.nc.L1::evict_last.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ double ldg_stream(const double* p) {
  double r;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}
// step A with the W_1024 table in global memory (L1)
template <int SIGN, bool HALFZERO>
__device__ __forceinline__ void warp_fft1024_ag(double2 (&v)[32], const double2* tw, int lane) {
  if constexpr (HALFZERO) {
    dft_halfzero<32, SIGN>(v);
  } else {
    Dft<32, SIGN>::run(v);
  }
#pragma unroll
  for (int k = 1; k < 32; ++k) {
    const double2 t = ldg_keep(tw + k * 32 + lane);
    v[k] = cmul(v[k], SIGN < 0 ? t : cconj(t));
  }
}
// exchange through the tile + step B
template <int SIGN>
__device__ __forceinline__ void warp_fft1024_tb(double2 (&v)[32], double2* T, int w, int lane) {
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 32; ++k) T[tile_idx(32 * k + lane, w)] = v[k];
  __syncwarp();
#pragma unroll
  for (int l = 0; l < 32; ++l) v[l] = T[tile_idx(32 * lane + l, w)];
  Dft<32, SIGN>::run(v);
}
template <int SIGN, bool HALFZERO>
__device__ __forceinline__ void warp_fft1024_t(double2 (&v)[32], double2* T, int w, const double2* tw, int lane) {
  warp_fft1024_a<SIGN, HALFZERO>(v, tw, lane);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 32; ++k) T[tile_idx(32 * k + lane, w)] = v[k];
  __syncwarp();
#pragma unroll
  for (int l = 0; l < 32; ++l) v[l] = T[tile_idx(32 * lane + l, w)];
  Dft<32, SIGN>::run(v);
}

// W_P^e for the four-step twiddles, e < P, from two short tables:
// W_P^e = hi[e >> s] * lo[e & (2^s - 1)].
struct TwoLevel {
  const double2* hi;
  const double2* lo;
  int s;
};
template <int SIGN>
__device__ __forceinline__ double2 tw_p(const TwoLevel& t, uint32_t e) {
  const double2 a = __ldg(t.hi + (e >> t.s));
  const double2 b = __ldg(t.lo + (e & ((1u << t.s) - 1u)));
  const double2 w = cmul(a, b);
  return SIGN < 0 ? w : cconj(w);
}

}  // namespace agk
