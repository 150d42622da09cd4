// internal.h — device-side parameter blocks shared by the RHS, stepper and API translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "agk/agk.h"
#include "fft.cuh"
#include "stage.cuh"

namespace agk {

// Epilogue terms (eval_rhs = birth - death [+ sources | + shattering]); the term-level entry
// points birth_term / death_term / shattering_terms select subsets.
enum TermFlags : int {
  T_BIRTH = 1,       // + 0.5 * conv
  T_DEATH = 2,       // - n_s * rowsum_s
  T_DEATH_POS = 4,   // + n_s * rowsum_s (death_term's own sign)
  T_SOURCES = 8,     // + P_k at k-1
  T_SHATTER = 16,    // shattering terms with lambda
};

// Device addresses of the state vector an RHS reads: n + (*sel) * sel_stride when sel != null
// (the run loop double-buffers the state and flips an index instead of copying).
struct VecRef {
  const double* base;
  const int* sel;
  int64_t stride;
  __device__ __forceinline__ const double* get() const { return sel ? base + (*sel) * stride : base; }
};

// Everything an RHS evaluation needs, by value in every kernel.
struct RhsArgs {
  VecRef n;             // input state (m); with a fused stage (st.on): the stage's base x
  StageIn st;           // fused RK stage: the RHS input is n + tau * sum a_j y_j (stage.cuh)
  double* stg_out;      // fused stage: the first kernel stores the stage vector here (m) for the others
  double* out;          // output S(n) (m)
  const int* skip;      // if non-null and *skip != 0 the whole evaluation is skipped
  int64_t m;
  int r;                // all ranks
  int rf;               // unique ranks (FFT count)
  const double* ut;     // r x m: U transposed (ut[a*m + i] = U(i+1, a))
  const double* v;      // r x m: V as in the reference
  const int* uniq_rank; // rf: original rank index of unique rank ub
  const double* uniq_weight; // rf: fold weight (1 + number of folded copies)
  const int* rank_map;  // r: unique index of rank a, +1000000 if folded swapped
  const double* u0;     // r: U(1, a)
  const double* v0;     // r: V(a, 1)
  int flags;            // TermFlags
  double lambda;
  const int64_t* src_k; // 1-based
  const double* src_rate;
  int nsrc;
  // four-step geometry
  int log2p;
  int n1, n2;           // P = n1 * n2
  // scratch
  double2* y;           // group intermediate (gsize * P)
  double2* acc;         // (n1/2 + 1) * n2 accumulator, then G rows
  double* partials;     // rf * nblk_colfwd * 4
  double* scalars;      // r (w_a) + 2 (pair_gain, mono_gain)
  int pfd;           // fast path: L2 prefetch distance of the column/row passes (items)
  int nblk_colfwd;
  TwTable tw_n1, tw_n2, tw_small;
  TwoLevel twp;
  // warp fast path (P = 2^21): column-major (U,V) per unique rank, n in grid layout, tables
  const double2* uvg;
  double* ng;
  const double2* tw32;     // [k1*32 + l] = W_1024^{l k1}
  const double2* tw2048h;  // [r*32 + l] = W_2048^{l + 32 r}
  double* dvec;            // m: the non-birth part of S (death, sources, shattering)
  // dense kernel (rhs_dense.cu): K m x m row-major, row sums, shattering-gain terms per row,
  // per-chunk birth partials (dense_chunks(m) x m)
  const double* kd;
  double* drow;
  double* dpair;
  double* dpart;
  int dbg;                 // experiment switches (AGK_DBG), 0 in production
  unsigned long long* tl;  // timeline stamps (AGK_DBG & 512, experiments build), else null
};

// Launch geometry and per-handle tables for one problem size.
struct RhsPlan {
  int small;     // 1: single-CTA path (P <= 4096)
  int fast;      // 1: warp-synchronous path (P = 2^21)
  int dense;     // 1: DenseKernel path (rhs_dense.cu); no FFT
  int log2p;
  int n1, n2, c, cp;
  int gsize;     // ranks per group in the four-step path
  int launches;  // kernels per RHS
  // SM count (grid sizing of the fast path)
  int nsm;
};

// kernel classes for per-launch timing
enum KernelClass { K_SMALL = 0, K_COL_FWD = 1, K_ROW = 2, K_COL_INV = 3, K_TRANSPOSE = 4, K_DVEC = 5, K_ROW_INV = 6, K_DENSE_ROWS = 7, K_DENSE_BIRTH = 8 };

// Programmatic dependent launch (PDL) along the chain of kernels of one RHS and of one RK trial:
// a kernel launched with pdl = true is scheduled while its predecessor drains, runs only a
// prologue that touches immutable data (twiddle tables, kernel factors) and shared memory, then
// pdl_entry()/griddepcontrol.wait before anything written by earlier launches, and triggers its
// own dependents only after that wait — so a dependent overlaps its immediate predecessor only.
// AGK_PDL=0 turns it off (ordinary stream serialisation); per-kernel timing marks also do.
// Experiment knobs (tools/ab.sh, tools/timeline.py, tools/tune.py): read from the environment
// ONLY in a library built with -DAGK_EXPERIMENTS (`make EXPERIMENTS=1`). The production library
// ignores the environment entirely, so no stray variable can change the plan or skip work.
#ifdef AGK_EXPERIMENTS
int knob(const char* name, int dflt);
#define AGK_XDBG(a, bits) (((a).dbg & (bits)) != 0)
#define AGK_TL(a, k, what) tl_stamp((a).tl, k, what)
#define AGK_PFDIST(a) ((a).pfd)
#else
inline int knob(const char*, int dflt) { return dflt; }
#define AGK_XDBG(a, bits) false
#define AGK_TL(a, k, what) ((void)0)
#define AGK_PFDIST(a) 1  // L2 prefetch distance of the row pass (items), measured best
#endif
bool pdl_enabled();
int pdl_mask();  // AGK_PDLMASK experiment bits (default all)
#ifndef AGK_CK
#define AGK_CK(...)                   \
  do {                                \
    cudaError_t e_ = (__VA_ARGS__);   \
    if (e_ != cudaSuccess) return e_; \
  } while (0)
#endif
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                            Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, args...);
}
#ifdef __CUDACC__
// timeline stamp of kernel class k (0 first arrival, 1 first start of work, 2 last exit), %globaltimer ns
__device__ __forceinline__ void tl_stamp(unsigned long long* tl, int k, int what) {
  if (tl && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    if (what < 2) atomicMin(tl + 3 * k + what, t);
    else atomicMax(tl + 3 * k + what, t);
  }
}
unsigned long long* timeline_ptr();  // rhs_w.cu: device address of the timeline array
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_entry() {
  pdl_wait();
  pdl_trigger();
}
#endif

// host-side launchers (rhs.cu)
void rhs_make_plan(int64_t m, int rf, RhsPlan* plan);
cudaError_t rhs_launch(const RhsPlan& plan, const RhsArgs& a, cudaStream_t s);
// same, recording ev[i] after the i-th kernel (class cls[i]); *n = kernels launched
cudaError_t rhs_launch_marked(const RhsPlan& plan, const RhsArgs& a, cudaStream_t s, cudaEvent_t* ev, int* cls,
                              int cap, int* n);
size_t rhs_y_elems(const RhsPlan& plan);
size_t rhs_acc_elems(const RhsPlan& plan);
size_t rhs_partial_elems(const RhsPlan& plan, int rf);
cudaError_t rhs_set_smem_limits();
// warp fast path (rhs_w.cu)
cudaError_t rhs_w_set_smem_limits();
cudaError_t rhs_w_launch(const RhsPlan& p, const RhsArgs& a, cudaStream_t s, void (*mark)(void*, int, cudaStream_t),
                         void* mk);

// dense-kernel path (rhs_dense.cu)
int dense_chunks(int64_t m);
cudaError_t rhs_dense_launch(const RhsPlan& p, const RhsArgs& a, cudaStream_t s, void (*mark)(void*, int, cudaStream_t),
                             void* mk);
// per-CTA maxima of the dense row sums of n into rmax[nblk] (Euler bound)
cudaError_t launch_dense_rowmax(const RhsArgs& md, VecRef n, double* rmax, int nblk, cudaStream_t s);

// Injected fakes (AGK_RHS_DECAY, ...) as one elementwise kernel.
cudaError_t fake_rhs_launch(int kind, double param, VecRef n, double* out, int64_t m,
                            const int* skip, cudaStream_t s);

}  // namespace agk
