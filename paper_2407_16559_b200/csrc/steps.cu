// steps.cu — RK stage combinations, fused final pass + reductions, the device step controller
// and the graph that runs the trial loop without host round trips.
//
// Replaces the reference steppers and controllers (src/steppers.cpp:11-300) and the run loop
// (src/simulator.cpp:112-229):
//   * k_comb: one HBM pass per stage combination (stage = n + tau * sum a_ij k_j), with the
//     reference's coefficient tableau (steppers.hpp:59-74) and expression structure;
//   * the final combination of a trial (n4/n5 of RKF45, the half-step state of step doubling,
//     the fixed-step result) also produces, in the same pass, every reduction the controller
//     needs: ||n5-n4||^2 (or ||half-full||^2), finiteness of both vectors, min and max|.| (the
//     negativity floor, steppers.cpp:44-50), ||cand||^2 (relative mode) and the N/M1/M2
//     moments of the candidate (simulator.cpp:130-145) — fixed-order CTA partials;
//   * k_controller: one warp reduces the partials in fixed order and applies the reference's
//     accept/reject rules (fehlberg_adaptive 246-291, step_doubling_adaptive 188-244,
//     fixed_step 161-186), the run-loop landing/slack/proposal bookkeeping (simulator.cpp:
//     170-217), records and snapshots, and sets the CUDA-graph WHILE condition.
#include <cmath>

#include "steps.cuh"

namespace agk {

constexpr double kErrFloor = 1e-300;             // steppers.cpp:11
constexpr double kNegativeRejectFraction = 1e-3; // steppers.cpp:14
constexpr int kRedThreads = 256;

struct OutRef {
  double* base;
  const int* sel;
  int64_t stride;
  int flip;
  __device__ __forceinline__ double* get() const {
    if (!sel) return base;
    const int c = *sel;
    return base + (flip ? 1 - c : c) * stride;
  }
};

struct CombArgs {
  VecRef x;
  const double* y[6];
  OutRef out;
  const double* other;  // C_*_OUT with RED in doubling: the full-step state
  double* n5;           // C_F_OUT: optional n5 store (when ctl->store_n5)
  const DevCtl* ctl;
  double tau_mul;
  int64_t m;
  double* red;
};

__device__ __forceinline__ bool finite_d(double x) { return isfinite(x); }

// the y slot each input of a combination comes from
__host__ __device__ constexpr int comb_slot(int kind, int j) { return kind == C_F_OUT && j > 0 ? j + 1 : j; }

template <int KIND, bool RED>
__global__ void __launch_bounds__(kRedThreads) k_comb(CombArgs a) {
  pdl_entry();
  const double t = a.tau_mul * a.ctl->tau;
  const double* __restrict__ x = a.x.get();
  double* __restrict__ out = a.out.get();
  const bool store5 = (KIND == C_F_OUT) && a.ctl->store_n5;
  double acc[RF_N];
  if (RED) {
#pragma unroll
    for (int q = 0; q < RF_N; ++q) acc[q] = 0.0;
    acc[RF_MIN] = __longlong_as_double(0x7ff0000000000000LL);
  }
  constexpr int NY = comb_inputs(KIND);
  // one element: the stage combination, its store, and the fused reductions of the final pass
  // returns the output value o; the caller stores it (and n5 = `other` for C_F_OUT)
  auto elem = [&](int64_t i, double xi, const double* yy, double ovi, double& other) -> double {
    double o;
    other = 0.0;
    using namespace rkf;
    if constexpr (KIND == C_F_OUT) {  // inputs k1, k3, k4, k5, k6
      comb_f_out(t, xi, yy, o, other);
    } else {
      o = comb_value<KIND>(t, xi, yy);  // the same expression as a fused stage (stage.cuh)
    }
    const double n5v = other;
    if (RED) {
      if (KIND != C_F_OUT && a.other) other = ovi;
      if (KIND == C_F_OUT || a.other) {
        const double d = o - other;
        acc[RF_ERR2] += d * d;
        if (!finite_d(other)) acc[RF_NF_OTHER] = 1.0;
      }
      if (!finite_d(o)) acc[RF_NF_CAND] = 1.0;
      const double kk = (double)(i + 1);
      acc[RF_L2SQ] += o * o;
      acc[RF_MOM0] += o;
      acc[RF_MOM1] += kk * o;
      acc[RF_MOM2] += kk * kk * o;
      acc[RF_MIN] = o < acc[RF_MIN] ? o : acc[RF_MIN];
      const double ab = fabs(o);
      acc[RF_MAXABS] = acc[RF_MAXABS] < ab ? ab : acc[RF_MAXABS];
    }
    other = n5v;
    return o;
  };
  // kU element pairs (16-byte loads) per thread per step, all loads issued before any
  // arithmetic: a pass over 8 MiB vectors needs that memory-level parallelism from 2 CTAs per SM
  // (the partial-sum CTAs). Odd m: the same with single elements.
  constexpr int kU = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool want_other = RED && KIND != C_F_OUT && a.other;
  if ((a.m & 1) == 0) {
    const int64_t mp = a.m / 2;
    auto ld2 = [](const double* p, int64_t k) { return reinterpret_cast<const double2*>(p)[k]; };
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < mp; i0 += kU * stride) {
      double2 xv[kU], yv[NY][kU], ov[kU];
#pragma unroll
      for (int q = 0; q < kU; ++q) {
        const int64_t k = i0 + q * stride < mp ? i0 + q * stride : i0;  // clamped: unpredicated loads
        xv[q] = ld2(x, k);
#pragma unroll
        for (int j = 0; j < NY; ++j) yv[j][q] = ld2(a.y[comb_slot(KIND, j)], k);
        ov[q] = want_other ? ld2(a.other, k) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int q = 0; q < kU; ++q) {
        const int64_t k = i0 + q * stride;
        if (k >= mp) break;
        double y0[NY], y1[NY];
#pragma unroll
        for (int j = 0; j < NY; ++j) {
          y0[j] = yv[j][q].x;
          y1[j] = yv[j][q].y;
        }
        double f0, f1;
        const double o0 = elem(2 * k, xv[q].x, y0, ov[q].x, f0);
        const double o1 = elem(2 * k + 1, xv[q].y, y1, ov[q].y, f1);
        reinterpret_cast<double2*>(out)[k] = make_double2(o0, o1);
        if (store5) reinterpret_cast<double2*>(a.n5)[k] = make_double2(f0, f1);
      }
    }
  } else {
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < a.m; i0 += kU * stride) {
      double xv[kU], yv[NY][kU], ov[kU];
#pragma unroll
      for (int q = 0; q < kU; ++q) {
        const int64_t i = i0 + q * stride < a.m ? i0 + q * stride : i0;
        xv[q] = x[i];
#pragma unroll
        for (int j = 0; j < NY; ++j) yv[j][q] = a.y[comb_slot(KIND, j)][i];
        ov[q] = want_other ? a.other[i] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < kU; ++q) {
        const int64_t i = i0 + q * stride;
        if (i >= a.m) break;
        double yy[NY];
#pragma unroll
        for (int j = 0; j < NY; ++j) yy[j] = yv[j][q];
        double f0;
        out[i] = elem(i, xv[q], yy, ov[q], f0);
        if (store5) a.n5[i] = f0;
      }
    }
  }
  if (RED) {
    __shared__ double red[kRedThreads / 32][RF_N];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < RF_N; ++q) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, acc[q], off);
        if (q == RF_MIN) acc[q] = o < acc[q] ? o : acc[q];
        else if (q == RF_MAXABS || q == RF_NF_CAND || q == RF_NF_OTHER) acc[q] = acc[q] < o ? o : acc[q];
        else acc[q] += o;
      }
      if (lane == 0) red[warp][q] = acc[q];
    }
    __syncthreads();
    if (threadIdx.x < RF_N) {
      const int q = threadIdx.x;
      double s = red[0][q];
      for (int w = 1; w < kRedThreads / 32; ++w) {
        const double o = red[w][q];
        if (q == RF_MIN) s = o < s ? o : s;
        else if (q == RF_MAXABS || q == RF_NF_CAND || q == RF_NF_OTHER) s = s < o ? o : s;
        else s += o;
      }
      a.red[blockIdx.x * RF_N + q] = s;
    }
  }
}

// Moments of the current state (for the t = 0 record), partials [blk][3].
__global__ void __launch_bounds__(kRedThreads) k_state_moments(VecRef xr, int64_t m, double* part) {
  const double* x = xr.get();
  double s[3] = {0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const double kk = (double)(i + 1), o = x[i];
    s[0] += o;
    s[1] += kk * o;
    s[2] += kk * kk * o;
  }
  __shared__ double red[kRedThreads / 32][3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], off);
    if (lane == 0) red[warp][q] = s[q];
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) t += red[w][threadIdx.x];
    part[blockIdx.x * 3 + threadIdx.x] = t;
  }
}

// w_a partial dot products V_a . n, grid (nblk, r) -> dots[a*nblk + b]
__global__ void __launch_bounds__(kRedThreads) k_rank_dots(const double* v, VecRef xr, int64_t m, double* dots) {
  const double* x = xr.get();
  const int a = blockIdx.y, nb = gridDim.x;
  const double* va = v + (int64_t)a * m;
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)nb * blockDim.x) s += va[i] * x[i];
  __shared__ double red[kRedThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) t += red[w];
    dots[a * nb + blockIdx.x] = t;
  }
}

// Per-CTA max over s of rowsum_s = sum_a U_sa w_a (NaN-ignoring, from 0 as the reference's
// std::max fold), partials [blk].
__global__ void __launch_bounds__(kRedThreads) k_rowsum_max(const double* ut, int r, int64_t m, const double* dots,
                                                            int ndot, double* rmax) {
  extern __shared__ double w[];
  for (int a = threadIdx.x; a < r; a += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < ndot; ++b) s += dots[a * ndot + b];
    w[a] = s;
  }
  __syncthreads();
  double pk = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    double rs = 0.0;
    for (int a = 0; a < r; ++a) rs += ut[(int64_t)a * m + i] * w[a];
    pk = (pk < rs) ? rs : pk;
  }
  __shared__ double red[kRedThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double o = __shfl_xor_sync(0xffffffffu, pk, off);
    pk = (pk < o) ? o : pk;
  }
  if (lane == 0) red[warp] = pk;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < kRedThreads / 32; ++q) t = (t < red[q]) ? red[q] : t;
    rmax[blockIdx.x] = t;
  }
}

__device__ double reduce_max_seq(const double* p, int n) {
  double t = 0.0;
  for (int q = 0; q < n; ++q) t = (t < p[q]) ? p[q] : t;
  return t;
}

__global__ void k_euler_final(const double* rmax, int n, double a, double* out) {
  const double peak = reduce_max_seq(rmax, n);
  *out = !(peak > 0.0) ? __longlong_as_double(0x7ff0000000000000LL) : a / peak;
}

// ------------------------------------------------------------------ controller

__device__ __forceinline__ double dmax(double a, double b) { return (a < b) ? b : a; }  // std::max
__device__ __forceinline__ double dclamp(double v, double lo, double hi) {           // std::clamp
  return (v < lo) ? lo : (hi < v) ? hi : v;
}
__device__ __forceinline__ double inf_d() { return __longlong_as_double(0x7ff0000000000000LL); }
__device__ __forceinline__ double nan_d() { return __longlong_as_double(0x7ff8000000000000LL); }

// Records go to a device ring; the controller pauses the WHILE loop when the ring is full so
// the host can drain it (agk_run), hence the slot is never one the host has not copied yet.
__device__ void push_record(DevCtl* c, double tau, double err) {
  if (c->rec_buf && c->nrec - c->rec_drained < c->rec_cap) {
    agk_record& r = c->rec_buf[c->nrec % c->rec_cap];
    r.t = c->t;
    r.tau = tau;
    r.density = c->mom[0];
    r.mass = c->mom[1];
    r.m2 = c->mom[2];
    r.error_estimate = err;
    r.rhs_evals = c->evals;
    r.rejects = c->rejects_total;
  }
  c->nrec += 1;
  c->last_rec_t = c->t;
}

__device__ void ctl_abort(DevCtl* c, int status, double tau_used) {
  c->status = status;
  c->tau_used = tau_used;
  c->done = 1;
  if (c->run_mode == RUN_LOOP) {
    c->abort_t = c->t;
    c->abort_tau = tau_used > 0.0 ? tau_used : c->tau_try;  // simulator.cpp:188
    c->rejects_total += c->step_rejects;
  }
}

// Head of a step of the run loop (simulator.cpp:170-183) and of the first trial (tau_min check,
// steppers.cpp:203-207 / 258-262).
__device__ void begin_step(DevCtl* c) {
  if (!(c->t < c->t_end)) {
    c->done = 1;
    return;
  }
  double t_target = c->t_end;
  if (c->snap_idx < c->nsnap && c->snap_times[c->snap_idx] < c->t_end) t_target = c->snap_times[c->snap_idx];
  const double remaining = t_target - c->t;
  const double slack = 1e-12 * dmax(1.0, fabs(t_target));
  const int shortened = remaining - c->proposal <= slack;
  c->t_target = t_target;
  c->remaining = remaining;
  c->shortened = shortened;
  c->tau_try = shortened ? remaining : c->proposal;
  c->tau = c->tau_try;
  c->step_rejects = 0;
  c->step_evals = 0;
  c->tau_used = 0.0;
  c->tau_next = 0.0;
  c->err = nan_d();
  if (c->mode == AGK_ADAPTIVE && c->tau < c->tau_min) ctl_abort(c, AGK_STEP_TAU_UNDERFLOW, c->tau);
}

__device__ void take_snapshots(DevCtl* c) {
  c->snap_from = c->snap_idx;
  while (c->snap_idx < c->nsnap && c->snap_times[c->snap_idx] == c->t) ++c->snap_idx;  // simulator.cpp:149-156
  c->snap_to = c->snap_idx;
}

__global__ void k_prologue(DevCtl* c, const double* mom_part, int nmom, const double* rmax, int nrmax,
                           cudaGraphConditionalHandle h) {
  if (threadIdx.x != 0) return;
  c->snap_from = c->snap_to = 0;
  if (c->resume) {  // continuing a run paused to drain the record ring: the loop state stands
    c->resume = 0;
    c->paused = 0;
    cudaGraphSetConditional(h, c->done ? 0u : 1u);
    return;
  }
  c->paused = 0;
  double s[3] = {0.0, 0.0, 0.0};
  for (int b = 0; b < nmom; ++b)
    for (int q = 0; q < 3; ++q) s[q] += mom_part[b * 3 + q];
  c->mom[0] = s[0];
  c->mom[1] = s[1];
  c->mom[2] = s[2];
  c->done = 0;
  c->status = AGK_STEP_OK;
  c->snap_from = c->snap_to = 0;
  c->k1_valid = 0;
  if (c->run_mode == RUN_LOOP) {
    c->t = 0.0;
    if (c->record != AGK_RECORD_NONE) push_record(c, 0.0, nan_d());
    c->next_record_t = c->record_interval;
    take_snapshots(c);
    double proposal;
    if (c->mode == AGK_FIXED) {
      proposal = c->tau_fixed;
    } else if (c->initial_tau > 0.0) {
      proposal = c->initial_tau;
    } else {
      proposal = inf_d();
      if (c->has_model) {
        const double peak = reduce_max_seq(rmax, nrmax);
        proposal = !(peak > 0.0) ? inf_d() : 0.25 / peak;  // euler_stability_bound(n0, 0.25)
      }
      if (!isfinite(proposal) || proposal <= 0.0) proposal = 0.01;  // kFallbackInitialTau
      if (c->t_end > 0.0) proposal = (c->t_end < proposal) ? c->t_end : proposal;
    }
    c->proposal = proposal;
    begin_step(c);
    if (!c->done && c->rec_buf && c->nrec - c->rec_drained >= c->rec_cap) c->paused = 1;
  } else {
    c->tau = c->tau_try;
    c->step_rejects = 0;
    c->step_evals = 0;
    c->err = nan_d();
    c->tau_used = 0.0;
    c->tau_next = 0.0;
    if (c->mode == AGK_ADAPTIVE && c->tau < c->tau_min) ctl_abort(c, AGK_STEP_TAU_UNDERFLOW, c->tau);
  }
  cudaGraphSetConditional(h, (c->done || c->paused) ? 0u : 1u);
}

__global__ void __launch_bounds__(32) k_controller(DevCtl* c, const double* part, int nblk,
                                                   cudaGraphConditionalHandle h) {
  pdl_entry();
  // fixed-order reduction of the final pass' CTA partials
  const int lane = threadIdx.x;
  double v[RF_N];
#pragma unroll
  for (int q = 0; q < RF_N; ++q) v[q] = 0.0;
  v[RF_MIN] = inf_d();
  for (int b = lane; b < nblk; b += 32) {
#pragma unroll
    for (int q = 0; q < RF_N; ++q) {
      const double o = part[b * RF_N + q];
      if (q == RF_MIN) v[q] = o < v[q] ? o : v[q];
      else if (q == RF_MAXABS || q == RF_NF_CAND || q == RF_NF_OTHER) v[q] = v[q] < o ? o : v[q];
      else v[q] += o;
    }
  }
#pragma unroll
  for (int q = 0; q < RF_N; ++q) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double o = __shfl_xor_sync(0xffffffffu, v[q], off);
      if (q == RF_MIN) v[q] = o < v[q] ? o : v[q];
      else if (q == RF_MAXABS || q == RF_NF_CAND || q == RF_NF_OTHER) v[q] = v[q] < o ? o : v[q];
      else v[q] += o;
    }
  }
  if (lane != 0) return;
  c->snap_from = c->snap_to = 0;
  const int per = c->stepper == AGK_RK2 ? 2 : (c->stepper == AGK_RK4 ? 4 : 6);
  const bool nf_cand = v[RF_NF_CAND] != 0.0, nf_other = v[RF_NF_OTHER] != 0.0;
  bool accept = false;
  if (c->mode == AGK_FIXED) {  // fixed_step (steppers.cpp:161-186)
    c->evals += per;
    c->step_evals += per;
    c->tau_used = c->tau;
    c->tau_next = c->tau;
    c->err = c->stepper == AGK_RKF45 ? sqrt(v[RF_ERR2]) : nan_d();
    if (nf_cand) ctl_abort(c, AGK_STEP_NONFINITE, c->tau);
    else accept = true;
  } else {
    const bool fehlberg = c->body == BODY_FEHLBERG;
    const int evals = fehlberg ? 6 : 3 * per;
    c->evals += evals;
    c->step_evals += evals;
    double err = sqrt(v[RF_ERR2]);
    const bool finite = !nf_cand && !nf_other && (fehlberg ? isfinite(err) : true);
    if (!finite) {
      err = inf_d();
    } else {
      if (c->relative_error) err /= dmax(1.0, sqrt(v[RF_L2SQ]));
      if (v[RF_MIN] < -kNegativeRejectFraction * v[RF_MAXABS]) err = inf_d();
    }
    const double safety = c->safety > 0.0 ? c->safety : (fehlberg ? 0.9 : 0.25);
    double factor = 0.0;
    if (fehlberg) factor = dclamp(safety * pow(c->tol / dmax(err, kErrFloor), 0.2), c->shrink_min, c->growth_max);
    if (err > c->tol) {
      c->tau *= fehlberg ? factor : 0.5;
      c->k1_valid = 1;  // n unchanged: S(n) in K1 is reused by the retry
      if (++c->step_rejects > c->max_rejects) {
        ctl_abort(c, finite ? AGK_STEP_TOO_MANY_REJECTS : AGK_STEP_NONFINITE, c->tau);
      } else if (c->tau < c->tau_min) {
        ctl_abort(c, AGK_STEP_TAU_UNDERFLOW, c->tau);
      }
    } else {
      accept = true;
      c->tau_used = c->tau;
      c->err = err;
      if (fehlberg) {
        c->tau_next = factor * c->tau;
      } else {
        const double p = c->stepper == AGK_RK2 ? 2.0 : 4.0;
        const double raw = safety * c->tau * pow(c->tol / dmax(err, kErrFloor), 1.0 / p);
        c->tau_next = dclamp(raw, c->shrink_min * c->tau, c->growth_max * c->tau);
      }
    }
  }
  if (accept) {
    c->cur ^= 1;
    c->k1_valid = 0;
    c->mom[0] = v[RF_MOM0];
    c->mom[1] = v[RF_MOM1];
    c->mom[2] = v[RF_MOM2];
    if (c->run_mode == RUN_ADVANCE) {
      c->done = 1;
    } else {
      c->accepted += 1;
      c->rejects_total += c->step_rejects;
      const bool landed = c->tau_used == c->tau_try;
      c->t = (landed && c->tau_try == c->remaining) ? c->t_target : c->t + c->tau_used;
      if (c->mode == AGK_ADAPTIVE && (!c->shortened || c->step_rejects > 0)) c->proposal = c->tau_next;
      if (c->record == AGK_RECORD_EVERY_STEP) {
        push_record(c, c->tau_used, c->err);
      } else if (c->record == AGK_RECORD_INTERVAL && c->t >= c->next_record_t) {
        push_record(c, c->tau_used, c->err);
        c->next_record_t = c->record_interval * (floor(c->t / c->record_interval) + 1.0);
      }
      take_snapshots(c);
      begin_step(c);
      // the ring is full: leave the WHILE loop (not done) so the host drains it and resumes
      if (!c->done && c->rec_buf && c->nrec - c->rec_drained >= c->rec_cap) c->paused = 1;
    }
  }
  cudaGraphSetConditional(h, (c->done || c->paused) ? 0u : 1u);
}

// Deep copies of the accepted state for the snapshot times the controller just reached.
__global__ void k_snap_copy(const DevCtl* c, const double* state, int64_t m) {
  pdl_entry();
  const int from = c->snap_from, to = c->snap_to;
  if (to <= from || !c->snap_buf) return;
  const double* x = state + c->cur * m;
  for (int q = from; q < to; ++q)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
      c->snap_buf[q * m + i] = x[i];
}

// ------------------------------------------------------------------ graph construction

int red_blocks_for(int64_t m) {
  int64_t b = (m + 2047) / 2048;
  if (b < 1) b = 1;
  if (b > 296) b = 296;
  return (int)b;
}


template <int KIND, bool RED>
static cudaError_t comb(CombArgs a, int nblk, cudaStream_t s) {
  AGK_CK(launch_k(k_comb<KIND, RED>, nblk, kRedThreads, 0, s, pdl_enabled() && (pdl_mask() & 16), a));
  return cudaGetLastError();
}

cudaError_t launch_euler_bound(const RhsArgs& md, VecRef n, double a, double* aux, int naux, double* out_dev,
                               cudaStream_t s) {
  double* dots = aux + naux * 4;
  double* rmax = aux + naux * 3;
  if (md.kd) {
    AGK_CK(launch_dense_rowmax(md, n, rmax, naux, s));
  } else {
    k_rank_dots<<<dim3(naux, md.r), kRedThreads, 0, s>>>(md.v, n, md.m, dots);
    k_rowsum_max<<<naux, kRedThreads, md.r * sizeof(double), s>>>(md.ut, md.r, md.m, dots, naux, rmax);
  }
  k_euler_final<<<1, 1, 0, s>>>(rmax, naux, a, out_dev);
  return cudaGetLastError();
}

cudaError_t build_step_graph(int body, int stepper, const RhsEnqueue& rhs, const StepBuffers& b, DevCtl* ctl,
                             int64_t m, const RhsArgs* model, cudaStream_t s, cudaGraphExec_t* exec,
                             int* kernels_per_trial) {
  cudaGraph_t g = nullptr;
  AGK_CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  AGK_CK(cudaGraphConditionalHandleCreate(&h, g, 0, 0));

  const VecRef state{b.state, &ctl->cur, m};
  const OutRef cand{b.state, &ctl->cur, m, 1};
  const int nb = b.nred;

  // ---- prologue: moments of the initial state, Euler bound partials, controller setup
  AGK_CK(cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  double* mom = b.aux;
  double* rmax = b.aux + b.naux * 3;
  double* dots = b.aux + b.naux * 4;
  k_state_moments<<<b.naux, kRedThreads, 0, s>>>(state, m, mom);
  if (model && model->kd) {
    AGK_CK(launch_dense_rowmax(*model, state, rmax, b.naux, s));
  } else if (model) {
    k_rank_dots<<<dim3(b.naux, model->r), kRedThreads, 0, s>>>(model->v, state, m, dots);
    k_rowsum_max<<<b.naux, kRedThreads, model->r * sizeof(double), s>>>(model->ut, model->r, m, dots, b.naux, rmax);
  }
  k_prologue<<<1, 32, 0, s>>>(ctl, mom, b.naux, rmax, model ? b.naux : 0, h);
  k_snap_copy<<<nb, kRedThreads, 0, s>>>(ctl, b.state, m);
  AGK_CK(cudaGetLastError());
  {
    cudaStreamCaptureStatus st;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    AGK_CK(cudaStreamGetCaptureInfo(s, &st, nullptr, nullptr, &deps, &ndeps));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    AGK_CK(cudaGraphAddNode(&cn, g, deps, ndeps, &cp));
    AGK_CK(cudaStreamUpdateCaptureDependencies(s, &cn, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t done_g = nullptr;
    AGK_CK(cudaStreamEndCapture(s, &done_g));

    // ---- body: one trial
    cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
    AGK_CK(cudaStreamBeginCaptureToGraph(s, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  }
  int nk = 0, nrhs = 0;
  const int* k1skip = &ctl->k1_valid;
  double* const* K = b.k;
  CombArgs ca{};
  ca.ctl = ctl;
  ca.m = m;
  ca.red = b.red;
  ca.n5 = b.n5;
  auto st_args = [&](VecRef x, double* out, std::initializer_list<const double*> ys, double tmul) {
    CombArgs r = ca;
    r.x = x;
    r.out = OutRef{out, nullptr, 0, 0};
    int q = 0;
    for (const double* y : ys) r.y[q++] = y;
    r.tau_mul = tmul;
    r.other = nullptr;
    return r;
  };
  auto plain = [](const double* p) { return VecRef{p, nullptr, 0}; };
  // RHS of the stage x + tau * tmul * sum_j a_j ys[j] (CombKind `kind`): fused into the RHS's first
  // kernel when the RHS supports it, else a stage-combination pass into b.stg and the RHS of b.stg
  const bool fuse = rhs.stage_fusable();
  int nfused = 0;
  auto stage_rhs = [&](int kind, VecRef x, std::initializer_list<const double*> ys, double tmul,
                       double* out) -> cudaError_t {
    if (fuse) {
      StageIn st{};
      st.on = 1;
      st.kind = kind;
      int q = 0;
      for (const double* y : ys) st.y[q++] = y;
      st.tau = &ctl->tau;
      st.tau_mul = tmul;
      ++nfused;
      return rhs.stage(x, st, b.stg, out, s);
    }
    const CombArgs ca2 = st_args(x, b.stg, ys, tmul);
    switch (kind) {
      case C_RK2_ST: AGK_CK((comb<C_RK2_ST, false>(ca2, nb, s))); break;
      case C_RK4_STH: AGK_CK((comb<C_RK4_STH, false>(ca2, nb, s))); break;
      case C_RK4_ST1: AGK_CK((comb<C_RK4_ST1, false>(ca2, nb, s))); break;
      case C_F2: AGK_CK((comb<C_F2, false>(ca2, nb, s))); break;
      case C_F3: AGK_CK((comb<C_F3, false>(ca2, nb, s))); break;
      case C_F4: AGK_CK((comb<C_F4, false>(ca2, nb, s))); break;
      case C_F5: AGK_CK((comb<C_F5, false>(ca2, nb, s))); break;
      default: AGK_CK((comb<C_F6, false>(ca2, nb, s))); break;
    }
    return rhs(plain(b.stg), out, nullptr, s);
  };

  if (body == BODY_FEHLBERG) {
    AGK_CK(rhs(state, K[0], k1skip, s));
    AGK_CK(stage_rhs(C_F2, state, {K[0]}, 1.0, K[1]));
    AGK_CK(stage_rhs(C_F3, state, {K[0], K[1]}, 1.0, K[2]));
    AGK_CK(stage_rhs(C_F4, state, {K[0], K[1], K[2]}, 1.0, K[3]));
    AGK_CK(stage_rhs(C_F5, state, {K[0], K[1], K[2], K[3]}, 1.0, K[4]));
    AGK_CK(stage_rhs(C_F6, state, {K[0], K[1], K[2], K[3], K[4]}, 1.0, K[5]));
    CombArgs fa = st_args(state, nullptr, {K[0], K[1], K[2], K[3], K[4], K[5]}, 1.0);
    fa.out = cand;
    AGK_CK(comb<C_F_OUT, true>(fa, nb, s));
    nk = 6;
    nrhs = 6;
  } else {
    // one rk2/rk4 step from x with tau*tmul into `out` (or the candidate); k1 is S(x) in k1buf
    auto step = [&](VecRef x, const double* k1buf, bool k1_needed, const int* k1skip_, double tmul,
                    double* out_plain, bool to_cand, const double* other) -> cudaError_t {
      if (k1_needed) {
        AGK_CK(rhs(x, const_cast<double*>(k1buf), k1skip_, s));
        ++nrhs;
      }
      CombArgs fa{};
      if (stepper == AGK_RK2) {
        AGK_CK(stage_rhs(C_RK2_ST, x, {k1buf}, tmul, K[1]));
        fa = st_args(x, out_plain, {k1buf, K[1]}, tmul);
        nk += 2;
        nrhs += 1;
      } else {
        AGK_CK(stage_rhs(C_RK4_STH, x, {k1buf}, tmul, K[1]));
        AGK_CK(stage_rhs(C_RK4_STH, x, {K[1]}, tmul, K[2]));
        AGK_CK(stage_rhs(C_RK4_ST1, x, {K[2]}, tmul, K[3]));
        fa = st_args(x, out_plain, {k1buf, K[1], K[2], K[3]}, tmul);
        nk += 4;
        nrhs += 3;
      }
      if (to_cand) {
        fa.out = cand;
        fa.other = other;
        if (stepper == AGK_RK2) AGK_CK((comb<C_RK2_OUT, true>(fa, nb, s)));
        else AGK_CK((comb<C_RK4_OUT, true>(fa, nb, s)));
      } else {
        if (stepper == AGK_RK2) AGK_CK((comb<C_RK2_OUT, false>(fa, nb, s)));
        else AGK_CK((comb<C_RK4_OUT, false>(fa, nb, s)));
      }
      return cudaSuccess;
    };
    if (body == BODY_FIXED) {
      AGK_CK(step(state, K[0], true, k1skip, 1.0, nullptr, true, nullptr));
    } else {
      // full step, then two half steps; S(n) is shared by the full and first half step
      AGK_CK(step(state, K[0], true, k1skip, 1.0, b.full, false, nullptr));
      AGK_CK(step(state, K[0], false, nullptr, 0.5, b.mid, false, nullptr));
      AGK_CK(step(plain(b.mid), K[6], true, nullptr, 0.5, nullptr, true, b.full));
    }
  }
  AGK_CK(launch_k(k_controller, 1, 32, 0, s, pdl_enabled() && (pdl_mask() & 16), ctl, (const double*)b.red, nb, h));
  AGK_CK(launch_k(k_snap_copy, nb, kRedThreads, 0, s, pdl_enabled() && (pdl_mask() & 16), (const DevCtl*)ctl, (const double*)b.state, m));
  nk += 2;
  AGK_CK(cudaGetLastError());
  cudaGraph_t bg = nullptr;
  AGK_CK(cudaStreamEndCapture(s, &bg));
  AGK_CK(cudaGraphInstantiate(exec, g, 0));
  AGK_CK(cudaGraphDestroy(g));
  if (kernels_per_trial) *kernels_per_trial = nk - nfused + nrhs * rhs.launches();
  return cudaSuccess;
}

}  // namespace agk
