// steps.cuh — device-side step controller state and stepper launch interface.
#pragma once
#include "internal.h"

namespace agk {

enum BodyKind { BODY_FIXED = 0, BODY_DOUBLING = 1, BODY_FEHLBERG = 2 };
enum RunMode { RUN_ADVANCE = 0, RUN_LOOP = 1 };

// Reduction fields of the fused final-combination pass (one row of doubles per CTA).
enum RedField {
  RF_ERR2 = 0,   // sum (cand - other)^2  (n5-n4 for the embedded pair, half-full for doubling)
  RF_L2SQ = 1,   // sum cand^2
  RF_MOM0 = 2,   // sum cand          (N, density)
  RF_MOM1 = 3,   // sum k cand        (M1, mass)
  RF_MOM2 = 4,   // sum k^2 cand      (M2)
  RF_MIN = 5,    // min cand
  RF_MAXABS = 6, // max |cand|
  RF_NF_CAND = 7,  // 1 if cand has a non-finite entry
  RF_NF_OTHER = 8, // 1 if the other vector has a non-finite entry
  RF_N = 9
};

// Controller state in device memory. Host writes the configuration block before a launch and
// reads the result after; every kernel of the captured graphs reads what it needs from here,
// so one instantiated graph serves every tau / tol / t_end.
struct DevCtl {
  // configuration
  int stepper, mode, max_rejects, relative_error;
  double tol, safety, growth_max, shrink_min, tau_min, tau_fixed;
  int run_mode, body;
  double t_end, initial_tau;
  int nsnap, record;
  const double* snap_times;
  double* snap_buf;
  double record_interval;
  agk_record* rec_buf;   // device ring of rec_cap records (drained by the host between segments)
  int64_t rec_cap;
  long long rec_drained; // records the host has copied out of the ring
  int resume;            // 1: relaunch after a drain pause (the prologue keeps the loop state)
  int paused;            // set by the controller when the ring is full: WHILE exits, not done
  int store_n5, has_model;
  // trial / step state
  int cur, k1_valid;
  double t, tau, proposal, tau_try, remaining, t_target;
  int shortened, step_rejects, step_evals;
  int done, status;
  double tau_used, tau_next, err;
  unsigned long long evals, accepted, rejects_total;
  double abort_t, abort_tau;
  int snap_idx, snap_from, snap_to;
  long long nrec;
  double last_rec_t;     // t of the last record pushed (closing-record rule, simulator.cpp:219-222)
  double next_record_t;
  double mom[3];
};

struct StepBuffers {
  double* state;  // 2 x m (double-buffered accepted state)
  double* k[7];   // K1..K6, K1b (S of the mid state in step doubling)
  double* stg;
  double* full;
  double* mid;
  double* n5;     // optional n5 store for rk_step
  double* red;    // reduction partials nblk x RF_N
  int nred;       // CTAs of the fused vector passes
  double* aux;    // prologue partials (moments, rank dots, row-sum max)
  int naux;
};

// Build (capture) the graph of a stepper body + controller on `s`. rhs(in, out, skip) must
// enqueue one RHS evaluation on `s`.
struct RhsEnqueue {
  virtual cudaError_t operator()(VecRef in, double* out, const int* skip, cudaStream_t s) const = 0;
  virtual int launches() const = 0;  // kernels one call enqueues
  // Fused stage: one RHS of the stage x + tau * sum_j a_j y_j (StageIn) whose first kernel forms
  // the stage itself and stores it to stg, in place of a stage-combination kernel + RHS(stg).
  virtual bool stage_fusable() const { return false; }
  virtual cudaError_t stage(VecRef, const StageIn&, double*, double*, cudaStream_t) const { return cudaErrorNotSupported; }
  virtual ~RhsEnqueue() = default;
};

cudaError_t build_step_graph(int body, int stepper, const RhsEnqueue& rhs, const StepBuffers& b,
                             DevCtl* ctl, int64_t m, const RhsArgs* model, cudaStream_t s,
                             cudaGraphExec_t* exec, int* kernels_per_trial);

// Euler stability bound a / max_s rowsum_s on device (rhs.cpp:284-294); result in *out_dev.
cudaError_t launch_euler_bound(const RhsArgs& model, VecRef n, double a, double* aux, int naux,
                               double* out_dev, cudaStream_t s);

int red_blocks_for(int64_t m);

}  // namespace agk
