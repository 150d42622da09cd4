/* agk.h — C ABI of the B200-native low-rank Smoluchowski RHS + adaptive Runge–Kutta path.
 *
 * Drop-in boundary for the reference `aggkin` hot path (/root/reference/proj). Every entry
 * point below names the reference interface it replaces (file:line). Plain pointers and sizes
 * only; no CUDA or torch types cross this boundary. All arithmetic is IEEE fp64 on the GPU
 * (sm_100a); there is no CPU fallback: creating a handle without a usable B200 fails with
 * AGK_ERR_NO_DEVICE.
 *
 * Ownership and threading (mirrors RhsWorkspace, rhs.hpp:42-44): a handle owns its device
 * buffers, one CUDA stream and its captured graphs. Calls on different handles may run
 * concurrently from different host threads; one handle must not be used by two threads at
 * once. Errors: an agk_status, and agk_last_error(handle) for the message (the reference
 * throws std::invalid_argument with the same conditions). No entry point changes the calling
 * thread's current CUDA device.
 *
 * Stream ordering of device pointers (AGK_MEM_DEVICE): the handle's stream is a BLOCKING
 * stream, so it is ordered after all work previously queued on the legacy default stream
 * (stream 0, e.g. torch's default stream) and that stream waits for it. Inputs produced on any
 * other stream must be complete before the call (synchronize that stream or record/wait an
 * event); the paper_2407_16559_b200 Python wrapper synchronizes torch's current stream for CUDA
 * tensors. Every call except agk_rhs_eval_async returns after its outputs are written.
 */
#ifndef AGK_AGK_H
#define AGK_AGK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AGK_ABI_VERSION 3

typedef enum {
  AGK_OK = 0,
  AGK_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  AGK_ERR_NO_DEVICE = 2,        /* no sm_100 device visible: the path refuses to run */
  AGK_ERR_CUDA = 3,             /* CUDA runtime failure (message in agk_last_error) */
  AGK_ERR_OUT_OF_MEMORY = 4
} agk_status;

/* ModelVariant (rhs.hpp:30) */
typedef enum { AGK_AGGREGATION = 0, AGK_AGGREGATION_SOURCES = 1, AGK_AGGREGATION_SHATTERING = 2 } agk_variant;

/* Where the n/out pointers of an eval/step call live. */
typedef enum { AGK_MEM_HOST = 0, AGK_MEM_DEVICE = 1 } agk_mem;

/* ModelSpec with a LowRankFactors kernel (rhs.hpp:32-40, kernels.hpp:26-35). Factors are
 * copied to the device at create time (the handle keeps its own copy), so the host arrays may
 * be freed afterwards. Layouts are the reference's: U is m x r row-major (U(i,a) =
 * u[(i-1)*r + a]), V is r x m row-major (V(a,j) = v[a*m + j-1]). */
typedef struct {
  size_t m;                 /* truncation size, >= 2 */
  size_t r;                 /* rank, >= 1 */
  const double* u;
  const double* v;
  int variant;              /* agk_variant */
  const uint64_t* source_k; /* aggregation_sources: 1-based sizes (SourceTerm::rates) */
  const double* source_rate;
  size_t num_sources;
  double shatter_rate;      /* aggregation_shattering: lambda >= 0 */
  int device;               /* CUDA device ordinal; -1 = current device */
  const double* k;          /* DenseKernel (kernels.hpp:38-43): m x m row-major, K(i,j) =
                               k[(i-1)*m + j-1]. Non-NULL selects the dense path (rhs.cpp
                               dense branches 37-45, 153-159, 197-205) and r/u/v are ignored;
                               m <= 2^17. NULL: the low-rank factors u/v. (ABI version 2) */
} agk_model_desc;

/* Injected right-hand sides: the reference's stepper tests bind these to RhsFn
 * (steppers.hpp:12; test_steppers.cpp:15-17, 251-253, 405-408, 424-434). They run on the
 * device like the model RHS, so the controller under test is the production one. */
typedef enum {
  AGK_RHS_MODEL = 0,
  AGK_RHS_DECAY = 1,     /* out = -n */
  AGK_RHS_STILL = 2,     /* out = 0 */
  AGK_RHS_DRAIN = 3,     /* out[0] = -param, out[i>0] = 0 */
  AGK_RHS_BURST_INF = 4, /* out = +inf */
  AGK_RHS_BURST_NAN = 5  /* out = NaN */
} agk_rhs_kind;

typedef struct agk_rhs agk_rhs;

/* RhsWorkspace + ModelSpec in one handle. Replaces: ModelSpec::validate (rhs.cpp:63-72),
 * RhsWorkspace::prepare (rhs.cpp:74-85) and the per-call rank dedupe (rhs.cpp:96-124), which
 * is evaluated once here with the reference's bitwise rule. */
agk_status agk_rhs_create(const agk_model_desc* desc, agk_rhs** out);
/* Handle whose RHS is one of the injected fakes (kind != AGK_RHS_MODEL), size m. */
agk_status agk_rhs_create_fake(int kind, size_t m, double param, int device, agk_rhs** out);
void agk_rhs_destroy(agk_rhs* h);
size_t agk_rhs_size(const agk_rhs* h);
/* Number of distinct FFT ranks after dedupe, and the per-rank fold weights (r values). */
size_t agk_rhs_unique_ranks(const agk_rhs* h);

/* eval_rhs (rhs.cpp:212-235; rhs.hpp:89-90): out = S(n). Adds exactly 1 to the evaluation
 * counter. n/out are host or device pointers of m doubles (agk_mem). Synchronous. */
agk_status agk_rhs_eval(agk_rhs* h, const double* n, double* out, int where);
/* Same on the handle's stream without synchronizing (device pointers only). */
agk_status agk_rhs_eval_async(agk_rhs* h, const double* n_dev, double* out_dev);
/* birth_term (rhs.cpp:87-151), death_term (rhs.cpp:162-168), shattering_terms
 * (rhs.cpp:170-210). These do not count evaluations, like the reference. */
agk_status agk_birth_term(agk_rhs* h, const double* n, double* out, int where);
agk_status agk_death_term(agk_rhs* h, const double* n, double* out, int where);
agk_status agk_shattering_terms(agk_rhs* h, const double* n, double lambda, double* out, int where);
/* euler_stability_bound (rhs.cpp:284-294); +inf when the state gives no bound. */
agk_status agk_euler_stability_bound(agk_rhs* h, const double* n, double a, double* bound, int where);
/* RhsWorkspace::evals / reset_evals (rhs.hpp:49-50). */
uint64_t agk_rhs_evals(const agk_rhs* h);
void agk_rhs_reset_evals(agk_rhs* h);

/* StepperKind, StepMode, StepControl (steppers.hpp:14-36). */
typedef enum { AGK_RK2 = 0, AGK_RK4 = 1, AGK_RKF45 = 2 } agk_stepper;
typedef enum { AGK_FIXED = 0, AGK_ADAPTIVE = 1 } agk_mode;
typedef struct {
  int stepper;        /* agk_stepper */
  int mode;           /* agk_mode */
  double tau;         /* fixed mode step */
  double tol;         /* adaptive tolerance */
  double safety;      /* 0 = per-rule default (0.25 doubling, 0.9 Fehlberg) */
  double growth_max;  /* 2 */
  double shrink_min;  /* 0.5 */
  double tau_min;     /* 1e-12 */
  int max_rejects;    /* 40 */
  int relative_error; /* 0 */
} agk_control;
/* The reference defaults (steppers.hpp:18-36). */
void agk_control_defaults(agk_control* c);
/* StepControl::validate (steppers.cpp:71-86). */
agk_status agk_control_validate(const agk_control* c);

/* StepStatus / StepOutcome (steppers.hpp:38-50); error_estimate is NaN when unavailable. */
typedef enum { AGK_STEP_OK = 0, AGK_STEP_NONFINITE = 1, AGK_STEP_TOO_MANY_REJECTS = 2, AGK_STEP_TAU_UNDERFLOW = 3 } agk_step_status;
typedef struct {
  double tau_used;
  double tau_next;
  double error_estimate;
  int rejects;
  int rhs_evals;
  int status; /* agk_step_status */
} agk_outcome;

/* rk2_step / rk4_step / rkf45_step (steppers.cpp:98-159): one explicit step at exactly tau.
 * For rkf45, out = n4, out5 = n5 (may be NULL) and *err = ||n5-n4||_2 (may be NULL). */
agk_status agk_rk_step(agk_rhs* h, int stepper, const double* n, double tau, double* out,
                       double* out5, double* err, int where);
/* advance (steppers.cpp:293-300 → fixed_step 161-186, step_doubling_adaptive 188-244,
 * fehlberg_adaptive 246-291). The whole trial loop runs on the device. state_out receives the
 * accepted state (left untouched unless status == AGK_STEP_OK). */
agk_status agk_advance(agk_rhs* h, const double* n, double tau, const agk_control* c,
                       agk_outcome* out, double* state_out, int where);

/* RecordMode (simulator.hpp:22) */
typedef enum { AGK_RECORD_EVERY_STEP = 0, AGK_RECORD_INTERVAL = 1, AGK_RECORD_NONE = 2 } agk_record_mode;

/* SimulationConfig (simulator.hpp:24-37) with InitialKind::custom: the model is the handle's. */
typedef struct {
  agk_control control;
  double t_end;
  const double* initial;         /* m host doubles */
  double initial_tau;            /* 0 = Euler bound a=1/4, fallback 0.01 (simulator.cpp:158-168) */
  const double* snapshot_times;  /* strictly ascending within [0, t_end] */
  size_t num_snapshots;
  int record;                    /* agk_record_mode */
  double record_interval;
} agk_run_desc;

/* ObservableRecord (simulator.hpp:39-48) */
typedef struct {
  double t, tau, density, mass, m2, error_estimate;
  uint64_t rhs_evals, rejects;
} agk_record;

/* Record stream (ABI 3): called on the calling thread, in order, with every record the run
 * produces, the closing record (simulator.cpp:219-222) included. The device keeps records in
 * a ring buffer and pauses the WHILE graph to drain it into the sink, so no record is dropped
 * whatever the run length (the reference RunReport keeps them all, simulator.cpp:130-145). */
typedef void (*agk_record_sink)(void* user, const agk_record* recs, size_t n);

/* RunReport (simulator.hpp:52-64). Caller-provided buffers may be NULL. */
typedef struct {
  int termination;           /* 0 completed, 1 aborted */
  int abort_status;          /* agk_step_status that aborted the run */
  double abort_t, abort_tau;
  double final_t;
  uint64_t total_rhs_evals, total_accepted, total_rejects;
  double wall_seconds;
  double* final_state;       /* in: host buffer of m doubles, or NULL */
  double* snapshots;         /* in: host buffer num_snapshots x m, or NULL */
  size_t num_snapshots_taken;
  agk_record* records;       /* in: host buffer, or NULL */
  size_t records_capacity;
  size_t num_records;        /* produced; the first records_capacity are also stored in records */
  agk_record_sink record_sink; /* in: receives every record (ABI 3), or NULL */
  void* sink_user;
} agk_run_report;

/* run (simulator.cpp:112-229): the whole integration runs as one device-resident CUDA graph
 * (conditional WHILE node over trials); the host waits once at the end. */
agk_status agk_run(agk_rhs* h, const agk_run_desc* d, agk_run_report* rep);

/* Last error message for this handle (or the calling thread's last create failure if h is
 * NULL). Valid until the next call on the same handle. */
const char* agk_last_error(const agk_rhs* h);
const char* agk_describe_status(int step_status); /* describe (simulator.cpp:98-110) */

/* Device-side timing hook for bench.py: launches `count` back-to-back eval_rhs on device
 * buffers through the captured per-RHS graph, and returns the elapsed device milliseconds
 * measured with CUDA events on the handle's stream. Counts `count` evaluations. */
agk_status agk_rhs_eval_timed(agk_rhs* h, const double* n_dev, double* out_dev, int count,
                              float* elapsed_ms);
/* Number of kernel launches one eval_rhs issues (for bench.py's gpu_launches). */
int agk_rhs_launches_per_eval(const agk_rhs* h);

/* Per-launch device time of one eval_rhs, averaged over `reps` evaluations: CUDA events are
 * recorded on the handle's stream between consecutive kernels. ms[i] and cls[i] (kernel class:
 * 0 single-CTA, 1 column-forward, 2 row, 3 column-inverse) for i < *n (at most cap). Counts
 * `reps` evaluations. Also reports the plan: log2 P, N1, N2, ranks per group. */
agk_status agk_rhs_profile(agk_rhs* h, const double* n_dev, double* out_dev, int reps, double* ms, int* cls,
                           int cap, int* n, int* plan4);

#ifdef __cplusplus
}
#endif
#endif /* AGK_AGK_H */
