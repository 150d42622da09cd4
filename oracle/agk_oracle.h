/* agk_oracle.h — CPU restatement of the reference hot path. TEST INFRASTRUCTURE ONLY.
 *
 * This is the parity checker for the B200 path, not a product path: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * It restates, in plain C11, the algorithms of the reference `aggkin` library
 * (/root/reference/proj, C++20):
 *   - low-rank RHS   : src/rhs.cpp:24-46 (row sums), 87-151 (birth), 162-168 (death),
 *                      170-210 (shattering), 212-235 (eval_rhs), 284-294 (Euler bound)
 *   - dense RHS      : the DenseKernel branches of the same functions, rhs.cpp:37-45 (row sums),
 *                      153-159 (birth), 197-205 (shattering gains)
 *   - FFT            : src/fft.cpp:64-137 (built-in radix-2; the reference build here has no FFTW)
 *   - steppers       : src/steppers.cpp:11-50 (helpers), 94-159 (steps), 161-300 (controllers)
 *   - run loop       : src/simulator.cpp:112-229
 * in the same floating-point operation order, so that compiled with the reference's own
 * Release flags (-O3 -DNDEBUG, proj/CMakeLists.txt:8-10) it is bitwise identical to the
 * reference built from its sources (oracle/_ref, see oracle/Makefile). tests/test_oracle_pin.py
 * checks that identity, plus the reference's own hand values and committed run goldens.
 *
 * Parity pinned: against oracle/_ref (reference compiled from source) and against the
 * reference's committed goldens (proj/out/<*>/summary.txt counts) and test hand values.
 */
#ifndef AGK_ORACLE_H
#define AGK_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ModelVariant (rhs.hpp:30) */
enum { ORA_AGGREGATION = 0, ORA_AGGREGATION_SOURCES = 1, ORA_AGGREGATION_SHATTERING = 2 };

/* Which right-hand side drives the steppers: the model, or one of the injected fakes the
 * reference's stepper tests bind to RhsFn (test_steppers.cpp:15-17, 251-253, 405-408, 424-434). */
enum {
  ORA_RHS_MODEL = 0,
  ORA_RHS_DECAY = 1,     /* out = -n */
  ORA_RHS_STILL = 2,     /* out = 0 */
  ORA_RHS_DRAIN = 3,     /* out[0] = -param, out[i>0] = 0 */
  ORA_RHS_BURST_INF = 4, /* out = +inf */
  ORA_RHS_BURST_NAN = 5  /* out = NaN */
};

typedef struct {
  size_t m, r;
  const double* u; /* m x r row-major: U(i,a) = u[(i-1)*r + a] (kernels.hpp:32) */
  const double* v; /* r x m row-major: V(a,j) = v[a*m + j-1]   (kernels.hpp:33) */
  int variant;
  const uint64_t* source_k; /* 1-based sizes, in application order */
  const double* source_rate;
  size_t num_sources;
  double shatter_rate;
  const double* k; /* DenseKernel (kernels.hpp:38-43): m x m row-major, K(i,j) = k[(i-1)*m + j-1];
                      when non-NULL the kernel is dense and r/u/v are ignored */
} ora_model;

/* Returns 0 on success, -1 on invalid argument (the reference throws std::invalid_argument). */
int ora_eval_rhs(const ora_model* model, const double* n, double* out);
int ora_birth_term(const ora_model* model, const double* n, double* out);
int ora_death_term(const ora_model* model, const double* n, double* out);
int ora_shattering_terms(const ora_model* model, const double* n, double lambda, double* out);
int ora_euler_stability_bound(const ora_model* model, const double* n, double a, double* bound);
/* Dense literal-sum oracle of eval_rhs_dense_oracle (rhs.cpp:237-282) evaluated on the
 * low-rank factors' entries K(i,j) = sum_a U(i,a) V(a,j) (kernels.cpp LowRankFactors::entry). */
int ora_eval_rhs_dense(const ora_model* model, const double* n, double* out);
/* The same RHS with every intermediate in long double (agk_truth.c): accuracy yardstick. */
int ora_eval_rhs_truth(const ora_model* model, const double* n, double* out);

/* StepControl (steppers.hpp:18-36) */
enum { ORA_RK2 = 0, ORA_RK4 = 1, ORA_RKF45 = 2 };
enum { ORA_FIXED = 0, ORA_ADAPTIVE = 1 };
typedef struct {
  int stepper, mode;
  double tau, tol, safety, growth_max, shrink_min, tau_min;
  int max_rejects, relative_error;
} ora_control;
void ora_control_defaults(ora_control* c);

/* StepStatus / StepOutcome (steppers.hpp:38-50) */
enum { ORA_STEP_OK = 0, ORA_STEP_NONFINITE = 1, ORA_STEP_TOO_MANY_REJECTS = 2, ORA_STEP_TAU_UNDERFLOW = 3 };
typedef struct {
  double tau_used, tau_next, error_estimate;
  int rejects, rhs_evals, status;
} ora_outcome;

typedef struct {
  int kind;              /* ORA_RHS_* */
  double param;          /* drain rate */
  const ora_model* model;/* kind == ORA_RHS_MODEL */
  uint64_t evals;        /* RhsWorkspace::evals() equivalent */
} ora_rhs;

/* Single steps (steppers.cpp:98-159). rkf45 returns ||n5-n4||_2 through *err. */
int ora_rk_step(ora_rhs* rhs, int stepper, size_t m, const double* n, double tau, double* out,
                double* out5, double* err);
/* advance (steppers.cpp:293-300). state_out gets the outcome state (m values). Returns -1
 * for the argument errors the reference throws on. */
int ora_advance(ora_rhs* rhs, size_t m, const double* n, double tau, const ora_control* c,
                ora_outcome* o, double* state_out);

/* SimulationConfig / RunReport subset (simulator.hpp:24-64). */
typedef struct {
  ora_control control;
  double t_end;
  const double* initial; /* m values */
  double initial_tau;
  const double* snapshot_times;
  size_t num_snapshots;
  int record;            /* 0 every_step, 1 interval, 2 none (RecordMode) */
  double record_interval;
} ora_run_desc;

typedef struct {
  double t, tau, density, mass, m2, error_estimate;
  uint64_t rhs_evals, rejects;
} ora_record;

typedef struct {
  int termination;      /* 0 completed, 1 aborted */
  int abort_status;     /* ORA_STEP_* that aborted */
  double abort_t, abort_tau, final_t;
  uint64_t total_rhs_evals, total_accepted, total_rejects;
  double* final_state;  /* caller buffer (m) or NULL */
  double* snapshots;    /* caller buffer (num_snapshots x m) or NULL */
  size_t num_snapshots_taken;
  ora_record* records;  /* caller buffer or NULL */
  size_t records_capacity;
  size_t num_records;   /* total produced (may exceed capacity; extra ones dropped) */
} ora_run_report;

int ora_run(ora_rhs* rhs, size_t m, const ora_run_desc* d, ora_run_report* rep);

/* Reference writers (report_io.cpp:32-98, bench.cpp:126-171), exported by oracle/_ref only: the
 * byte-compatibility checkers of paper_2407_16559_b200/report_io.py. abort_reason: "" when the
 * run completed. Bench: schemes[ns] (ORA_RK*), cells (mode[nc], value[nc]); results row-major
 * [scheme][cell] with status 1 = completed; notes[ns*nc] (NULL entries = ""). */
int ref_write_run_outputs(const ora_run_report* rep, size_t m, const double* snapshot_times,
                          const char* abort_reason, double wall_seconds, const char* dir);
int ref_write_bench_outputs(const int* schemes, size_t ns, const int* cell_mode, const double* cell_value,
                            size_t nc, const uint64_t* evals, const uint64_t* accepted, const uint64_t* rejected,
                            const double* wall, const int* completed, const char* const* notes, const char* dir);

#ifdef __cplusplus
}
#endif
#endif
