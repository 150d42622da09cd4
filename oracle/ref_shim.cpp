// ref_shim.cpp — C entry points over the REFERENCE library compiled from its own sources.
// TEST INFRASTRUCTURE ONLY (see oracle/Makefile): links /root/reference/proj/src/{rhs,fft,
// kernels,steppers,simulator}.cpp into oracle/_ref/libaggkin_ref.so so tests can compare the
// C restatement (agk_oracle.c) and the B200 path against the reference itself. Same struct
// layouts as agk_oracle.h; entry points are named ref_* instead of ora_*.
#include <cmath>
#include <cstring>
#include <limits>
#include <span>
#include <stdexcept>
#include <vector>

#include "agk_oracle.h"
#include "aggkin/analysis.hpp"
#include "aggkin/bench.hpp"
#include "aggkin/config.hpp"
#include "aggkin/report_io.hpp"
#include "aggkin/rhs.hpp"
#include "aggkin/simulator.hpp"
#include "aggkin/steppers.hpp"

using namespace aggkin;

namespace {

ModelSpec to_spec(const ora_model* md) {
  ModelSpec spec;
  spec.variant = static_cast<ModelVariant>(md->variant);
  spec.m = md->m;
  if (md->k) {
    DenseKernel d;
    d.m = md->m;
    d.k.assign(md->k, md->k + md->m * md->m);
    spec.kernel = std::move(d);
  } else {
    LowRankFactors f;
    f.m = md->m;
    f.r = md->r;
    f.u.assign(md->u, md->u + md->m * md->r);
    f.v.assign(md->v, md->v + md->m * md->r);
    spec.kernel = std::move(f);
  }
  for (size_t q = 0; q < md->num_sources; ++q)
    spec.sources.rates.emplace_back(static_cast<std::size_t>(md->source_k[q]), md->source_rate[q]);
  spec.shatter_rate = md->shatter_rate;
  return spec;
}

StepControl to_control(const ora_control* c) {
  StepControl s;
  s.stepper = static_cast<StepperKind>(c->stepper);
  s.mode = static_cast<StepMode>(c->mode);
  s.tau = c->tau;
  s.tol = c->tol;
  s.safety = c->safety;
  s.growth_max = c->growth_max;
  s.shrink_min = c->shrink_min;
  s.tau_min = c->tau_min;
  s.max_rejects = c->max_rejects;
  s.relative_error = c->relative_error != 0;
  return s;
}

RhsFn to_fn(ora_rhs* f, ModelSpec* spec, RhsWorkspace* ws) {
  switch (f->kind) {
    case ORA_RHS_MODEL:
      return [spec, ws, f](std::span<const double> n, std::span<double> out) {
        eval_rhs(*spec, n, *ws, out);
        f->evals = ws->evals();
      };
    case ORA_RHS_DECAY:
      return [f](std::span<const double> n, std::span<double> out) {
        f->evals += 1;
        for (std::size_t i = 0; i < n.size(); ++i) out[i] = -n[i];
      };
    case ORA_RHS_STILL:
      return [f](std::span<const double>, std::span<double> out) {
        f->evals += 1;
        for (double& x : out) x = 0.0;
      };
    case ORA_RHS_DRAIN:
      return [f](std::span<const double>, std::span<double> out) {
        f->evals += 1;
        out[0] = -f->param;
        for (std::size_t i = 1; i < out.size(); ++i) out[i] = 0.0;
      };
    case ORA_RHS_BURST_INF:
      return [f](std::span<const double>, std::span<double> out) {
        f->evals += 1;
        for (double& x : out) x = std::numeric_limits<double>::infinity();
      };
    default:
      return [f](std::span<const double>, std::span<double> out) {
        f->evals += 1;
        for (double& x : out) x = std::numeric_limits<double>::quiet_NaN();
      };
  }
}

}  // namespace

extern "C" {

int ref_eval_rhs(const ora_model* md, const double* n, double* out) try {
  const ModelSpec spec = to_spec(md);
  RhsWorkspace ws;
  eval_rhs(spec, std::span<const double>(n, md->m), ws, std::span<double>(out, md->m));
  return 0;
} catch (const std::exception&) {
  return -1;
}

int ref_birth_term(const ora_model* md, const double* n, double* out) try {
  const ModelSpec spec = to_spec(md);
  RhsWorkspace ws;
  birth_term(spec.kernel, std::span<const double>(n, md->m), ws, std::span<double>(out, md->m));
  return 0;
} catch (const std::exception&) {
  return -1;
}

int ref_death_term(const ora_model* md, const double* n, double* out) try {
  const ModelSpec spec = to_spec(md);
  RhsWorkspace ws;
  death_term(spec.kernel, std::span<const double>(n, md->m), ws, std::span<double>(out, md->m));
  return 0;
} catch (const std::exception&) {
  return -1;
}

int ref_shattering_terms(const ora_model* md, const double* n, double lambda, double* out) try {
  const ModelSpec spec = to_spec(md);
  RhsWorkspace ws;
  shattering_terms(spec.kernel, std::span<const double>(n, md->m), lambda, ws,
                   std::span<double>(out, md->m));
  return 0;
} catch (const std::exception&) {
  return -1;
}

int ref_euler_stability_bound(const ora_model* md, const double* n, double a, double* bound) try {
  const ModelSpec spec = to_spec(md);
  *bound = euler_stability_bound(spec.kernel, std::span<const double>(n, md->m), a);
  return 0;
} catch (const std::exception&) {
  return -1;
}

int ref_rk_step(ora_rhs* f, int stepper, size_t m, const double* n, double tau, double* out,
                double* out5, double* err) try {
  ModelSpec spec;
  if (f->kind == ORA_RHS_MODEL) spec = to_spec(f->model);
  RhsWorkspace ws;
  const RhsFn fn = to_fn(f, &spec, &ws);
  StepperWorkspace sw;
  std::span<const double> ns(n, m);
  std::span<double> os(out, m);
  if (stepper == ORA_RK2) {
    rk2_step(fn, ns, tau, os, sw);
  } else if (stepper == ORA_RK4) {
    rk4_step(fn, ns, tau, os, sw);
  } else {
    std::vector<double> tmp(m);
    const double e = rkf45_step(fn, ns, tau, os, out5 ? std::span<double>(out5, m) : std::span<double>(tmp), sw);
    if (err) *err = e;
  }
  return 0;
} catch (const std::exception&) {
  return -1;
}

int ref_advance(ora_rhs* f, size_t m, const double* n, double tau, const ora_control* c,
                ora_outcome* o, double* state_out) try {
  ModelSpec spec;
  if (f->kind == ORA_RHS_MODEL) spec = to_spec(f->model);
  RhsWorkspace ws;
  const RhsFn fn = to_fn(f, &spec, &ws);
  StepperWorkspace sw;
  const StepOutcome res = advance(fn, std::span<const double>(n, m), tau, to_control(c), sw);
  o->tau_used = res.tau_used;
  o->tau_next = res.tau_next;
  o->error_estimate = res.error_estimate;
  o->rejects = res.rejects;
  o->rhs_evals = res.rhs_evals;
  o->status = static_cast<int>(res.status);
  std::memset(state_out, 0, m * sizeof(double));
  if (res.state.size() == m) std::memcpy(state_out, res.state.data(), m * sizeof(double));
  return 0;
} catch (const std::exception&) {
  return -1;
}

int ref_run(ora_rhs* f, size_t m, const ora_run_desc* d, ora_run_report* rep) try {
  if (f->kind != ORA_RHS_MODEL) return -1;  // run() always drives eval_rhs
  SimulationConfig cfg;
  cfg.model = to_spec(f->model);
  cfg.control = to_control(&d->control);
  cfg.t_end = d->t_end;
  cfg.initial.kind = InitialKind::custom;
  cfg.initial.values.assign(d->initial, d->initial + m);
  cfg.initial_tau = d->initial_tau;
  cfg.snapshot_times.assign(d->snapshot_times, d->snapshot_times + d->num_snapshots);
  cfg.record = static_cast<RecordMode>(d->record);
  cfg.record_interval = d->record_interval;
  const RunReport r = run(cfg);
  rep->termination = r.termination == Termination::completed ? 0 : 1;
  rep->abort_status = 0;
  if (r.termination == Termination::aborted) {
    for (int s = 1; s <= 3; ++s)
      if (r.abort_reason == describe(static_cast<StepStatus>(s))) rep->abort_status = s;
  }
  rep->abort_t = r.abort_t;
  rep->abort_tau = r.abort_tau;
  rep->final_t = r.final_state.t;
  rep->total_rhs_evals = r.total_rhs_evals;
  rep->total_accepted = r.total_accepted;
  rep->total_rejects = r.total_rejects;
  if (rep->final_state) std::memcpy(rep->final_state, r.final_state.n.data(), m * sizeof(double));
  rep->num_snapshots_taken = r.snapshots.size();
  if (rep->snapshots)
    for (std::size_t q = 0; q < r.snapshots.size(); ++q)
      std::memcpy(rep->snapshots + q * m, r.snapshots[q].second.data(), m * sizeof(double));
  rep->num_records = r.records.size();
  if (rep->records)
    for (std::size_t q = 0; q < r.records.size() && q < rep->records_capacity; ++q) {
      const auto& x = r.records[q];
      rep->records[q] = ora_record{x.t, x.tau, x.density, x.mass, x.m2, x.error_estimate, x.rhs_evals, x.rejects};
    }
  return 0;
} catch (const std::exception&) {
  return -1;
}

}  // extern "C"

extern "C" int ref_write_run_outputs(const ora_run_report* r, size_t m, const double* snapshot_times,
                                     const char* abort_reason, double wall_seconds, const char* dir) {
  try {
    RunReport rep;
    for (size_t q = 0; q < r->num_records && q < r->records_capacity; ++q) {
      const ora_record& x = r->records[q];
      ObservableRecord o;
      o.t = x.t;
      o.tau = x.tau;
      o.density = x.density;
      o.mass = x.mass;
      o.m2 = x.m2;
      o.error_estimate = x.error_estimate;
      o.rhs_evals = x.rhs_evals;
      o.rejects = x.rejects;
      rep.records.push_back(o);
    }
    for (size_t q = 0; q < r->num_snapshots_taken; ++q)
      rep.snapshots.emplace_back(snapshot_times[q], std::vector<double>(r->snapshots + q * m, r->snapshots + (q + 1) * m));
    rep.final_state.t = r->final_t;
    if (r->final_state) rep.final_state.n.assign(r->final_state, r->final_state + m);
    rep.termination = r->termination ? Termination::aborted : Termination::completed;
    rep.abort_reason = abort_reason ? abort_reason : "";
    rep.abort_t = r->abort_t;
    rep.abort_tau = r->abort_tau;
    rep.total_rhs_evals = r->total_rhs_evals;
    rep.total_accepted = r->total_accepted;
    rep.total_rejects = r->total_rejects;
    rep.wall_seconds = wall_seconds;
    write_run_outputs(rep, dir);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

extern "C" int ref_write_bench_outputs(const int* schemes, size_t ns, const int* cell_mode, const double* cell_value,
                                       size_t nc, const uint64_t* evals, const uint64_t* accepted,
                                       const uint64_t* rejected, const double* wall, const int* completed,
                                       const char* const* notes, const char* dir) {
  try {
    ExperimentConfig cfg;
    for (size_t i = 0; i < ns; ++i) cfg.bench_schemes.push_back(static_cast<StepperKind>(schemes[i]));
    for (size_t c = 0; c < nc; ++c) cfg.bench_cells.push_back(BenchCell{static_cast<StepMode>(cell_mode[c]), cell_value[c]});
    std::vector<BenchResult> res(ns * nc);
    for (size_t i = 0; i < ns * nc; ++i) {
      res[i].scheme = cfg.bench_schemes[i / nc];
      res[i].cell = cfg.bench_cells[i % nc];
      res[i].rhs_evals = evals[i];
      res[i].accepted = accepted[i];
      res[i].rejected = rejected[i];
      res[i].wall_seconds = wall[i];
      res[i].completed = completed[i] != 0;
      res[i].note = (notes && notes[i]) ? notes[i] : "";
    }
    write_bench_outputs(cfg, res, dir);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}


// Config text -> serialize_config(parse_config_text(text)) (config.cpp:131-438), or the error
// message: returns 0 (serialized), 1 (ConfigError), 2 (other exception); out is NUL-terminated.
extern "C" int ref_parse_config(const char* text, char* out, size_t cap) {
  std::string s;
  int rc = 0;
  try {
    s = serialize_config(parse_config_text(text));
  } catch (const ConfigError& e) {
    s = e.what();
    rc = 1;
  } catch (const std::exception& e) {
    s = e.what();
    rc = 2;
  }
  const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
  std::memcpy(out, s.data(), n);
  out[n] = '\0';
  return rc;
}

// kernel_entry (kernels.cpp:36-57); variant 0 constant, 1 brownian, 2 free_molecular, 3 factors
extern "C" int ref_kernel_entry(int variant, double alpha, size_t i, size_t j, double* out) try {
  KernelSpec spec;
  spec.variant = static_cast<KernelVariant>(variant);
  spec.alpha = alpha;
  *out = kernel_entry(spec, i, j);
  return 0;
} catch (const std::exception&) {
  return -1;
}

// fit_power_law / fit_cutoff (analysis.cpp:59-75): res = {beta, k_lo, k_hi, rms, used, excluded}
extern "C" int ref_fit(const double* n, size_t m, double lam, int cutoff, size_t k_lo, size_t k_hi,
                       double* res) try {
  const std::span<const double> s(n, m);
  const SlopeFit f = cutoff ? fit_cutoff(s, lam, k_lo, k_hi) : fit_power_law(s, k_lo, k_hi);
  res[0] = f.beta;
  res[1] = (double)f.k_lo;
  res[2] = (double)f.k_hi;
  res[3] = f.residual_rms;
  res[4] = (double)f.points_used;
  res[5] = (double)f.points_excluded;
  return 0;
} catch (const std::exception&) {
  return -1;
}
