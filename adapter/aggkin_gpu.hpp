// aggkin_gpu.hpp — drop-in C++ adapter: the reference `aggkin` operator API (rhs.hpp,
// steppers.hpp, simulator.hpp) served by the B200 C ABI (include/agk/agk.h).
//
// A reference maintainer includes this header next to the reference's own headers and links
// libagk_b200.so. The reference's value types are used unchanged (ModelSpec, StepControl,
// StepOutcome, SimulationConfig, RunReport); only the workspace type differs, because the
// device handle owns the factors, scratch and graphs that RhsWorkspace owns on the CPU:
//
//   reference                                        adapter (namespace aggkin::gpu)
//   RhsWorkspace ws;                                 GpuWorkspace ws(model);
//   eval_rhs(model, n, ws, out)   (rhs.hpp:89)       eval_rhs(model, n, ws, out)
//   birth_term / death_term / shattering_terms       same names, GpuWorkspace&
//   euler_stability_bound(kernel, n, a) (rhs.hpp:99) euler_stability_bound(ws, n, a)
//   advance(rhs, n, tau, control, step_ws) (steppers.hpp:109)
//                                                    advance(ws, n, tau, control)
//   run(config)                   (simulator.hpp:75) run(config)
//   RhsFn                          (steppers.hpp:12) as_rhs_fn(ws) (parity only: host copies)
//
// Errors: argument errors throw std::invalid_argument (as the reference), CUDA failures and a
// missing B200 throw std::runtime_error. There is no CPU fallback.
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <span>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "agk/agk.h"
#include "aggkin/rhs.hpp"
#include "aggkin/simulator.hpp"
#include "aggkin/steppers.hpp"

namespace aggkin::gpu {

inline void check(agk_status st, const agk_rhs* h) {
  if (st == AGK_OK) return;
  const std::string msg = agk_last_error(h);
  if (st == AGK_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error("agk: " + msg);
}

inline agk_control to_control(const StepControl& c) {
  agk_control a;
  a.stepper = static_cast<int>(c.stepper);
  a.mode = static_cast<int>(c.mode);
  a.tau = c.tau;
  a.tol = c.tol;
  a.safety = c.safety;
  a.growth_max = c.growth_max;
  a.shrink_min = c.shrink_min;
  a.tau_min = c.tau_min;
  a.max_rejects = c.max_rejects;
  a.relative_error = c.relative_error ? 1 : 0;
  return a;
}

// RhsWorkspace + the model's device copy. One per concurrent caller (rhs.hpp:42-44).
class GpuWorkspace {
 public:
  explicit GpuWorkspace(const ModelSpec& model, int device = -1) : m_(model.m) {
    model.validate();
    const auto* lr = std::get_if<LowRankFactors>(&model.kernel);
    const auto* dk = std::get_if<DenseKernel>(&model.kernel);  // dense path: rhs_dense.cu
    std::vector<uint64_t> k;
    std::vector<double> rate;
    for (const auto& [kk, rr] : model.sources.rates) {
      k.push_back(kk);
      rate.push_back(rr);
    }
    agk_model_desc d{};
    d.m = model.m;
    if (lr) {
      d.r = lr->r;
      d.u = lr->u.data();
      d.v = lr->v.data();
    } else {
      d.k = dk->k.data();
    }
    d.variant = static_cast<int>(model.variant);
    d.source_k = k.data();
    d.source_rate = rate.data();
    d.num_sources = k.size();
    d.shatter_rate = model.shatter_rate;
    d.device = device;
    check(agk_rhs_create(&d, &h_), nullptr);
  }
  GpuWorkspace(const GpuWorkspace&) = delete;
  GpuWorkspace& operator=(const GpuWorkspace&) = delete;
  ~GpuWorkspace() { agk_rhs_destroy(h_); }

  std::uint64_t evals() const { return agk_rhs_evals(h_); }
  void reset_evals() { agk_rhs_reset_evals(h_); }
  agk_rhs* handle() const { return h_; }
  std::size_t size() const { return m_; }

 private:
  agk_rhs* h_ = nullptr;
  std::size_t m_;
};

inline void check_sizes(const GpuWorkspace& ws, std::span<const double> n, std::span<double> out) {
  if (n.size() != ws.size() || out.size() != ws.size())
    throw std::invalid_argument("state size does not match model");
}

// eval_rhs (rhs.cpp:212-235); counts one evaluation
inline void eval_rhs(const ModelSpec&, std::span<const double> n, GpuWorkspace& ws, std::span<double> out) {
  check_sizes(ws, n, out);
  check(agk_rhs_eval(ws.handle(), n.data(), out.data(), AGK_MEM_HOST), ws.handle());
}
inline void birth_term(std::span<const double> n, GpuWorkspace& ws, std::span<double> out) {
  check_sizes(ws, n, out);
  check(agk_birth_term(ws.handle(), n.data(), out.data(), AGK_MEM_HOST), ws.handle());
}
inline void death_term(std::span<const double> n, GpuWorkspace& ws, std::span<double> out) {
  check_sizes(ws, n, out);
  check(agk_death_term(ws.handle(), n.data(), out.data(), AGK_MEM_HOST), ws.handle());
}
inline void shattering_terms(std::span<const double> n, double lambda, GpuWorkspace& ws, std::span<double> out) {
  check_sizes(ws, n, out);
  check(agk_shattering_terms(ws.handle(), n.data(), lambda, out.data(), AGK_MEM_HOST), ws.handle());
}
inline double euler_stability_bound(GpuWorkspace& ws, std::span<const double> n, double a) {
  double b = 0.0;
  check(agk_euler_stability_bound(ws.handle(), n.data(), a, &b, AGK_MEM_HOST), ws.handle());
  return b;
}

// advance (steppers.cpp:293-300): the whole trial loop and controller on the device
inline StepOutcome advance(GpuWorkspace& ws, std::span<const double> n, double tau, const StepControl& control) {
  const agk_control c = to_control(control);
  agk_outcome o{};
  std::vector<double> state(n.size());
  check(agk_advance(ws.handle(), n.data(), tau, &c, &o, state.data(), AGK_MEM_HOST), ws.handle());
  StepOutcome res;
  res.tau_used = o.tau_used;
  res.tau_next = o.tau_next;
  res.error_estimate = o.error_estimate;
  res.rejects = o.rejects;
  res.rhs_evals = o.rhs_evals;
  res.status = static_cast<StepStatus>(o.status);
  if (res.status == StepStatus::ok) res.state = std::move(state);
  return res;
}

// RhsFn seam (steppers.hpp:12) so the reference's own CPU steppers can drive the device RHS
// (host copies per call: a parity tool, not the fast path).
inline RhsFn as_rhs_fn(GpuWorkspace& ws) {
  return [&ws](std::span<const double> n, std::span<double> out) {
    check(agk_rhs_eval(ws.handle(), n.data(), out.data(), AGK_MEM_HOST), ws.handle());
  };
}

// run (simulator.cpp:112-229) as one device-resident CUDA graph
inline RunReport run(const SimulationConfig& config, int device = -1) {
  config.validate();
  GpuWorkspace ws(config.model, device);
  const StateVector init = initial_state(config);
  agk_run_desc d{};
  d.control = to_control(config.control);
  d.t_end = config.t_end;
  d.initial = init.n.data();
  d.initial_tau = config.initial_tau;
  d.snapshot_times = config.snapshot_times.data();
  d.num_snapshots = config.snapshot_times.size();
  d.record = static_cast<int>(config.record);
  d.record_interval = config.record_interval;
  const std::size_t m = config.model.m;
  std::vector<double> final_state(m), snaps(config.snapshot_times.size() * m);
  std::vector<agk_record> recs(config.record == RecordMode::none ? 1 : 1 << 16);
  agk_run_report rep{};
  rep.final_state = final_state.data();
  rep.snapshots = snaps.empty() ? nullptr : snaps.data();
  rep.records = config.record == RecordMode::none ? nullptr : recs.data();
  rep.records_capacity = config.record == RecordMode::none ? 0 : recs.size();
  check(agk_run(ws.handle(), &d, &rep), ws.handle());
  RunReport out;
  out.termination = rep.termination == 0 ? Termination::completed : Termination::aborted;
  out.abort_reason = rep.termination == 0 ? "" : describe(static_cast<StepStatus>(rep.abort_status));
  out.abort_t = rep.abort_t;
  out.abort_tau = rep.abort_tau;
  out.total_rhs_evals = rep.total_rhs_evals;
  out.total_accepted = rep.total_accepted;
  out.total_rejects = rep.total_rejects;
  out.wall_seconds = rep.wall_seconds;
  out.final_state.n = std::move(final_state);
  out.final_state.t = rep.final_t;
  for (std::size_t q = 0; q < rep.num_snapshots_taken; ++q)
    out.snapshots.emplace_back(config.snapshot_times[q],
                               std::vector<double>(snaps.begin() + q * m, snaps.begin() + (q + 1) * m));
  const std::size_t nrec = rep.num_records < rep.records_capacity ? rep.num_records : rep.records_capacity;
  for (std::size_t q = 0; q < nrec; ++q) {
    ObservableRecord r;
    r.t = recs[q].t;
    r.tau = recs[q].tau;
    r.density = recs[q].density;
    r.mass = recs[q].mass;
    r.m2 = recs[q].m2;
    r.error_estimate = recs[q].error_estimate;
    r.rhs_evals = recs[q].rhs_evals;
    r.rejects = recs[q].rejects;
    out.records.push_back(r);
  }
  return out;
}

}  // namespace aggkin::gpu
