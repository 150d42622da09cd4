// aggkin_gpu.hpp — drop-in C++ adapter: the reference `aggkin` operator API (rhs.hpp,
// steppers.hpp, simulator.hpp) served by the B200 C ABI (include/agk/agk.h).
//
// A reference maintainer includes this header next to the reference's own headers and links
// libagk_b200.so. The reference's value types are used unchanged (ModelSpec, StepControl,
// StepOutcome, SimulationConfig, RunReport); only the workspace type differs, because the
// device handle owns the factors, scratch and graphs that RhsWorkspace owns on the CPU:
//
//   reference                                        adapter (namespace aggkin::gpu)
//   RhsWorkspace ws;                                 GpuWorkspace ws;
//   eval_rhs(model, n, ws, out)   (rhs.hpp:89)       eval_rhs(model, n, ws, out)
//   birth_term / death_term / shattering_terms       same names and arguments, GpuWorkspace&
//   euler_stability_bound(kernel, n, a) (rhs.hpp:99) same (or (ws, n, a) on a bound workspace)
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
#include <cstring>
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

// Identity of a ModelSpec for the workspace's binding check: sizes, variant, lambda, sources
// and a 64-bit hash of the factor (or dense kernel) bytes. Hashing reads U and V once per call
// (~2 bytes/cycle); that is the price of honouring a per-call model like the reference
// (rhs.hpp:89-90) in this host-copy parity seam. The fast path (agk_advance / agk_run) binds once.
struct ModelFingerprint {
  std::size_t m = 0, r = 0;
  int variant = -1, dense = 0;
  std::uint64_t lambda_bits = 0, hash = 0;
  std::vector<std::pair<std::size_t, double>> sources;
  bool operator==(const ModelFingerprint&) const = default;

  static std::uint64_t mix(std::uint64_t h, const double* p, std::size_t n) {
    const auto* w = reinterpret_cast<const std::uint64_t*>(p);
    std::uint64_t a = h ^ 0x9e3779b97f4a7c15ull, b = h + n, c = ~h, d = h * 31;
    std::size_t i = 0;
    for (; i + 4 <= n; i += 4) {  // four independent lanes
      a = (a ^ w[i]) * 0x100000001b3ull;
      b = (b ^ w[i + 1]) * 0x100000001b3ull;
      c = (c ^ w[i + 2]) * 0x100000001b3ull;
      d = (d ^ w[i + 3]) * 0x100000001b3ull;
    }
    for (; i < n; ++i) a = (a ^ w[i]) * 0x100000001b3ull;
    return a ^ (b << 1) ^ (c << 2) ^ (d << 3) ^ (a >> 29) ^ (b >> 31);
  }
  static ModelFingerprint of(const ModelSpec& model) {
    ModelFingerprint f = of_kernel(model.kernel, model.m);
    f.variant = static_cast<int>(model.variant);
    std::memcpy(&f.lambda_bits, &model.shatter_rate, sizeof(double));
    for (const auto& [k, rate] : model.sources.rates) f.sources.emplace_back(k, rate);
    return f;
  }
  static ModelFingerprint of_kernel(const KernelRep& kernel, std::size_t m) {
    ModelFingerprint f;
    f.m = m;
    if (const auto* lr = std::get_if<LowRankFactors>(&kernel)) {
      f.r = lr->r;
      f.hash = mix(mix(1, lr->u.data(), lr->u.size()), lr->v.data(), lr->v.size());
    } else if (const auto* dk = std::get_if<DenseKernel>(&kernel)) {
      f.dense = 1;
      f.hash = mix(2, dk->k.data(), dk->k.size());
    }
    return f;
  }
  bool same_kernel(const ModelFingerprint& o) const { return m == o.m && r == o.r && dense == o.dense && hash == o.hash; }
};

// RhsWorkspace (rhs.hpp:45-70) on the device: the handle holds the model's device copy, its
// scratch and graphs. Like the reference workspace it is model-agnostic at the API: every call
// takes a ModelSpec, and a call with a model other than the bound one rebinds the handle (the
// reference re-prepares only on a size change, rhs.cpp:74-85; here the factors live on the
// device, so any model change re-uploads them). One per concurrent caller (rhs.hpp:42-44).
class GpuWorkspace {
 public:
  explicit GpuWorkspace(int device = -1) : device_(device) {}
  explicit GpuWorkspace(const ModelSpec& model, int device = -1) : device_(device) { bind(model); }
  GpuWorkspace(const GpuWorkspace&) = delete;
  GpuWorkspace& operator=(const GpuWorkspace&) = delete;
  ~GpuWorkspace() { agk_rhs_destroy(h_); }

  // RhsWorkspace::evals / reset_evals: the count survives rebinding
  std::uint64_t evals() const { return evals_base_ + (h_ ? agk_rhs_evals(h_) : 0); }
  void reset_evals() {
    evals_base_ = 0;
    if (h_) agk_rhs_reset_evals(h_);
  }
  agk_rhs* handle() const { return h_; }
  std::size_t size() const { return m_; }

  // Handle for a term function of `kernel` (birth_term, death_term, shattering_terms and the
  // Euler bound take a KernelRep, rhs.hpp:75-99): any binding with the same kernel serves, since
  // the term selection and lambda are per call.
  agk_rhs* bind_kernel(const KernelRep& kernel, std::size_t m) {
    if (h_ && ModelFingerprint::of_kernel(kernel, m).same_kernel(fp_)) return h_;
    ModelSpec model;
    model.m = m;
    model.kernel = kernel;
    return bind(model);
  }

  // Handle for `model`: the bound one if the fingerprint matches, else a fresh binding.
  agk_rhs* bind(const ModelSpec& model) {
    model.validate();
    ModelFingerprint f = ModelFingerprint::of(model);
    if (h_ && f == fp_) return h_;
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
    d.device = device_;
    agk_rhs* nh = nullptr;
    check(agk_rhs_create(&d, &nh), nullptr);
    if (h_) {
      evals_base_ += agk_rhs_evals(h_);
      agk_rhs_destroy(h_);
    }
    h_ = nh;
    m_ = model.m;
    fp_ = std::move(f);
    return h_;
  }

 private:
  agk_rhs* h_ = nullptr;
  std::size_t m_ = 0;
  int device_ = -1;
  std::uint64_t evals_base_ = 0;
  ModelFingerprint fp_;
};

inline void check_sizes(const GpuWorkspace& ws, std::span<const double> n, std::span<double> out) {
  if (n.size() != ws.size() || out.size() != ws.size())
    throw std::invalid_argument("state size does not match model");
}

// eval_rhs (rhs.cpp:212-235; rhs.hpp:89-90): the model is a per-call argument, as in the
// reference; counts one evaluation on the workspace
inline void eval_rhs(const ModelSpec& model, std::span<const double> n, GpuWorkspace& ws, std::span<double> out) {
  agk_rhs* h = ws.bind(model);
  check_sizes(ws, n, out);
  check(agk_rhs_eval(h, n.data(), out.data(), AGK_MEM_HOST), h);
}
// birth_term / death_term / shattering_terms (rhs.hpp:75-86): the reference signatures, a
// per-call KernelRep; these do not count evaluations, like the reference
inline void birth_term(const KernelRep& kernel, std::span<const double> n, GpuWorkspace& ws, std::span<double> out) {
  agk_rhs* h = ws.bind_kernel(kernel, n.size());
  check_sizes(ws, n, out);
  check(agk_birth_term(h, n.data(), out.data(), AGK_MEM_HOST), h);
}
inline void death_term(const KernelRep& kernel, std::span<const double> n, GpuWorkspace& ws, std::span<double> out) {
  agk_rhs* h = ws.bind_kernel(kernel, n.size());
  check_sizes(ws, n, out);
  check(agk_death_term(h, n.data(), out.data(), AGK_MEM_HOST), h);
}
inline void shattering_terms(const KernelRep& kernel, std::span<const double> n, double lambda, GpuWorkspace& ws,
                             std::span<double> out) {
  agk_rhs* h = ws.bind_kernel(kernel, n.size());
  check_sizes(ws, n, out);
  check(agk_shattering_terms(h, n.data(), lambda, out.data(), AGK_MEM_HOST), h);
}
// euler_stability_bound (rhs.hpp:99): the reference signature takes no workspace; the device
// needs one, so the calling thread keeps one (rebound when the kernel changes)
inline double euler_stability_bound(const KernelRep& kernel, std::span<const double> n, double a) {
  thread_local GpuWorkspace ws;
  agk_rhs* h = ws.bind_kernel(kernel, n.size());
  double b = 0.0;
  check(agk_euler_stability_bound(h, n.data(), a, &b, AGK_MEM_HOST), h);
  return b;
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
  RunReport out;
  agk_run_report rep{};
  rep.final_state = final_state.data();
  rep.snapshots = snaps.empty() ? nullptr : snaps.data();
  // every record, streamed from the device's record ring (simulator.cpp:130-145, 209-222)
  rep.record_sink = [](void* user, const agk_record* recs, std::size_t n) {
    auto& v = *static_cast<std::vector<ObservableRecord>*>(user);
    for (std::size_t q = 0; q < n; ++q) {
      ObservableRecord r;
      r.t = recs[q].t;
      r.tau = recs[q].tau;
      r.density = recs[q].density;
      r.mass = recs[q].mass;
      r.m2 = recs[q].m2;
      r.error_estimate = recs[q].error_estimate;
      r.rhs_evals = recs[q].rhs_evals;
      r.rejects = recs[q].rejects;
      v.push_back(r);
    }
  };
  rep.sink_user = &out.records;
  check(agk_run(ws.handle(), &d, &rep), ws.handle());
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
  if (out.records.size() != rep.num_records) throw std::runtime_error("agk: record stream incomplete");
  return out;
}

}  // namespace aggkin::gpu
