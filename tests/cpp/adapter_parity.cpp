// adapter_parity.cpp — the drop-in check: the reference's own C++ API (compiled from its sources)
// side by side with adapter/aggkin_gpu.hpp over the B200 C ABI, in one process.
// Built by tests/cpp/Makefile into build/adapter_parity; run by tests/test_gpu_adapter.py.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "aggkin_gpu.hpp"
#include "aggkin/kernels.hpp"

using namespace aggkin;

static int failures = 0;
static void expect(bool ok, const char* what, double a = 0, double b = 0) {
  std::printf("%s %s (%.6g vs %.6g)\n", ok ? "PASS" : "FAIL", what, a, b);
  if (!ok) ++failures;
}

static double rel_max_diff(std::span<const double> got, std::span<const double> want) {
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < got.size(); ++i) {
    num = std::max(num, std::abs(got[i] - want[i]));
    den = std::max(den, std::abs(want[i]));
  }
  return den > 0.0 ? num / den : num;
}

static ModelSpec make_model(ModelVariant variant, const KernelSpec& spec, std::size_t m) {
  ModelSpec model;
  model.variant = variant;
  model.m = m;
  model.kernel = build_factors(spec, m);
  if (variant == ModelVariant::aggregation_sources) model.sources.rates = {{1, 1.0}, {std::min<std::size_t>(m, 100), 0.1}};
  if (variant == ModelVariant::aggregation_shattering) model.shatter_rate = 0.01;
  return model;
}

int main() {
  std::mt19937_64 rng(0x5eed5eed);
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  const KernelSpec specs[] = {{KernelVariant::constant, 0.0, {}},
                              {KernelVariant::generalized_brownian, 1.0 / 3.0, {}},
                              {KernelVariant::generalized_brownian, 0.95, {}}};
  // 1. eval_rhs: reference vs adapter, every variant, small and four-step sizes
  double worst = 0.0;
  for (std::size_t m : {std::size_t{16}, std::size_t{1000}, std::size_t{5000}, std::size_t{1} << 16}) {
    for (const auto& spec : specs) {
      // at m = 2^16 the alpha = 0.95 kernel spans ~9 decades and the reference's own packed-FFT
      // rounding reaches ~5e-12 (tests/test_gpu_rhs.py checks that case against the exact RHS)
      if (m > 5000 && spec.alpha > 0.5) continue;
      for (auto variant : {ModelVariant::aggregation, ModelVariant::aggregation_sources,
                           ModelVariant::aggregation_shattering}) {
        const ModelSpec model = make_model(variant, spec, m);
        RhsWorkspace cpu_ws;
        gpu::GpuWorkspace gpu_ws(model);
        std::vector<double> n(m), a(m), b(m);
        for (double& x : n) x = uni(rng);
        eval_rhs(model, n, cpu_ws, a);
        gpu::eval_rhs(model, n, gpu_ws, b);
        worst = std::max(worst, rel_max_diff(b, a));
        if (gpu_ws.evals() != 1) ++failures;
      }
    }
  }
  expect(worst <= 1e-11, "eval_rhs adapter vs reference, max normwise", worst, 1e-11);

  // 2. advance: the device controller vs the reference controller on the reference RHS
  {
    const ModelSpec model = make_model(ModelVariant::aggregation_shattering, specs[2], 256);
    RhsWorkspace cpu_ws;
    const RhsFn rhs = [&](std::span<const double> in, std::span<double> out) { eval_rhs(model, in, cpu_ws, out); };
    gpu::GpuWorkspace gws(model);
    std::vector<double> n(256);
    for (double& x : n) x = uni(rng);
    for (auto kind : {StepperKind::rk2, StepperKind::rk4, StepperKind::rkf45}) {
      StepControl c;
      c.stepper = kind;
      c.tol = 1e-8;
      StepperWorkspace sw;
      const StepOutcome want = advance(rhs, n, 0.5, c, sw);
      const StepOutcome got = gpu::advance(gws, n, 0.5, c);
      expect(got.status == want.status && got.rejects == want.rejects && got.rhs_evals == want.rhs_evals,
             "advance: status / rejects / evals identical", got.rejects, want.rejects);
      expect(std::abs(got.tau_used - want.tau_used) <= 1e-8 * want.tau_used, "advance: tau_used", got.tau_used,
             want.tau_used);
      expect(rel_max_diff(got.state, want.state) <= 1e-8, "advance: state", rel_max_diff(got.state, want.state), 1e-8);
    }
  }

  // 3. run: device-resident loop vs reference run on the reference's committed config
  //    (proj/configs/aggregation_small.cfg -> out/aggregation_small/summary.txt: 1572/128/3)
  {
    SimulationConfig cfg;
    cfg.model = make_model(ModelVariant::aggregation, specs[0], 256);
    cfg.control.stepper = StepperKind::rk4;
    cfg.control.tol = 1e-8;
    cfg.t_end = 10.0;
    cfg.snapshot_times = {1.0, 10.0};
    cfg.record = RecordMode::every_step;
    const RunReport want = run(cfg);
    const RunReport got = gpu::run(cfg);
    expect(got.total_rhs_evals == 1572 && got.total_accepted == 128 && got.total_rejects == 3,
           "run: aggregation_small golden counts", (double)got.total_accepted, 128.0);
    expect(got.records.size() == want.records.size(), "run: record count", (double)got.records.size(),
           (double)want.records.size());
    expect(got.snapshots.size() == 2 && got.snapshots[1].first == 10.0, "run: snapshots land exactly",
           (double)got.snapshots.size(), 2.0);
    expect(rel_max_diff(got.final_state.n, want.final_state.n) <= 1e-10, "run: final state",
           rel_max_diff(got.final_state.n, want.final_state.n), 1e-10);
  }

  // 4. the RhsFn seam: the reference's own CPU steppers driving the device RHS
  {
    const ModelSpec model = make_model(ModelVariant::aggregation_sources, specs[1], 2000);
    RhsWorkspace cpu_ws;
    gpu::GpuWorkspace gws(model);
    const RhsFn cpu_rhs = [&](std::span<const double> in, std::span<double> out) { eval_rhs(model, in, cpu_ws, out); };
    const RhsFn gpu_rhs = gpu::as_rhs_fn(gws);
    std::vector<double> n(2000, 0.0);
    StepControl c;
    c.tol = 1e-7;
    StepperWorkspace s1, s2;
    const StepOutcome a = advance(cpu_rhs, n, 0.1, c, s1);
    const StepOutcome b = advance(gpu_rhs, n, 0.1, c, s2);
    expect(a.rejects == b.rejects && rel_max_diff(b.state, a.state) <= 1e-10, "RhsFn seam: reference steppers on the device RHS",
           rel_max_diff(b.state, a.state), 1e-10);
  }
  // 5. one workspace, two models (rhs.hpp:89-90: the model is a per-call argument): the
  //    workspace rebinds on a model change and the eval counter carries over
  {
    const std::size_t m = 3000;
    const ModelSpec a = make_model(ModelVariant::aggregation, specs[1], m);
    const ModelSpec b = make_model(ModelVariant::aggregation_shattering, specs[2], m);
    RhsWorkspace cpu_ws;
    gpu::GpuWorkspace gws;
    std::vector<double> n(m), want(m), got(m);
    for (double& x : n) x = uni(rng);
    double worst2 = 0.0;
    for (const ModelSpec* model : {&a, &b, &a, &b}) {
      eval_rhs(*model, n, cpu_ws, want);
      gpu::eval_rhs(*model, n, gws, got);
      worst2 = std::max(worst2, rel_max_diff(got, want));
    }
    expect(worst2 <= 1e-11, "two models through one workspace: eval_rhs follows the model argument", worst2, 1e-11);
    expect(gws.evals() == 4 && cpu_ws.evals() == 4, "two models: eval counter carries over rebinding",
           (double)gws.evals(), 4.0);
    std::vector<double> wt(m), gt(m);
    death_term(b.kernel, n, cpu_ws, wt);
    gpu::death_term(b.kernel, n, gws, gt);
    const double d1 = rel_max_diff(gt, wt);
    birth_term(a.kernel, n, cpu_ws, wt);
    gpu::birth_term(a.kernel, n, gws, gt);
    const double d2 = rel_max_diff(gt, wt);
    shattering_terms(b.kernel, n, 0.02, cpu_ws, wt);
    gpu::shattering_terms(b.kernel, n, 0.02, gws, gt);
    const double d3 = rel_max_diff(gt, wt);
    expect(std::max({d1, d2, d3}) <= 1e-11, "two models: term functions follow the kernel argument",
           std::max({d1, d2, d3}), 1e-11);
    const double eb_want = euler_stability_bound(b.kernel, n, 0.25), eb_got = gpu::euler_stability_bound(b.kernel, n, 0.25);
    expect(std::abs(eb_got - eb_want) <= 1e-12 * eb_want, "euler_stability_bound with the reference signature",
           eb_got, eb_want);
  }

  // 6. run with more records than the device ring holds (1 << 16): every record comes back
  //    (simulator.cpp:130-145, 209-222)
  {
    SimulationConfig cfg;
    cfg.model = make_model(ModelVariant::aggregation, specs[0], 64);
    cfg.control.stepper = StepperKind::rk2;
    cfg.control.mode = StepMode::fixed;
    cfg.control.tau = 1e-3;
    cfg.t_end = 150.0;
    cfg.snapshot_times = {75.0};
    cfg.record = RecordMode::every_step;
    const RunReport want = run(cfg);
    const RunReport got = gpu::run(cfg);
    bool same = got.records.size() == want.records.size();
    double dt = 0.0, dd = 0.0;
    for (std::size_t q = 0; same && q < want.records.size(); ++q) {
      same = got.records[q].rhs_evals == want.records[q].rhs_evals && got.records[q].rejects == want.records[q].rejects;
      dt = std::max(dt, std::abs(got.records[q].t - want.records[q].t) / std::max(1.0, want.records[q].t));
      dd = std::max(dd, std::abs(got.records[q].density - want.records[q].density) / want.records[q].density);
    }
    expect(want.records.size() > 100000 && same, "run: > 65536 records, counts identical record by record",
           (double)got.records.size(), (double)want.records.size());
    expect(dt <= 1e-12 && dd <= 1e-9, "run: long record stream t and density", dt, dd);
    expect(got.total_accepted == want.total_accepted && got.snapshots.size() == 1, "run: long run counters",
           (double)got.total_accepted, (double)want.total_accepted);
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
