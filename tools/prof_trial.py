"""Per-trial device time inside agk.run against the stand-alone RHS time, for BASELINE configs:
python tools/prof_trial.py CONFIG:HORIZON ... [--steppers rkf45,rk4,rk2]
(trial overhead = stage combinations, final pass, controller, snapshot copy, WHILE iteration)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_16559_b200 as agk
from paper_2407_16559_b200.configs import baseline_config
ST = {"rk2": agk.RK2, "rk4": agk.RK4, "rkf45": agk.RKF45}
steppers = "rkf45"
specs = []
for a in sys.argv[1:]:
    if a.startswith("--steppers"):
        steppers = a.split("=")[1]
    else:
        specs.append(a)
for spec in specs or ["5:20"]:
    c, hz = spec.split(":")
    cfg = baseline_config(int(c))
    m = cfg["u"].shape[0]
    ws = agk.RhsWorkspace(agk.Model(cfg["u"], cfg["v"], cfg["variant"], cfg["sources"], cfg["lam"]))
    nd = torch.from_numpy(np.random.default_rng(0).random(m)).cuda(); od = torch.empty_like(nd)
    agk.eval_rhs_timed(ws, nd, od, 5)
    rhs_us = 1e3 * agk.eval_rhs_timed(ws, nd, od, 50) / 50
    for s in steppers.split(","):
        ctl = agk.StepControl(stepper=ST[s], tol=cfg["tol"])
        agk.run(ws, agk.SimulationConfig(ctl, float(hz) / 50, cfg["n0"]))  # instantiate the graph
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = agk.run(ws, agk.SimulationConfig(ctl, float(hz), cfg["n0"]))
        wall = time.perf_counter() - t0
        trials = rep.total_accepted + rep.total_rejects
        print(f"config {c} {s}: rhs {rhs_us:.1f} us; run {wall:.3f} s, {trials} trials, {rep.total_rhs_evals} rhs, "
              f"{1e6 * wall / trials:.1f} us/trial, {1e6 * wall / rep.total_rhs_evals:.1f} us per counted rhs")
    ws.close()
