"""Adaptive solve measurements for BASELINE configs 1-5 (time to t_end on the device).

For each config: per-RHS device time (CUDA events, captured graph), then agk.run to a horizon
(the full t_end where it finishes in the time budget, else a prefix), reporting wall time,
accepted steps, rejects, RHS evals, device-time per RHS inside the run, and the CPU oracle's
per-RHS time for the extrapolated CPU time-to-t_end (SURVEY §8d parity plan).
Usage: python tools/runs.py [config ...] [--horizon c:t ...] [--cpu]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2407_16559_b200 as agk  # noqa: E402
from paper_2407_16559_b200.configs import baseline_config  # noqa: E402

STEPPERS = {"rk2": agk.RK2, "rk4": agk.RK4, "rkf45": agk.RKF45}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", type=int, default=[1, 2, 3, 5])
    ap.add_argument("--horizon", nargs="*", default=[])
    ap.add_argument("--steppers", default="rkf45")
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "runs.json"))
    args = ap.parse_args()
    horizons = {int(h.split(":")[0]): float(h.split(":")[1]) for h in args.horizon}
    results = []
    for c in args.configs:
        cfg = baseline_config(c)
        m = cfg["u"].shape[0]
        ws = agk.RhsWorkspace(agk.Model(cfg["u"], cfg["v"], cfg["variant"], cfg["sources"], cfg["lam"]))
        nd = torch.from_numpy(np.random.default_rng(0).random(m) * np.exp(-np.arange(m) / (m / 8))).cuda()
        od = torch.empty_like(nd)
        agk.eval_rhs_timed(ws, nd, od, 5)
        rhs_ms = agk.eval_rhs_timed(ws, nd, od, 50) / 50
        cpu_rhs_s = None
        if args.cpu:
            from oracle.oracle import Model, Oracle
            o = Oracle("reference") if os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libaggkin_ref.so")) else Oracle("port")
            om = Model(cfg["u"], cfg["v"], cfg["variant"], cfg["sources"], cfg["lam"])
            reps = 3 if m >= (1 << 16) else 20
            t0 = time.perf_counter()
            for _ in range(reps):
                o.eval_rhs(om, nd.cpu().numpy())
            cpu_rhs_s = (time.perf_counter() - t0) / reps
        for sname in args.steppers.split(","):
            t_end = horizons.get(c, cfg["t_end"])
            ctl = agk.StepControl(stepper=STEPPERS[sname], tol=cfg["tol"])
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep = agk.run(ws, agk.SimulationConfig(ctl, t_end, cfg["n0"]))
            wall = time.perf_counter() - t0
            fs = rep.final_state
            r = dict(config=c, m=m, r=cfg["u"].shape[1], unique_ranks=ws.unique_ranks(), stepper=sname,
                     tol=cfg["tol"], t_end_full=cfg["t_end"], horizon=t_end, complete=t_end == cfg["t_end"],
                     termination=rep.termination, final_t=rep.final_t, wall_s=wall,
                     accepted=rep.total_accepted, rejects=rep.total_rejects, rhs_evals=rep.total_rhs_evals,
                     accepted_per_s=rep.total_accepted / wall, us_per_rhs_in_run=1e6 * wall / max(rep.total_rhs_evals, 1),
                     rhs_graph_us=1e3 * rhs_ms, N=float(fs.sum()), M1=float(np.dot(np.arange(1, m + 1), fs)),
                     cpu_rhs_s=cpu_rhs_s,
                     cpu_time_to_horizon_extrapolated_s=(cpu_rhs_s * rep.total_rhs_evals) if cpu_rhs_s else None)
            print(json.dumps(r), flush=True)
            results.append(r)
        ws.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(results, f, indent=1)


if __name__ == "__main__":
    main()
