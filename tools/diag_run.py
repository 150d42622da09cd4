"""Diagnostic (test infrastructure; uses the oracle): restart comparison of a long adaptive run.
The device integrates CASE to t0; from that state both the device and the CPU oracle (port, pinned
bitwise to the reference) integrate a further dt with every step recorded; prints both
trajectories' statistics (N(t) spread, tau range, accepted/rejects) and the final distances.
  python tools/diag_run.py c5_m4096_rk2 99000 1000"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2407_16559_b200 as agk
from oracle import oracle as O
from tests.golden.make_parity_runs import CASES, CONFIG, STEPPERS
from tests.helpers import factors

name, t0, dt = sys.argv[1], float(sys.argv[2]), float(sys.argv[3])
cfg, m, st, t_end = CASES[name]
kind, variant, sources, lam, init, tol = CONFIG[cfg]
u, v = factors("constant", m) if kind == "constant" else factors("brownian2", m) if kind == "brownian2" else factors("brownian", m, float(kind[8:]))
n0 = np.zeros(m)
if init == "mono":
    n0[0] = 1.0
ws = agk.RhsWorkspace(agk.Model(u, v, variant, list(sources), lam))
ctl = agk.StepControl(stepper=STEPPERS[st], tol=tol)
r0 = agk.run(ws, agk.SimulationConfig(ctl, t0, n0))
x0 = np.array(r0.final_state)
print(f"device to t0={t0}: accepted {r0.total_accepted} rejects {r0.total_rejects} N {x0.sum():.15g}")
rg = agk.run(ws, agk.SimulationConfig(ctl, dt, x0, record=agk.RECORD_EVERY_STEP))
om = O.Model(u, v, variant, list(sources), lam)
ro = O.Oracle("port").run(om, x0, O.Control(stepper=STEPPERS[st], mode=O.ADAPTIVE, tol=tol), dt,
                           record=O.RECORD_EVERY_STEP, records_capacity=2000000)
def stats(tag, recs, acc, rej, fs):
    N = np.array([r["density"] if isinstance(r, dict) else r.density for r in recs])
    tau = np.array([r["tau"] if isinstance(r, dict) else r.tau for r in recs])
    err = np.array([r["error_estimate"] if isinstance(r, dict) else r.error_estimate for r in recs])
    print(f"{tag}: accepted {acc} rejects {rej} records {len(recs)} N final {fs.sum():.15g} "
          f"N range [{N.min():.12g}, {N.max():.12g}] tau range [{tau[1:].min():.4g}, {tau[1:].max():.4g}] median {np.median(tau[1:]):.4g} "
          f"err median {np.median(err[1:]):.3g} max {err[1:].max():.3g}")
    return N, tau
fg = np.array(rg.final_state)
Ng, tg = stats("device", rg.records, rg.total_accepted, rg.total_rejects, fg)
fo = np.array(ro["final_state"])
No, to = stats("oracle", ro["records"], ro["total_accepted"], ro["total_rejects"], fo)
print(f"final N rel diff {abs(fg.sum() - fo.sum()) / fo.sum():.3e}, state normwise {np.max(np.abs(fg - fo)) / np.max(np.abs(fo)):.3e}")
k = min(len(Ng), len(No), 12)
print("first records N (device | oracle), tau:")
for i in range(k):
    print(f"  {Ng[i]:.15g} {tg[i]:.6g} | {No[i]:.15g} {to[i]:.6g}")
