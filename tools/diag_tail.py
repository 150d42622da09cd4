"""Diagnostic: the last accepted steps of a long device run (every step recorded): where in the
controller's accept/reject cycle the run ends. A final N off the steady value by ~1e-6 right after
a large step, back to it a few steps later, is the wander tests/test_gpu_parity_runs.py measures on
the reference's own trajectory (CASE__fluct.npz).   python tools/diag_tail.py c5_m4096_rk2"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2407_16559_b200 as agk
from tests.golden.make_parity_runs import CASES, CONFIG, STEPPERS
from tests.helpers import factors

name = sys.argv[1]
cfg, m, st, t_end = CASES[name]
kind, variant, sources, lam, init, tol = CONFIG[cfg]
u, v = factors("brownian2", m) if kind == "brownian2" else factors("constant", m)
n0 = np.zeros(m)
if init == "mono":
    n0[0] = 1.0
ws = agk.RhsWorkspace(agk.Model(u, v, variant, list(sources), lam))
rep = agk.run(ws, agk.SimulationConfig(agk.StepControl(stepper=STEPPERS[st], tol=tol), t_end, n0,
                                       record=agk.RECORD_EVERY_STEP))
recs = rep.records
N = np.array([r["density"] for r in recs])
tau = np.array([r["tau"] for r in recs])
print(f"{name}: accepted {rep.total_accepted} rejects {rep.total_rejects} records {len(recs)} final N {N[-1]:.15g}")
print(f"median N over the last 2000 records {np.median(N[-2000:]):.15g}; min {N[-2000:].min():.12g} max {N[-2000:].max():.12g}")
ref = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "parity", f"{name}__ref.npz"))
print(f"reference final N {float(ref['N']):.15g}; device final - reference {abs(N[-1] - float(ref['N'])) / float(ref['N']):.3e}; "
      f"device median - reference {abs(np.median(N[-2000:]) - float(ref['N'])) / float(ref['N']):.3e}")
print("last 14 records: t, tau, N, (N - median)/median")
med = np.median(N[-2000:])
for r in recs[-14:]:
    print(f"  {r['t']:.6f} {r['tau']:.6g} {r['density']:.15g} {(r['density'] - med) / med:+.2e}")
