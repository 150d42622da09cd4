"""Bitwise check of fused RK stages (experiments build): prints a hash of rk_step / advance
outputs for several shapes; run with AGK_FUSE_STAGES=1 and =0 and compare the lines."""
import hashlib, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("AGK_LIB", os.path.join(ROOT, "paper_2407_16559_b200", "libagk_b200_exp.so"))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import paper_2407_16559_b200 as agk  # noqa: E402
from tests.helpers import factors  # noqa: E402

def h(x):
    return hashlib.sha1(np.ascontiguousarray(x).tobytes()).hexdigest()[:12]

for m in (1000, 4096, 1 << 16, 1 << 20):
    u, v = factors("brownian2", m)
    ws = agk.RhsWorkspace(agk.Model(u, v, agk.AGGREGATION_SOURCES, [(1, 1.0)], 0.0))
    n = np.random.default_rng(m).random(m) * np.exp(-np.arange(m) / (m / 8))
    out = [f"m={m}"]
    for st in (agk.RK2, agk.RK4, agk.RKF45):
        o, o5, e = agk._rk(ws, st, n, 0.01, want5=(st == agk.RKF45))
        out.append(f"{st}:{h(o)}")
        if m == 4096:
            np.save(os.path.join(ROOT, "gpurun_out", f"fc_{os.environ.get('AGK_FUSE_STAGES')}_{st}.npy"), o)
    if m == 4096:
        k = agk.eval_rhs(ws, n)
        np.save(os.path.join(ROOT, "gpurun_out", f"fc_{os.environ.get('AGK_FUSE_STAGES')}_rhs.npy"), k)
    r = agk.advance(ws, n, 0.5, agk.StepControl(stepper=agk.RK2, tol=1e-6))
    out.append(f"adv:{h(r.state)}:{r.rejects}")
    print(" ".join(out), flush=True)
    ws.close()
