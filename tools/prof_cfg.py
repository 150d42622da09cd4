"""Per-launch device times of one RHS for a BASELINE config (event markers between kernels)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_16559_b200 as agk
from paper_2407_16559_b200.configs import baseline_config
for c in [int(x) for x in sys.argv[1:]] or [1, 2, 3, 4, 5]:
    cfg = baseline_config(c)
    m = cfg["u"].shape[0]
    ws = agk.RhsWorkspace(agk.Model(cfg["u"], cfg["v"], cfg["variant"], cfg["sources"], cfg["lam"]))
    nd = torch.from_numpy(np.random.default_rng(0).random(m)).cuda(); od = torch.empty_like(nd)
    agk.eval_rhs_timed(ws, nd, od, 5)
    g = agk.eval_rhs_timed(ws, nd, od, 50) / 50
    prof, plan = agk.profile_rhs(ws, nd, od, 10)
    print(f"config {c}: graph {1e3*g:.1f} us/RHS, plan {plan}, launches " + ", ".join(f"{k}:{1e3*t:.1f}" for k, t in prof))
    ws.close()
