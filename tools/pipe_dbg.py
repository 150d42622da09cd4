"""One config-4 RHS with AGK_DBG timing switches (per-CTA phase times printed by k_pipe)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_16559_b200 as agk
from paper_2407_16559_b200.configs import baseline_config
cfg = baseline_config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
m = cfg["u"].shape[0]
ws = agk.RhsWorkspace(agk.Model(cfg["u"], cfg["v"], cfg["variant"], cfg["sources"], cfg["lam"]))
nd = torch.from_numpy(np.random.default_rng(0).random(m)).cuda(); od = torch.empty_like(nd)
for _ in range(3):
    agk.eval_rhs(ws, nd.cpu().numpy())
torch.cuda.synchronize()
print("---", flush=True)
t = agk.eval_rhs_timed(ws, nd, od, 4) / 4
torch.cuda.synchronize()
print(f"graph {1e3*t:.1f} us/RHS", flush=True)
