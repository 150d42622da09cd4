"""A few RHS evaluations of one BASELINE config (a short command for ncu):
python tools/prof_one.py CONFIG [REPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_16559_b200 as agk  # noqa: E402
from paper_2407_16559_b200.configs import baseline_config  # noqa: E402

c = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = baseline_config(c)
m = cfg["u"].shape[0]
ws = agk.RhsWorkspace(agk.Model(cfg["u"], cfg["v"], cfg["variant"], cfg["sources"], cfg["lam"]))
nd = torch.from_numpy(np.random.default_rng(0).random(m)).cuda()
od = torch.empty_like(nd)
for _ in range(reps):
    agk.eval_rhs(ws, nd)
torch.cuda.synchronize()
print("ok", float(agk.eval_rhs(ws, nd).abs().sum()))
