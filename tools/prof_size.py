"""RHS graph time at arbitrary sizes (Brownian + 2 kernel, R = 3 -> R_f = 2, sources):
python tools/prof_size.py M [M ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_16559_b200 as agk
from oracle import oracle as O
out = []
for m in [int(x) for x in sys.argv[1:]]:
    u, v = O.brownian_plus2_factors(m)
    ws = agk.RhsWorkspace(agk.Model(u, v, O.SOURCES, [(1, 1.0)], 0.0))
    nd = torch.from_numpy(np.random.default_rng(0).random(m)).cuda(); od = torch.empty_like(nd)
    agk.eval_rhs_timed(ws, nd, od, 5)
    out.append(f"m={m}: {1e3 * agk.eval_rhs_timed(ws, nd, od, 50) / 50:.1f} us")
    ws.close()
print("; ".join(out))
