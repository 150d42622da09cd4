"""Evaluate the config-4 RHS a few times (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_16559_b200 as agk
from paper_2407_16559_b200.configs import random_config4
m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
r = int(sys.argv[2]) if len(sys.argv) > 2 else 16
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
U, V, n = random_config4(m, r)
ws = agk.RhsWorkspace(agk.Model(U, V))
nd = torch.from_numpy(n).cuda()
od = torch.empty_like(nd)
for _ in range(reps):
    agk._check(agk.load_library().agk_rhs_eval_async(ws.handle, nd.data_ptr(), od.data_ptr()), ws.handle)
torch.cuda.synchronize()
print("ok", float(od.sum()))
