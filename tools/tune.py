"""Time the config-4 RHS under kernel variants (AGK_VARIANT) and rank-group sizes."""
import itertools, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json
sys.path.insert(0, %r)
import torch, paper_2407_16559_b200 as agk
from paper_2407_16559_b200.configs import random_config4
U, V, n = random_config4()
ws = agk.RhsWorkspace(agk.Model(U, V))
nd = torch.from_numpy(n).cuda(); od = torch.empty_like(nd)
agk.eval_rhs_timed(ws, nd, od, 5)
ms = agk.eval_rhs_timed(ws, nd, od, 30) / 30
prof, plan = agk.profile_rhs(ws, nd, od, 3)
cls = {}
for c, t in prof: cls[c] = cls.get(c, 0) + t
print(json.dumps(dict(ms=ms, cls=cls, plan=plan, chk=float(od.abs().sum()))))
''' % ROOT
variants = sys.argv[1].split(",") if len(sys.argv) > 1 else ["0"]
groups = sys.argv[2].split(",") if len(sys.argv) > 2 else ["1"]
for v, g in itertools.product(variants, groups):
    # AGK_* knobs are read only by the experiments build (make -C paper_2407_16559_b200 exp)
    env = dict(os.environ, AGK_VARIANT=v, AGK_RANK_GROUP=g,
               AGK_LIB=os.path.join(ROOT, "paper_2407_16559_b200", "libagk_b200_exp.so"))
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-500:]
    print(f"variant={v} group={g}: {line}", flush=True)
