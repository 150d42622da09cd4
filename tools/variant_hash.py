"""SHA-256 of S(n) at BASELINE configs under the current AGK_* knobs (experiments build): variants that
claim the same arithmetic must print the same hashes.  python tools/variant_hash.py [CONFIG ...]"""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_16559_b200 as agk
from paper_2407_16559_b200.configs import baseline_config
out = []
for c in [int(x) for x in sys.argv[1:]] or [4, 5]:
    cfg = baseline_config(c)
    m = cfg["u"].shape[0]
    ws = agk.RhsWorkspace(agk.Model(cfg["u"], cfg["v"], cfg["variant"], cfg["sources"], cfg["lam"]))
    nd = torch.from_numpy(np.random.default_rng(0).random(m)).cuda()
    s = agk.eval_rhs(ws, nd).cpu().numpy()
    out.append(f"c{c}:{hashlib.sha256(s.tobytes()).hexdigest()[:16]}")
    ws.close()
print(" ".join(out))
