"""Timeline of one config-4 (or config-5: argv[1]) RHS in graph mode (AGK_DBG=512 kernel stamps, %globaltimer):
per kernel class the first CTA's arrival, the first CTA's start of work after its
programmatic-dependency wait, and the last CTA's exit, in us from the first arrival."""
import ctypes, os, sys
# AGK_* knobs are read only by the experiments build (make -C paper_2407_16559_b200 exp)
os.environ.setdefault("AGK_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                              "paper_2407_16559_b200", "libagk_b200_exp.so"))
os.environ["AGK_DBG"] = str(int(os.environ.get("AGK_DBG", "0")) | 512)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_16559_b200 as agk
from paper_2407_16559_b200.configs import baseline_config
cfg = baseline_config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)  # a P = 2^21 config: 4 or 5
m = cfg["u"].shape[0]
ws = agk.RhsWorkspace(agk.Model(cfg["u"], cfg["v"], cfg["variant"], cfg["sources"], cfg["lam"]))
n = cfg["n0"] if cfg.get("tol") is None else np.random.default_rng(0).random(m) * np.exp(-np.arange(m) / (m / 8))
nd = torch.from_numpy(np.ascontiguousarray(n)).cuda(); od = torch.empty_like(nd)
lib = agk.load_library()
buf = (ctypes.c_ulonglong * 24)()
names = ["transpose", "col_fwd", "row", "dvec", "col_inv", "dvec(D done)", "aux6", "aux7"]
# mid sizes (four-step kernels): slot 5 = column pass [first CTA scaled its operands | first CTA past its FFT |
# last CTA scaled its operands]; slot 6 = [first row CTA past its inverse FFT | - | last column CTA past its FFT];
# slot 7 = row pass [first CTA has its samples | first CTA past forward FFT + product | last CTA past them]
agk.eval_rhs_timed(ws, nd, od, 5)
for rep in range(3):
    lib.agk_dbg_timeline(buf, 1)
    ms = agk.eval_rhs_timed(ws, nd, od, 1)
    lib.agk_dbg_timeline(buf, 0)
    t = [[int(buf[3 * k + i]) for i in range(3)] for k in range(8)]
    NONE = (0, 2**64 - 1)
    t0 = min(t[k][0] for k in range(5) if t[k][0] not in NONE)
    print(f"rep {rep}: graph {1e3 * ms:.1f} us")
    for k in range(8):
        f = lambda x: "    -  " if x in NONE else f"{(x - t0) / 1e3:7.1f}"
        print(f"  {names[k]:14s} arrive {f(t[k][0])}  start {f(t[k][1])}  end {f(t[k][2])}")
