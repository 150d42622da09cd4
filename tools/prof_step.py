"""A few adaptive RKF45 trials of BASELINE config 5 (M = 2^20) through agk.run, for ncu launch lists
of the stepping kernels (stage combinations, controller) next to the RHS kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_16559_b200 as agk
from paper_2407_16559_b200.configs import baseline_config
cfg = baseline_config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
ws = agk.RhsWorkspace(agk.Model(cfg["u"], cfg["v"], cfg["variant"], cfg["sources"], cfg["lam"]))
ctl = agk.StepControl(stepper=agk.RKF45, tol=cfg["tol"])
rep = agk.run(ws, agk.SimulationConfig(ctl, float(sys.argv[2]) if len(sys.argv) > 2 else 0.05, cfg["n0"]))
torch.cuda.synchronize()
print("ok", rep.total_accepted, rep.total_rejects, rep.total_rhs_evals)
