"""Why a steady state held at the controller's stability limit cannot be pinned to 1e-8 at t_end
(CPU only, the reference against itself): config 5 at M = 4096 with RK2 step doubling, restarted
from the reference's own final state at t = 1e5 and run to 8 nearby horizons. The run loop
(simulator.cpp:170-217) shortens the last step to land on t_end, so the run ends wherever the
accept/reject cycle happens to be; right after one of the cycle's large steps N is off its steady
value by up to ~1e-6 and relaxes back within a few steps. tests/test_gpu_parity_runs.py therefore
holds the final values of these cases to the reference trajectory's own band (CASE__fluct.npz)."""
import os

import numpy as np

from oracle import oracle as O
from tests.golden.make_parity_runs import CASES, case_inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden", "parity")


def test_reference_final_value_depends_on_landing_phase():
    name = "c5_m4096_rk2"
    z = np.load(os.path.join(GOLD, f"{name}__ref.npz"))
    m = CASES[name][1]
    x0 = np.zeros(m)
    head = np.asarray(z["head"], dtype=np.float64)
    x0[: head.size] = head
    md, _, ctl, _ = case_inputs(name)
    try:
        o = O.Oracle("reference")
    except FileNotFoundError:
        o = O.Oracle("port")  # pinned bitwise to the reference (tests/test_oracle_pin.py)
    finals = np.array([o.run(md, x0, ctl, 100.0 + 0.137 * k)["final_state"].sum() for k in range(8)])
    spread = (finals.max() - finals.min()) / finals.mean()
    # measured 9.5e-7 over these horizons (N = 0.648094965 at t_end = 100.959, 0.64809558 elsewhere)
    assert spread > 1e-7, finals
    # ... while most horizons end on the steady value to 1e-8
    med = np.median(finals)
    assert np.sum(np.abs(finals - med) / med < 2e-8) >= 3, finals
