"""The Python front end (paper_2407_16559_b200/aggkin.py): a drop-in mirror
of the reference's ``aggkin`` module (python/bindings.cpp:128-241) over the device path.

CPU (pinned to the reference itself, tests/golden/config_cases.json from oracle/_ref):
  * parse_config_text -> serialize_config byte for byte, and every error message verbatim
    (config.cpp:131-438);
  * kernel_entry (kernels.cpp:36-57), fit_power_law / fit_cutoff (analysis.cpp:12-75);
  * build_factors / build_dense / initial_state restated from kernels.cpp / simulator.cpp.
GPU: the reference's own smoke checks (tests/python/test_smoke.py) through this module, and
run_text against the CPU oracle running the identical model (counts exact, state 1e-9).
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_16559_b200 import aggkin as A
from tests.helpers import rel_max_diff

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(open(os.path.join(HERE, "golden", "config_cases.json")))
VARIANT_NAMES = {0: "constant", 1: "brownian", 2: "free_molecular"}


@pytest.mark.parametrize("case", CASES["configs"], ids=lambda c: c["out"][:40])
def test_config_parse_matches_reference(case):
    if case["rc"] == 0:
        assert A.serialize_config(A.parse_config_text(case["text"])) == case["out"]
    else:
        with pytest.raises(A.ConfigError) as e:
            A.parse_config_text(case["text"])
        assert str(e.value) == case["out"]


def test_serialize_round_trip():
    for case in CASES["configs"]:
        if case["rc"] == 0:
            again = A.serialize_config(A.parse_config_text(case["out"]))
            assert again == case["out"]


def test_kernel_entry_matches_reference():
    for e in CASES["kernel_entries"]:
        got = A.kernel_entry(VARIANT_NAMES[e["variant"]], e["i"], e["j"], alpha=e["alpha"])
        assert got == e["value"], e


def test_kernel_entry_errors():
    with pytest.raises(ValueError):
        A.kernel_entry("constant", 0, 1)
    with pytest.raises(ValueError):
        A.kernel_entry("brownian", 1, 2, alpha=-1.0)
    with pytest.raises(ValueError):
        A.kernel_entry("linear", 1, 2)
    with pytest.raises(ValueError):
        A.kernel_entry("factors", 1, 2)


def test_fits_match_reference():
    k = np.arange(1, 2049, dtype=np.float64)
    rng = np.random.Generator(np.random.MT19937(7))
    series = [k ** -1.5, k ** -1.5 * np.exp(-1e-4 * k), k ** -2.2 * rng.uniform(0.9, 1.1, k.size)]
    series[2][100:140] = 0.0
    for f in CASES["fits"]:
        n = series[f["series"]]
        fn = (lambda: A.fit_cutoff(n, f["lam"], f["k_lo"], f["k_hi"])) if f["cutoff"] else \
            (lambda: A.fit_power_law(n, f["k_lo"], f["k_hi"]))
        r = fn()
        got = [r["beta"], r["k_lo"], r["k_hi"], r["residual_rms"], r["points_used"], r["points_excluded"]]
        assert got == f["res"], f


def test_fit_errors():
    with pytest.raises(ValueError):
        A.fit_power_law(np.ones(10), 5, 5)
    with pytest.raises(ValueError):
        A.fit_power_law(np.zeros(100), 1, 100)
    with pytest.raises(ValueError):
        A.fit_cutoff(np.ones(100), -1.0, 1, 100)


def test_builders_match_oracle_restatement():
    # libm pow per size, as kernels.cpp:74-85 (the entries equal kernel_entry's, pinned above)
    u, v = A.build_factors("brownian", 300, alpha=0.95)
    assert np.array_equal(u[:, 0], [math.pow(float(i), 0.95) for i in range(1, 301)])
    assert np.array_equal(u[:, 1], 1.0 / u[:, 0]) and np.array_equal(v, u.T[::-1])
    ou, ov = O.brownian_factors(300, 0.95)
    assert rel_max_diff(u, ou) <= 1e-15
    d = A.build_dense("free_molecular", 120)
    assert all(d[i - 1, j - 1] == A.kernel_entry("free_molecular", i, j) for i in (1, 7, 100) for j in (1, 2, 120))
    assert rel_max_diff(d, O.free_molecular_dense(120)) <= 1e-15
    d = A.build_dense("brownian", 50, alpha=1 / 3)
    assert np.array_equal(d, d.T)
    with pytest.raises(ValueError):
        A.build_factors("free_molecular", 10)
    with pytest.raises(ValueError):
        A.build_dense("constant", A.DENSE_SIZE_LIMIT + 1)


def test_initial_states():
    cfg = A.parse_config_text("model = aggregation\nkernel = constant\nm = 32\nstepper = rk2\nmode = fixed\n"
                              "tau = 0.1\nt_end = 1\ninitial = exponential\ninitial_scale = 4\n")
    n = A.initial_state(cfg)
    assert abs(float(np.dot(np.arange(1, 33), n)) - 1.0) < 1e-14  # unit mass (simulator.cpp:78-88)
    cfg.initial = A.MONODISPERSE
    n = A.initial_state(cfg)
    assert n[0] == 1.0 and n[1:].sum() == 0.0


def test_moments_and_oscillations_host():
    assert A.moments(np.array([0.0, 1.0, 0.0])) == (1.0, 2.0, 4.0)
    t = np.arange(0, 50.0001, 0.01)
    s = A.detect_oscillations(t, 1 + 0.1 * np.sin(t))
    assert s["cycle_count"] == 7
    assert np.allclose(s["periods"], 2 * math.pi, atol=0.05)


# ------------------------------------------------------------------------------------ GPU

RUN_CFG = """
model = aggregation
kernel = constant
m = 256
initial = monodisperse
stepper = rk4
mode = adaptive
tol = 1e-8
t_end = 2
snapshots = 1, 2
"""


@pytest.mark.gpu
def test_reference_smoke_checks_on_device(agk):
    # the reference's own python smoke checks (tests/python/test_smoke.py), same expectations
    n = np.zeros(3)
    n[0] = 1.0
    s = A.eval_rhs(n, model="aggregation", kernel="constant")
    assert s == pytest.approx([-1.0, 0.5, 0.0], abs=1e-14)
    withsrc = A.eval_rhs(n, model="sources", kernel="constant", sources=[(1, 1.0)])
    assert withsrc[0] == pytest.approx(0.0, abs=1e-14)
    rng = np.random.default_rng(42)
    n = rng.random(128)
    fast = A.eval_rhs(n, model="shattering", kernel="brownian", alpha=0.95, lam=0.01)
    dense = A.eval_rhs(n, model="shattering", kernel="brownian", alpha=0.95, lam=0.01, dense=True)
    assert np.max(np.abs(fast - dense)) <= 1e-12 * np.max(np.abs(dense))
    n = np.zeros(8)
    n[0] = 2.0
    assert A.euler_stability_bound(n, kernel="constant", a=0.25) == pytest.approx(0.125)
    report = A.run_text(RUN_CFG)
    assert report["termination"] == "completed"
    assert report["N"][-1] == pytest.approx(0.5, abs=1e-6)
    n2 = report["snapshots"][2.0]
    assert n2[0] == pytest.approx(0.25, abs=1e-6)
    assert n2[1] == pytest.approx(0.125, abs=1e-6)
    err = report["err"][1:]
    assert np.all(err[~np.isnan(err)] <= 1e-8)
    assert report["total_rhs_evals"] == report["rhs_evals"][-1]
    with pytest.raises(Exception, match="kernel"):
        A.run_text("model = aggregation\nm = 8\nstepper = rk2\nmode = fixed\ntau = 0.1\nt_end = 1\n")


@pytest.mark.gpu
def test_run_file(agk, tmp_path):
    cfg = tmp_path / "run.cfg"
    cfg.write_text(RUN_CFG)
    report = A.run_file(str(cfg))
    assert report["termination"] == "completed"
    assert report["final_t"] == 2.0


FRONTEND_RUNS = [
    "model = sources\nkernel = brownian\nalpha = 0.333\nm = 512\nsources = 1:1\nstepper = rkf45\n"
    "mode = adaptive\ntol = 1e-6\nt_end = 5\nsnapshots = 1, 5\nrecord = every_step\n",
    "model = shattering\nkernel = brownian\nalpha = 0.95\nm = 256\nlambda = 0.01\nstepper = rk2\n"
    "mode = adaptive\ntol = 1e-6\nt_end = 4\nrecord = interval\nrecord_interval = 0.5\n",
    "model = aggregation\nkernel = free_molecular\nm = 200\ninitial = exponential\ninitial_scale = 3\n"
    "stepper = rk4\nmode = fixed\ntau = 0.01\nt_end = 0.5\nrecord = none\n",
]


@pytest.mark.gpu
@pytest.mark.parametrize("text", FRONTEND_RUNS)
def test_run_text_matches_oracle(agk, oracle_port, text):
    cfg = A.parse_config_text(text)
    got = A.run_text(text)
    model, sim = A.to_simulation(cfg)
    om = O.Model(None if model.k is not None else model.u, None if model.k is not None else model.v, model.variant,
                 list(model.sources), model.shatter_rate, k=model.k)
    c = sim.control
    want = oracle_port.run(om, sim.initial, O.Control(stepper=c.stepper, mode=c.mode, tau=c.tau, tol=c.tol),
                           sim.t_end, snapshot_times=list(sim.snapshot_times), record=sim.record,
                           record_interval=sim.record_interval, records_capacity=100000)
    assert got["termination"] == ("completed", "aborted")[want["termination"]]
    assert got["total_accepted"] == want["total_accepted"]
    assert got["total_rejects"] == want["total_rejects"]
    assert got["total_rhs_evals"] == want["total_rhs_evals"]
    assert len(got["t"]) == want["num_records"]
    assert rel_max_diff(got["final_state"], want["final_state"]) <= 1e-9
