"""Pin the CPU oracle (agk_oracle.c) before trusting it.

1. Bitwise identity with the reference compiled from its own sources (oracle/_ref).
2. The reference's own hand values and known answers (tests/test_rhs.cpp, test_steppers.cpp,
   test_simulator.cpp, tests/python/test_smoke.py), restated here.
3. The reference's committed run goldens (proj/out/*/summary.txt counts) and the fixtures in
   tests/golden/ generated from oracle/_ref by tests/golden/make_golden.py.
CPU only (no GPU needed).
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import factors, rel_max_diff

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
KERNELS = [("constant", 0.0), ("brownian", 1.0 / 3.0), ("brownian", 0.95), ("brownian2", 0.0)]


def model(kind, m, alpha=0.0, variant=O.AGGREGATION, sources=(), lam=0.0):
    u, v = factors(kind, m, alpha)
    return O.Model(u, v, variant, list(sources), lam)


# ----------------------------------------------------------------- 1. port == reference bitwise

@pytest.mark.parametrize("m", [2, 3, 5, 16, 40, 96, 257, 1000])
@pytest.mark.parametrize("kind,alpha", KERNELS)
@pytest.mark.parametrize("variant", [O.AGGREGATION, O.SOURCES, O.SHATTERING])
def test_port_rhs_bitwise_equals_reference(oracle_port, oracle_ref, m, kind, alpha, variant):
    rng = np.random.default_rng(m * 31 + variant)
    md = model(kind, m, alpha, variant, [(1, 1.0), (min(m, 10), 0.1), (1, 0.5)], 0.01)
    for _ in range(3):
        n = rng.random(m)
        assert np.array_equal(oracle_port.eval_rhs(md, n), oracle_ref.eval_rhs(md, n))
        assert np.array_equal(oracle_port.birth_term(md, n), oracle_ref.birth_term(md, n))
        assert np.array_equal(oracle_port.death_term(md, n), oracle_ref.death_term(md, n))
        assert np.array_equal(oracle_port.shattering_terms(md, n, 0.3), oracle_ref.shattering_terms(md, n, 0.3))
        assert oracle_port.euler_stability_bound(md, n, 0.25) == oracle_ref.euler_stability_bound(md, n, 0.25)


def test_port_rhs_random_asymmetric_rank16_bitwise(oracle_port, oracle_ref):
    """Config-4-like asymmetric random kernel (no dedupe) plus a duplicated and a swapped rank."""
    rng = np.random.default_rng(7)
    m, r = 300, 6
    i = np.arange(1, m + 1.0)
    p = rng.uniform(-0.5, 0.5, r)
    u = rng.uniform(0.5, 1.5, r)[None, :] * i[:, None] ** p[None, :]
    v = rng.uniform(0.5, 1.5, r)[:, None] * i[None, :] ** (-p[:, None])
    u[:, 3] = u[:, 1]
    v[3] = v[1]          # rank 3 == rank 1 (same)
    u[:, 5] = v[0]
    v[5] = u[:, 0]       # rank 5 == rank 0 swapped
    md = O.Model(u, v, O.SHATTERING, [], 0.02)
    n = np.exp(-i / 50.0) * rng.uniform(0.9, 1.1, m)
    assert np.array_equal(oracle_port.eval_rhs(md, n), oracle_ref.eval_rhs(md, n))


FAKES = [(O.RHS_DECAY, 0.0), (O.RHS_STILL, 0.0), (O.RHS_DRAIN, 1.0), (O.RHS_BURST_INF, 0.0), (O.RHS_BURST_NAN, 0.0)]


@pytest.mark.parametrize("stepper", [O.RK2, O.RK4, O.RKF45])
@pytest.mark.parametrize("mode", [O.FIXED, O.ADAPTIVE])
@pytest.mark.parametrize("fake,param", FAKES)
def test_port_advance_fakes_bitwise(oracle_port, oracle_ref, stepper, mode, fake, param):
    n = np.array([0.1, 1.0, 0.3])
    ctl = O.Control(stepper=stepper, mode=mode, tau=0.1, tol=1e-3, max_rejects=5)
    a = oracle_port.advance(n, 1.0, ctl, kind=fake, param=param)
    b = oracle_ref.advance(n, 1.0, ctl, kind=fake, param=param)
    for key in ("tau_used", "tau_next", "rejects", "rhs_evals", "status"):
        assert a[key] == b[key], key
    assert (math.isnan(a["error_estimate"]) and math.isnan(b["error_estimate"])) or a["error_estimate"] == b["error_estimate"]
    assert np.array_equal(a["state"], b["state"], equal_nan=True)


@pytest.mark.parametrize("stepper", [O.RK2, O.RK4, O.RKF45])
@pytest.mark.parametrize("tol", [1e-4, 1e-8, 1e-12])
def test_port_advance_model_bitwise(oracle_port, oracle_ref, stepper, tol):
    md = model("brownian", 64, 0.95, O.SHATTERING, lam=0.01)
    n = np.random.default_rng(3).random(64)
    ctl = O.Control(stepper=stepper, tol=tol)
    a = oracle_port.advance(n, 0.5, ctl, model=md)
    b = oracle_ref.advance(n, 0.5, ctl, model=md)
    assert a["status"] == b["status"] and a["rejects"] == b["rejects"] and a["rhs_evals"] == b["rhs_evals"]
    assert a["tau_used"] == b["tau_used"] and a["tau_next"] == b["tau_next"]
    assert a["error_estimate"] == b["error_estimate"]
    assert np.array_equal(a["state"], b["state"], equal_nan=True)


@pytest.mark.parametrize("relative", [False, True])
def test_port_run_bitwise(oracle_port, oracle_ref, relative):
    md = model("brownian2", 200, 0.0, O.SOURCES, [(1, 1.0), (7, 0.2)])
    n0 = np.zeros(200)
    ctl = O.Control(stepper=O.RKF45, tol=1e-7, relative_error=relative)
    a = oracle_port.run(md, n0, ctl, 30.0, snapshot_times=[0.0, 1.5, 30.0], record=O.RECORD_INTERVAL,
                        record_interval=0.7, records_capacity=1000)
    b = oracle_ref.run(md, n0, ctl, 30.0, snapshot_times=[0.0, 1.5, 30.0], record=O.RECORD_INTERVAL,
                       record_interval=0.7, records_capacity=1000)
    for key in ("termination", "total_rhs_evals", "total_accepted", "total_rejects", "final_t", "num_records"):
        assert a[key] == b[key], key
    assert np.array_equal(a["final_state"], b["final_state"])
    assert np.array_equal(a["snapshots"], b["snapshots"])
    for ra, rb in zip(a["records"], b["records"]):
        for k in ra:
            assert (ra[k] == rb[k]) or (isinstance(ra[k], float) and math.isnan(ra[k]) and math.isnan(rb[k])), k


def test_port_run_abort_matches_reference(oracle_port, oracle_ref):
    md = model("constant", 32)
    n0 = np.zeros(32)
    n0[0] = 1.0
    ctl = O.Control(stepper=O.RK2, tol=1e-14, max_rejects=2, tau_min=1e-3)
    a = oracle_port.run(md, n0, ctl, 5.0, initial_tau=1.0)
    b = oracle_ref.run(md, n0, ctl, 5.0, initial_tau=1.0)
    assert a["termination"] == b["termination"] == 1
    for key in ("abort_status", "abort_t", "abort_tau", "total_rhs_evals", "total_rejects", "total_accepted"):
        assert a[key] == b[key], key


# ----------------------------------------------------------------- 2. reference hand values

def test_hand_values_birth_death_shattering(oracle_port):
    md = model("constant", 3)
    b = oracle_port.birth_term(md, [1.0, 0.0, 0.0])           # test_rhs.cpp:47-59
    assert b[0] == 0.0 and abs(b[1] - 0.5) <= 1e-14 * 0.5 and abs(b[2]) <= 1e-14
    d = oracle_port.death_term(md, [1.0, 0.0, 0.0])           # test_rhs.cpp:61-73
    assert abs(d[0] - 1.0) <= 1e-15 and d[1] == 0.0 and d[2] == 0.0
    s = oracle_port.shattering_terms(md, [0.0, 1.0, 0.0], 1.0)  # test_rhs.cpp:75-96
    assert abs(s[0] - 2.0) <= 1e-14 * 2 and abs(s[1] + 1.0) <= 1e-14 and s[2] == 0.0
    with pytest.raises(O.OracleError):
        oracle_port.shattering_terms(md, [0.0, 1.0, 0.0], -1.0)


def test_hand_values_eval_rhs(oracle_port):
    n = [1.0, 0.0, 0.0]                                       # test_rhs.cpp:116-143
    out = oracle_port.eval_rhs(model("constant", 3), n)
    assert abs(out[0] + 1.0) <= 1e-14 and abs(out[1] - 0.5) <= 1e-14 and abs(out[2]) <= 1e-14
    out = oracle_port.eval_rhs(model("constant", 3, variant=O.SOURCES, sources=[(1, 1.0)]), n)
    assert abs(out[0]) <= 1e-14 and abs(out[1] - 0.5) <= 1e-14
    out = oracle_port.eval_rhs(model("constant", 3, variant=O.SOURCES, sources=[(2, 0.25)]), [0.0, 0.0, 0.0])
    assert out[0] == 0.0 and out[1] == 0.25 and out[2] == 0.0


@pytest.mark.parametrize("m", [16, 64, 256])
@pytest.mark.parametrize("kind,alpha", KERNELS[:3])
@pytest.mark.parametrize("variant", [O.AGGREGATION, O.SOURCES, O.SHATTERING])
def test_low_rank_agrees_with_dense_oracle(oracle_port, m, kind, alpha, variant):
    """test_rhs.cpp:161-195 (<= 1e-12 normwise)."""
    rng = np.random.default_rng(29 + m)
    md = model(kind, m, alpha, variant, [(1, 1.0), (10, 0.1)], 0.01)
    for _ in range(3):
        n = rng.random(m)
        assert rel_max_diff(oracle_port.eval_rhs(md, n), oracle_port.eval_rhs_dense(md, n)) <= 1e-12


def test_euler_bound_hand_values(oracle_port):
    md = model("constant", 8)                                 # test_rhs.cpp:300-320
    n = np.zeros(8)
    n[0], n[4] = 1.5, 0.5
    assert abs(oracle_port.euler_stability_bound(md, n, 0.25) - 0.125) <= 1e-15
    assert math.isinf(oracle_port.euler_stability_bound(md, np.zeros(8), 0.25))


def test_stepper_hand_values(oracle_port):
    md = model("constant", 2)                                 # test_steppers.cpp:44-54
    out, _, _, _ = oracle_port.rk_step(O.RK2, [1.0, 0.0], 0.1, model=md)
    assert abs(out[0] - 0.90725) <= 1e-15 and abs(out[1] - 0.042875) <= 1e-15 * 0.05
    out, _, _, _ = oracle_port.rk_step(O.RK4, [1.0], 0.1, kind=O.RHS_DECAY)   # :98-103
    assert abs(out[0] - 0.9048375) <= 1e-15
    n4, n5, err, _ = oracle_port.rk_step(O.RKF45, [1.0], 0.1, kind=O.RHS_DECAY)  # :105-118
    assert abs(n5[0] - math.exp(-0.1)) <= 1e-7 and err <= 1e-7


def test_negativity_rejection_hand_values(oracle_port):
    """test_steppers.cpp:404-418: 4 rejects, tau 0.0625, state 0.0375."""
    o = oracle_port.advance([0.1, 1.0], 1.0, O.Control(stepper=O.RK2, tol=1.0), kind=O.RHS_DRAIN, param=1.0)
    assert o["status"] == O.STEP_OK and o["rejects"] == 4
    assert o["tau_used"] == 0.0625 and abs(o["state"][0] - 0.0375) <= 1e-14


def test_abort_statuses(oracle_port):
    """test_steppers.cpp:420-454."""
    o = oracle_port.advance([1.0, 1.0], 0.1, O.Control(stepper=O.RK2, mode=O.FIXED, tau=0.1), kind=O.RHS_BURST_INF)
    assert o["status"] == O.STEP_NONFINITE
    o = oracle_port.advance([1.0, 1.0], 0.1, O.Control(stepper=O.RK2, tol=1e-6, max_rejects=3), kind=O.RHS_BURST_NAN)
    assert o["status"] == O.STEP_NONFINITE and o["rejects"] == 4
    o = oracle_port.advance([1.0, 1.0], 1.0, O.Control(stepper=O.RK2, tol=1e300, tau_min=0.3), kind=O.RHS_DRAIN,
                            param=1e6)
    assert o["status"] == O.STEP_TAU_UNDERFLOW


def test_analytic_constant_kernel_run(oracle_port):
    """test_simulator.cpp:93-112 and acceptance #1 (analytic n_k(t))."""
    md = model("constant", 256)
    n0 = np.zeros(256)
    n0[0] = 1.0
    r = oracle_port.run(md, n0, O.Control(stepper=O.RK4, tol=1e-8), 2.0)
    n = r["final_state"]
    assert r["final_t"] == 2.0
    assert abs(n.sum() - 0.5) <= 1e-6
    for k in (1, 2):
        exact = 4.0 / 16.0 * (2.0 / 4.0) ** (k - 1)
        assert abs(n[k - 1] - exact) <= 1e-6


def test_fixed_step_counts(oracle_port):
    """test_simulator.cpp:226-238: 100 steps, 200 evals."""
    md = model("constant", 16)
    n0 = np.zeros(16)
    n0[0] = 1.0
    r = oracle_port.run(md, n0, O.Control(stepper=O.RK2, mode=O.FIXED, tau=0.01), 1.0)
    assert r["total_accepted"] == 100 and r["total_rhs_evals"] == 200 and r["total_rejects"] == 0


# ----------------------------------------------------------------- 3. committed goldens

def test_reference_out_goldens(oracle_port):
    """proj/out/aggregation_small and shattering_relaxation summary.txt counts."""
    md = model("constant", 256)
    n0 = np.zeros(256)
    n0[0] = 1.0
    r = oracle_port.run(md, n0, O.Control(stepper=O.RK4, tol=1e-8), 10.0, snapshot_times=[1.0, 10.0])
    assert (r["total_rhs_evals"], r["total_accepted"], r["total_rejects"]) == (1572, 128, 3)
    md = model("constant", 4096, variant=O.SHATTERING, lam=0.01)
    n0 = np.zeros(4096)
    n0[0] = 1.0
    r = oracle_port.run(md, n0, O.Control(stepper=O.RK4, tol=1e-6), 5000.0, snapshot_times=[500.0, 5000.0])
    assert (r["total_rhs_evals"], r["total_accepted"], r["total_rejects"]) == (1800, 149, 1)


def test_port_matches_golden_rhs_fixtures(oracle_port):
    g = np.load(os.path.join(GOLDEN, "golden_rhs.npz"))
    for c in range(int(g["count"][0])):
        m, var, kidx = (int(x) for x in g[f"c{c}_meta"])
        kind, alpha = KERNELS[kidx]
        srcs = [(1, 1.0), (min(m, 10), 0.1)] if var == O.SOURCES else []
        md = model(kind, m, alpha, var, srcs, 0.01 if var == O.SHATTERING else 0.0)
        assert np.array_equal(oracle_port.eval_rhs(md, g[f"c{c}_n"]), g[f"c{c}_S"]), c


def test_port_matches_golden_run_fixtures(oracle_port):
    with open(os.path.join(GOLDEN, "golden_runs.json")) as f:
        runs = json.load(f)
    for name, c in runs.items():
        md = model(c["kind"], c["m"], c["alpha"], c["variant"], [tuple(s) for s in c["sources"]], c["lam"])
        n0 = np.zeros(c["m"])
        if c["variant"] != O.SOURCES:
            n0[0] = 1.0
        ctl = O.Control(stepper=c["stepper"], mode=c["mode"], tau=c["value"] if c["mode"] == O.FIXED else 0.0,
                        tol=c["value"] if c["mode"] == O.ADAPTIVE else 1e-6)
        r = oracle_port.run(md, n0, ctl, c["t_end"], snapshot_times=c["snapshots"])
        assert (r["total_rhs_evals"], r["total_accepted"], r["total_rejects"]) == \
               (c["total_rhs_evals"], c["total_accepted"], c["total_rejects"]), name
        assert np.array_equal(r["final_state"], np.array(c["final_state"])), name


# ---------------------------------------------------------------- DenseKernel branches (§8f item 3)

@pytest.mark.parametrize("m", [2, 3, 17, 64, 300])
@pytest.mark.parametrize("variant", [O.AGGREGATION, O.SOURCES, O.SHATTERING])
def test_port_dense_bitwise_equals_reference(oracle_port, oracle_ref, m, variant):
    """The C restatement of the dense branches (rhs.cpp:37-45, 153-159, 197-205) is bitwise the
    reference's eval_rhs / terms / Euler bound on a DenseKernel (free-molecular, kernels.cpp:49-51)."""
    k = O.free_molecular_dense(m)
    src = [(1, 1.0), (min(m, 5), 0.1)] if variant == O.SOURCES else []
    md = O.Model(None, None, variant, src, 0.02, k=k)
    n = np.random.default_rng(m).random(m)
    for fn in ("eval_rhs", "birth_term", "death_term"):
        assert np.array_equal(getattr(oracle_port, fn)(md, n), getattr(oracle_ref, fn)(md, n)), fn
    assert np.array_equal(oracle_port.shattering_terms(md, n, 0.02), oracle_ref.shattering_terms(md, n, 0.02))
    assert oracle_port.euler_stability_bound(md, n, 0.25) == oracle_ref.euler_stability_bound(md, n, 0.25)


def test_port_dense_advance_bitwise(oracle_port, oracle_ref):
    m = 128
    md = O.Model(None, None, O.SOURCES, [(1, 1.0)], 0.0, k=O.free_molecular_dense(m))
    n = np.random.default_rng(3).random(m) * 0.1
    for stepper in (O.RK2, O.RK4, O.RKF45):
        a = oracle_port.advance(n, 0.01, O.Control(stepper=stepper, tol=1e-9), model=md)
        b = oracle_ref.advance(n, 0.01, O.Control(stepper=stepper, tol=1e-9), model=md)
        assert np.array_equal(a["state"], b["state"]) and a["rhs_evals"] == b["rhs_evals"]


def test_port_matches_golden_dense_fixtures(oracle_port):
    """tests/golden/golden_dense.npz: generated from the reference itself (make_golden.py)."""
    g = np.load(os.path.join(GOLDEN, "golden_dense.npz"))
    for c in range(int(g["count"][0])):
        m, var = (int(x) for x in g[f"c{c}_meta"])
        src = [(1, 1.0), (min(m, 10), 0.1)] if var == O.SOURCES else []
        md = O.Model(None, None, var, src, 0.01 if var == O.SHATTERING else 0.0, k=O.free_molecular_dense(m))
        n = g[f"c{c}_n"]
        assert np.array_equal(oracle_port.eval_rhs(md, n), g[f"c{c}_S"]), c
        assert oracle_port.euler_stability_bound(md, n, 0.25) == g[f"c{c}_bound"][0], c
