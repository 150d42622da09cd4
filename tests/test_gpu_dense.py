"""GPU parity of the DenseKernel path (rhs_dense.cu) through the C ABI against
the CPU oracle's dense branches, which are pinned bitwise to the reference compiled from source
(tests/test_oracle_pin.py::test_dense_*): kernel_row_sums rhs.cpp:37-45, birth_term 153-159,
shattering_terms 197-205, eval_rhs 212-235, euler_stability_bound 284-294, and the steppers /
run loop driving a dense model.

Tolerance: normwise relative error <= 1e-11 per RHS (north_star); the device sums the same
products in a different (fixed) order. Counts of steps / rejects / RHS evaluations exact.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import rel_max_diff

pytestmark = pytest.mark.gpu

TOL = 1e-11
SRC = [(1, 1.0), (5, 0.1), (1, 0.5)]


def make(agk, m, variant=O.AGGREGATION, lam=0.01):
    K = O.free_molecular_dense(m)
    src = [(k, r) for k, r in SRC if k <= m] if variant == O.SOURCES else []  # k in 1..m (rhs.cpp:50-60)
    om = O.Model(None, None, variant, src, lam, k=K)
    return om, agk.RhsWorkspace(agk.Model(None, None, variant, src, lam, k=K))


def state(m, seed):
    rng = np.random.default_rng(seed)
    return rng.random(m) * np.exp(-np.arange(m) / max(8.0, m / 6.0))


@pytest.mark.parametrize("m", [2, 3, 17, 64, 255, 256, 257, 1000, 1025, 3000])
@pytest.mark.parametrize("variant", [O.AGGREGATION, O.SOURCES, O.SHATTERING])
def test_dense_eval_rhs(agk, oracle_port, m, variant):
    om, ws = make(agk, m, variant)
    for q in range(2):
        n = state(m, 100 * m + q)
        want = oracle_port.eval_rhs(om, n)
        got = agk.eval_rhs(ws, n)
        assert rel_max_diff(got, want) <= TOL
    assert ws.evals() == 2


def test_dense_source_outside_range_rejected(agk):
    # ModelSpec::validate -> SourceTerm::validate throws invalid_argument (rhs.cpp:50-60, 63-66)
    K = O.free_molecular_dense(4)
    with pytest.raises(ValueError):
        agk.RhsWorkspace(agk.Model(None, None, O.SOURCES, [(5, 0.1)], 0.0, k=K))


@pytest.mark.parametrize("m", [64, 1000, 4097])
def test_dense_terms_and_bound(agk, oracle_port, m):
    om, ws = make(agk, m, O.SHATTERING, 0.02)
    n = state(m, 7)
    birth = agk.birth_term(ws, n)
    assert birth[0] == 0.0                                          # rhs.cpp:155
    assert rel_max_diff(birth, oracle_port.birth_term(om, n)) <= TOL
    assert rel_max_diff(agk.death_term(ws, n), oracle_port.death_term(om, n)) <= TOL
    assert rel_max_diff(agk.shattering_terms(ws, n, 0.02), oracle_port.shattering_terms(om, n, 0.02)) <= TOL
    b = agk.euler_stability_bound(ws, n, 0.25)
    assert abs(b - oracle_port.euler_stability_bound(om, n, 0.25)) <= 1e-12 * b
    assert ws.evals() == 0                                          # terms do not count


def test_dense_exact_zeros_and_determinism(agk):
    m = 500
    om, ws = make(agk, m)
    n = state(m, 3)
    n[100:] = 0.0
    a, b = agk.eval_rhs(ws, n), agk.eval_rhs(ws, n)
    assert np.array_equal(a, b)                                     # test_rhs.cpp:265-282
    assert np.all(agk.death_term(ws, n)[100:] == 0.0)               # n_s = 0 -> no loss


def test_dense_large(agk, oracle_port):
    m = 1 << 14                                                     # 2 GiB kernel on the device
    om, ws = make(agk, m, O.SHATTERING, 0.01)
    n = state(m, 11)
    assert rel_max_diff(agk.eval_rhs(ws, n), oracle_port.eval_rhs(om, n)) <= TOL


@pytest.mark.parametrize("stepper", [O.RK2, O.RK4, O.RKF45])
def test_dense_advance(agk, oracle_port, stepper):
    m = 300
    om, ws = make(agk, m, O.SOURCES)
    n = state(m, 5)
    g = agk.advance(ws, n, 0.01, agk.StepControl(stepper=stepper, tol=1e-8))
    w = oracle_port.advance(n, 0.01, O.Control(stepper=stepper, tol=1e-8), model=om)
    assert (g.status, g.rejects, g.rhs_evals) == (w["status"], w["rejects"], w["rhs_evals"])
    assert rel_max_diff(g.state, w["state"]) <= 1e-11


def test_dense_run(agk, oracle_port):
    m = 256
    om, ws = make(agk, m, O.AGGREGATION)
    n0 = np.zeros(m)
    n0[0] = 1.0
    g = agk.run(ws, agk.SimulationConfig(agk.StepControl(tol=1e-6), 5.0, n0))
    w = oracle_port.run(om, n0, O.Control(tol=1e-6), 5.0)
    assert g.termination == "completed" and w["termination"] == 0
    assert (g.total_accepted, g.total_rejects, g.total_rhs_evals) == \
           (w["total_accepted"], w["total_rejects"], w["total_rhs_evals"])
    assert rel_max_diff(g.final_state, w["final_state"]) <= 1e-9
