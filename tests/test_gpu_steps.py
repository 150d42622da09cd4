"""GPU parity of the RK steppers and the device step controller (reference steppers.cpp:94-300)
against the oracle, with the reference's injected RHS fakes (test_steppers.cpp) running on the
device and with the model RHS.

Exact (bitwise) where the arithmetic is exact in both (fakes with dyadic data, hand values);
otherwise 1e-12 relative on states and the controller's decisions identical.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import factors, rel_max_diff

pytestmark = pytest.mark.gpu


def model_ws(agk, kind, m, alpha=0.0, variant=O.AGGREGATION, sources=(), lam=0.0):
    u, v = factors(kind, m, alpha)
    return O.Model(u, v, variant, list(sources), lam), agk.RhsWorkspace(agk.Model(u, v, variant, list(sources), lam))


def ctl(agk, **kw):
    return agk.StepControl(**kw), O.Control(**kw)


def test_rk2_hand_value(agk):
    _, ws = model_ws(agk, "constant", 2)
    out = agk.rk2_step(ws, [1.0, 0.0], 0.1)   # test_steppers.cpp:44-54
    assert abs(out[0] - 0.90725) <= 1e-15 and abs(out[1] - 0.042875) <= 1e-15


def test_decay_multipliers(agk):
    ws = agk.fake_rhs(agk.RHS_DECAY, 2)
    out = agk.rk2_step(ws, [1.0, 2.0], 0.1)
    mult = 1.0 - 0.1 + 0.01 / 2
    assert abs(out[0] - mult) <= 1e-15 and abs(out[1] - 2 * mult) <= 2e-15
    ws1 = agk.fake_rhs(agk.RHS_DECAY, 1)
    assert abs(agk.rk4_step(ws1, [1.0], 0.1)[0] - 0.9048375) <= 1e-15
    n4, n5, err = agk.rkf45_step(ws1, [1.0], 0.1)
    assert abs(n5[0] - math.exp(-0.1)) <= 1e-7 and err <= 1e-7
    assert abs(err - abs(n5[0] - n4[0])) <= 1e-14 * err


def test_rk4_matches_scripted_oracle(agk, oracle_port):
    om, ws = model_ws(agk, "constant", 2)
    got = agk.rk4_step(ws, [1.0, 0.0], 0.1)
    want, _, _, _ = oracle_port.rk_step(O.RK4, [1.0, 0.0], 0.1, model=om)
    np.testing.assert_allclose(got, want, rtol=1e-15, atol=1e-17)


def test_rkf45_error_identity(agk, oracle_port):
    om, ws = model_ws(agk, "constant", 6)
    n = [0.5, 0.25, 0.125, 0.0625, 0.03125, 0.015625]
    n4, n5, err = agk.rkf45_step(ws, n, 0.2)
    w4, w5, werr, _ = oracle_port.rk_step(O.RKF45, n, 0.2, model=om)
    # err = ||n5 - n4|| is a difference of O(1) vectors: a one-ulp difference of any component
    # (the RHS values agree to ~1e-16, not bitwise) moves it by ~eps ||n||, which at err ~ 3e-7 is
    # ~1e-10 relative; the bar is that cancellation floor, stated absolutely
    assert abs(err - werr) <= 4e-16 * np.linalg.norm(w4) + 1e-12 * werr
    np.testing.assert_allclose(n4, w4, rtol=1e-14)


def test_zero_fixed_point(agk):
    _, ws = model_ws(agk, "constant", 4)
    for kind in (agk.RK2, agk.RK4, agk.RKF45):
        o = agk.fixed_step(ws, np.zeros(4), 0.3, kind)
        assert o.ok() and np.all(o.state == 0.0) and o.tau_next == 0.3
        if kind == agk.RKF45:
            assert o.error_estimate == 0.0


def test_fixed_step_bookkeeping(agk):
    ws = agk.fake_rhs(agk.RHS_DECAY, 2)
    n = [1.0, 0.5]
    o2 = agk.fixed_step(ws, n, 0.1, agk.RK2)
    assert o2.rhs_evals == 2 and math.isnan(o2.error_estimate)
    o4 = agk.fixed_step(ws, n, 0.1, agk.RK4)
    assert o4.rhs_evals == 4
    o45 = agk.fixed_step(ws, n, 0.1, agk.RKF45)
    assert o45.rhs_evals == 6 and not math.isnan(o45.error_estimate)
    n4, _, _ = agk.rkf45_step(ws, n, 0.1)
    assert np.array_equal(o45.state, n4)


FAKES = [("decay", 0.0), ("still", 0.0), ("drain", 1.0), ("burst_inf", 0.0), ("burst_nan", 0.0)]
FAKE_KIND = {"decay": O.RHS_DECAY, "still": O.RHS_STILL, "drain": O.RHS_DRAIN, "burst_inf": O.RHS_BURST_INF,
             "burst_nan": O.RHS_BURST_NAN}


@pytest.mark.parametrize("stepper", [O.RK2, O.RK4, O.RKF45])
@pytest.mark.parametrize("mode", [O.FIXED, O.ADAPTIVE])
@pytest.mark.parametrize("fake,param", FAKES)
def test_controller_on_fakes_matches_oracle(agk, oracle_port, stepper, mode, fake, param):
    n = np.array([0.1, 1.0, 0.3])
    kind = FAKE_KIND[fake]
    gc, oc = ctl(agk, stepper=stepper, mode=mode, tau=0.1, tol=1e-3, max_rejects=5)
    ws = agk.fake_rhs(kind, 3, param)
    g = agk.advance(ws, n, 1.0, gc)
    w = oracle_port.advance(n, 1.0, oc, kind=kind, param=param)
    assert g.status == w["status"]
    assert g.rejects == w["rejects"] and g.rhs_evals == w["rhs_evals"]
    # device pow is within 2 ulp of glibc's: tau after a reject agrees to ~1e-14 relative
    assert abs(g.tau_used - w["tau_used"]) <= 4e-14 * abs(w["tau_used"])
    if g.status == O.STEP_OK:
        assert abs(g.tau_next - w["tau_next"]) <= 1e-13 * abs(w["tau_next"])
        np.testing.assert_allclose(g.state, w["state"], rtol=1e-14, atol=1e-16)
        if math.isnan(w["error_estimate"]):
            assert math.isnan(g.error_estimate)
        else:
            assert abs(g.error_estimate - w["error_estimate"]) <= 1e-12 * max(w["error_estimate"], 1e-300)


def test_doubling_update_rule(agk, oracle_port):
    """test_steppers.cpp:206-270."""
    om, ws = model_ws(agk, "constant", 2)
    n = [1.0, 0.0]
    full = agk.rk2_step(ws, n, 0.1)
    mid = agk.rk2_step(ws, n, 0.05)
    half = agk.rk2_step(ws, mid, 0.05)
    err = float(np.sqrt(np.sum((half - full) ** 2)))
    o = agk.step_doubling_adaptive(ws, n, 0.1, agk.StepControl(stepper=agk.RK2, tol=err))
    assert o.ok() and o.rejects == 0 and o.tau_used == 0.1
    assert abs(o.error_estimate - err) <= 1e-12 * err
    assert abs(o.tau_next - 0.05) <= 1e-14
    assert np.array_equal(o.state, half) and o.rhs_evals == 6
    # zero right-hand side grows at the clamp
    still = agk.fake_rhs(agk.RHS_STILL, 2)
    o = agk.step_doubling_adaptive(still, n, 0.1, agk.StepControl(stepper=agk.RK2, tol=1e-10))
    assert o.ok() and o.error_estimate == 0.0 and abs(o.tau_next - 0.2) <= 1e-15
    # rejection halves the step
    o = agk.step_doubling_adaptive(ws, n, 0.1, agk.StepControl(stepper=agk.RK2, tol=1e-12))
    assert o.ok() and o.rejects > 0 and abs(o.tau_used - 0.1 / 2 ** o.rejects) <= 1e-15 and o.error_estimate <= 1e-12


def test_fehlberg_rules(agk, oracle_port):
    """test_steppers.cpp:287-330."""
    om, ws = model_ws(agk, "constant", 2)
    n = [1.0, 0.0]
    o = agk.fehlberg_adaptive(ws, n, 0.1, agk.StepControl(tol=1e-4))
    assert o.ok() and o.rejects == 0 and o.error_estimate <= 1e-4
    n4, _, err0 = agk.rkf45_step(ws, n, 0.1)
    assert np.array_equal(o.state, n4)
    assert 0.5 <= o.tau_next / o.tau_used <= 2.0
    o = agk.fehlberg_adaptive(ws, n, 0.1, agk.StepControl(tol=err0 * 0.99))
    assert o.ok() and o.rejects == 1
    factor = min(max(0.9 * (err0 * 0.99 / err0) ** 0.2, 0.5), 2.0)
    assert abs(o.tau_used - 0.1 * factor) <= 1e-14
    still = agk.fake_rhs(agk.RHS_STILL, 2)
    o = agk.fehlberg_adaptive(still, n, 0.1, agk.StepControl(tol=1e-8))
    assert o.ok() and abs(o.tau_next - 0.2) <= 1e-15


def test_negativity_rejection(agk):
    ws = agk.fake_rhs(agk.RHS_DRAIN, 2, 1.0)
    o = agk.step_doubling_adaptive(ws, [0.1, 1.0], 1.0, agk.StepControl(stepper=agk.RK2, tol=1.0))
    assert o.ok() and o.rejects == 4 and o.tau_used == 0.0625 and abs(o.state[0] - 0.0375) <= 1e-14


def test_abort_statuses(agk):
    burst = agk.fake_rhs(agk.RHS_BURST_INF, 2)
    assert agk.fixed_step(burst, [1.0, 1.0], 0.1, agk.RK2).status == agk.STEP_NONFINITE
    nanb = agk.fake_rhs(agk.RHS_BURST_NAN, 2)
    o = agk.step_doubling_adaptive(nanb, [1.0, 1.0], 0.1, agk.StepControl(stepper=agk.RK2, max_rejects=3))
    assert o.status == agk.STEP_NONFINITE and o.rejects == 4
    drain = agk.fake_rhs(agk.RHS_DRAIN, 2, 1e6)
    o = agk.step_doubling_adaptive(drain, [1.0, 1.0], 1.0, agk.StepControl(stepper=agk.RK2, tol=1e300, tau_min=0.3))
    assert o.status == agk.STEP_TAU_UNDERFLOW
    with pytest.raises(ValueError):
        agk.advance(drain, [1.0, 1.0], 0.0, agk.StepControl())
    with pytest.raises(ValueError):
        agk.step_doubling_adaptive(drain, [1.0, 1.0], 0.1, agk.StepControl(stepper=agk.RKF45))


def test_accepted_steps_satisfy_tol(agk):
    """test_steppers.cpp:332-354."""
    _, ws = model_ws(agk, "constant", 16)
    for kind in (agk.RK2, agk.RK4, agk.RKF45):
        c = agk.StepControl(stepper=kind, tol=1e-7)
        state = np.zeros(16)
        state[0] = 1.0
        tau = 0.5
        for _ in range(25):
            o = agk.advance(ws, state, tau, c)
            assert o.ok() and o.error_estimate <= 1e-7
            assert 0.5 - 1e-15 <= o.tau_next / o.tau_used <= 2.0 + 1e-15
            state, tau = o.state, o.tau_next


def test_bitwise_determinism(agk):
    """test_steppers.cpp:356-375."""
    _, ws1 = model_ws(agk, "constant", 32)
    _, ws2 = model_ws(agk, "constant", 32)
    n = np.zeros(32)
    n[0], n[3] = 0.7, 0.3
    c = agk.StepControl(stepper=agk.RK4, tol=1e-8)
    a = agk.step_doubling_adaptive(ws1, n, 0.25, c)
    b = agk.step_doubling_adaptive(ws2, n, 0.25, c)
    assert a.ok() and b.ok()
    assert a.tau_used == b.tau_used and a.tau_next == b.tau_next and a.error_estimate == b.error_estimate
    assert a.rejects == b.rejects and np.array_equal(a.state, b.state)


def test_convergence_orders(agk):
    """test_steppers.cpp:377-402."""
    ws = agk.fake_rhs(agk.RHS_DECAY, 1)
    for kind, nominal in ((agk.RK2, 2.0), (agk.RK4, 4.0)):
        errs = []
        for tau in (0.1, 0.05, 0.025):
            n = np.array([1.0])
            for _ in range(int(round(1.0 / tau))):
                n = agk.rk2_step(ws, n, tau) if kind == agk.RK2 else agk.rk4_step(ws, n, tau)
            errs.append(abs(n[0] - math.exp(-1.0)))
        assert abs(math.log2(errs[0] / errs[1]) - nominal) <= 0.3
        assert abs(math.log2(errs[1] / errs[2]) - nominal) <= 0.3


@pytest.mark.parametrize("stepper", [O.RK2, O.RK4, O.RKF45])
@pytest.mark.parametrize("m", [64, 20000])
def test_model_advance_matches_oracle(agk, oracle_port, stepper, m):
    om, ws = model_ws(agk, "brownian", m, 0.95, O.SHATTERING, lam=0.01)
    n = np.random.default_rng(3).random(m) * np.exp(-np.arange(m) / 30.0)
    gc, oc = ctl(agk, stepper=stepper, tol=1e-6)
    g = agk.advance(ws, n, 0.05, gc)
    w = oracle_port.advance(n, 0.05, oc, model=om)
    assert g.status == w["status"] and g.rejects == w["rejects"] and g.rhs_evals == w["rhs_evals"]
    # after a reject tau = tau0 * factor(err)^k and err carries ~1e-8 relative cancellation noise
    tol = 1e-12 if w["rejects"] == 0 else 1e-7
    assert abs(g.tau_used - w["tau_used"]) <= tol * w["tau_used"]
    assert rel_max_diff(g.state, w["state"]) <= max(1e-11, tol)
