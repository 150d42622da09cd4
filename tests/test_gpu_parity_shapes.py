"""Per-RHS and per-step parity at the BASELINE config shapes, against the REFERENCE ITSELF
(oracle/_ref: rhs.cpp / fft.cpp / steppers.cpp compiled from the reference's sources, built here
and shipped to the GPU box as a .so; the C restatement stands in only if _ref is missing).

Cases ("Next round" item 1):
  * config 3 shape: M = 2^17, generalized Brownian alpha = 0.9 (R = 2 -> R_f = 1), lambda = 0.01;
  * config 5 shape: M = 2^20, Brownian + 2 (R = 3 -> R_f = 2) with the monomer source;
  * config 4 shape: M = 2^20, R = 16 random kernel (std::mt19937_64 inputs), straight vs _ref;
  * the P = 2^21 warp path away from m = 2^20: odd m = 700001 and m = 2^20 - 3, both with
    R_f = 2 (k_dvec after the row pass) and with R_f = 16 (k_dvec beside it); R_f = 20 (two rank
    groups: the accumulating row launch);
  * the m in (2^20, 2^22] four-step paths (P = 2^22, 2^23): m = 2^20 + 1, 3 * 2^20, 2^22;
  * the four-step path at P = 2^18, 2^19, 2^20 (m = 100001, 200001, 400001, 2^19);
  * one RKF45 `advance` (the device trial loop + controller) at config 5 full shape.
Bar: north_star's 1e-11 max normwise relative error per RHS, exact zeros where the reference
has them. Measured values are appended to $AGK_PARITY_REPORT (JSON lines) when it is set.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import config4_inputs, factors, rel_max_diff

pytestmark = pytest.mark.gpu
TOL = 1e-11


@pytest.fixture(scope="module")
def ref():
    try:
        return O.Oracle("reference")
    except FileNotFoundError:
        return O.Oracle("port")  # pinned bitwise to _ref (tests/test_oracle_pin.py)


def report(case, **kw):
    path = os.environ.get("AGK_PARITY_REPORT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(dict(case=case, **kw)) + "\n")


def cfg3_state(m, rng):
    s = np.arange(1, m + 1, dtype=np.float64)
    return s ** -1.5 * np.exp(-s / 2000.0) * rng.uniform(0.9, 1.1, m)


def cfg5_state(m, rng):
    s = np.arange(1, m + 1, dtype=np.float64)
    n = 0.3 * s ** -1.5 * np.exp(-s / 5e4) * rng.uniform(0.9, 1.1, m)
    n[s > 6e5] = 0.0  # the unreached tail is exactly zero, as in a run from n0 = 0
    return n


def check(case, agk, ref, u, v, variant, sources, lam, n, want_rf=None):
    om = O.Model(u, v, variant, list(sources), lam)
    ws = agk.RhsWorkspace(agk.Model(u, v, variant, list(sources), lam))
    if want_rf is not None:
        assert ws.unique_ranks() == want_rf
    got = agk.eval_rhs(ws, n)
    want = ref.eval_rhs(om, n)
    d = rel_max_diff(got, want)
    report(case, m=int(n.size), rf=ws.unique_ranks(), rel_max_diff=d, oracle=ref.which)
    assert d <= TOL, (case, d)
    # exact zeros where the reference has them: death and shattering loss where n_s == 0
    zero = n == 0.0
    if zero.any():
        dt = agk.death_term(ws, n)
        assert np.all(dt[zero] == 0.0)
    assert agk.birth_term(ws, n)[0] == 0.0
    ws.close()
    return d


def test_config3_shape(agk, ref):
    m = 1 << 17
    u, v = factors("brownian", m, 0.9)
    rng = np.random.default_rng(3)
    check("c3_shape_smooth", agk, ref, u, v, O.SHATTERING, [], 0.01, cfg3_state(m, rng), want_rf=1)
    n0 = np.zeros(m)
    n0[0] = 1.0
    check("c3_shape_monodisperse", agk, ref, u, v, O.SHATTERING, [], 0.01, n0, want_rf=1)


def test_config5_shape(agk, ref):
    m = 1 << 20
    u, v = factors("brownian2", m)
    rng = np.random.default_rng(5)
    check("c5_shape", agk, ref, u, v, O.SOURCES, [(1, 1.0)], 0.0, cfg5_state(m, rng), want_rf=2)
    check("c5_shape_n0", agk, ref, u, v, O.SOURCES, [(1, 1.0)], 0.0, np.zeros(m), want_rf=2)


def test_config4_vs_reference(agk, ref):
    U, V, n = config4_inputs()
    check("c4_shape", agk, ref, U, V, O.AGGREGATION, [], 0.0, n, want_rf=16)


@pytest.mark.parametrize("m", [700001, (1 << 20) - 3])
def test_warp_path_odd_sizes(agk, ref, m):
    rng = np.random.default_rng(m)
    u, v = factors("brownian2", m)
    check(f"warp_m{m}_rf2", agk, ref, u, v, O.SOURCES, [(1, 1.0), (7, 0.5)], 0.0, cfg5_state(m, rng), want_rf=2)
    U, V, n = config4_inputs(m, 16)
    check(f"warp_m{m}_rf16_shatter", agk, ref, U, V, O.SHATTERING, [], 0.01, n, want_rf=16)


@pytest.mark.parametrize("m", [100001, 200001, 400001, 1 << 19])
def test_mid_four_step_sizes(agk, ref, m):
    """The four-step path between the config-3 shape and the warp path (P = 2^18, 2^19, 2^20: 8 points
    per thread in the forward column and row passes), odd sizes included."""
    rng = np.random.default_rng(m)
    u, v = factors("brownian2", m)
    check(f"mid_m{m}_rf2", agk, ref, u, v, O.SOURCES, [(1, 1.0), (5, 0.25)], 0.0, cfg5_state(m, rng), want_rf=2)
    u, v = factors("brownian", m, 0.9)
    check(f"mid_m{m}_shatter", agk, ref, u, v, O.SHATTERING, [], 0.01, cfg3_state(m, rng), want_rf=1)


def test_warp_path_two_rank_groups(agk, ref):
    """More unique ranks than one warp-path group holds (16): R_f = 20 -> groups of 16 + 4, i.e. the
    accumulating row launch (the Hermitian accumulator carried through global memory) followed by
    the closing one (rhs.cpp:126-149 summed over all ranks)."""
    m = 600001
    U, V, n = config4_inputs(m, 20)
    check("warp_m600001_rf20_two_groups", agk, ref, U, V, O.AGGREGATION, [], 0.0, n, want_rf=20)


@pytest.mark.parametrize("m", [(1 << 20) + 1, 3 << 20, 1 << 22])
def test_large_four_step(agk, ref, m):
    rng = np.random.default_rng(m)
    u, v = factors("brownian2", m)
    check(f"large_m{m}", agk, ref, u, v, O.SOURCES, [(1, 1.0)], 0.0, cfg5_state(m, rng), want_rf=2)


def test_config5_advance_rkf45(agk, ref):
    """One adaptive RKF45 step (fehlberg_adaptive, steppers.cpp:246-291) at config 5 full shape:
    the device trial loop and controller vs the reference's, from a mid-run-like state."""
    m = 1 << 20
    u, v = factors("brownian2", m)
    rng = np.random.default_rng(55)
    n = cfg5_state(m, rng)
    om = O.Model(u, v, O.SOURCES, [(1, 1.0)], 0.0)
    ws = agk.RhsWorkspace(agk.Model(u, v, O.SOURCES, [(1, 1.0)], 0.0))
    for tau in (0.05, 2.0):  # an accepted step, and one that needs rejects first
        ctl = agk.StepControl(stepper=agk.RKF45, tol=1e-6)
        g = agk.advance(ws, n, tau, ctl)
        w = ref.advance(n, tau, O.Control(stepper=O.RKF45, tol=1e-6), model=om)
        assert g.status == w["status"] == O.STEP_OK
        assert g.rejects == w["rejects"] and g.rhs_evals == w["rhs_evals"]
        dt = abs(g.tau_used - w["tau_used"]) / w["tau_used"]
        ds = rel_max_diff(g.state, w["state"])
        de = abs(g.error_estimate - w["error_estimate"]) / w["error_estimate"]
        report(f"c5_advance_rkf45_tau{tau}", rejects=g.rejects, tau_rel=dt, state_rel_max_diff=ds, err_rel=de,
               oracle=ref.which)
        if g.rejects == 0:
            assert dt == 0.0 and ds <= TOL, (dt, ds)
        else:
            # after a reject tau = tau0 * factor(err)^..., and err carries ~1e-8 relative roundoff
            assert dt <= 1e-8 and ds <= 1e-8, (dt, ds)
        assert de <= 1e-6  # ||n5 - n4|| is a difference of O(1) vectors: ~1e-8 relative noise in any build
