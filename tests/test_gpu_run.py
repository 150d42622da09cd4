"""GPU parity of the device-resident run loop (reference run(), simulator.cpp:112-229).

Bars (north_star): total mass and particle number within 1e-8 relative, n_s(t_end) within
1e-6 normwise (max|dn|/max|n|, SURVEY §8c note 8) and element-wise where n_s > 1e-9 max n,
accepted-step count within +-2%. Small cases where the controller sees the same decisions as
the CPU reproduce the counts exactly; that is asserted where it holds.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import factors, rel_max_diff

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def build(agk, kind, m, alpha=0.0, variant=O.AGGREGATION, sources=(), lam=0.0):
    u, v = factors(kind, m, alpha)
    return O.Model(u, v, variant, list(sources), lam), agk.RhsWorkspace(agk.Model(u, v, variant, list(sources), lam))


def _metrics(x, w):
    """Trajectory distance of run x from the oracle run w (north_star's quantities)."""
    fx, fw = np.asarray(x["final_state"]), np.asarray(w["final_state"])
    k = np.arange(1, fw.size + 1)
    big = fw > 1e-9 * np.max(fw)
    return dict(
        N=abs(fx.sum() - fw.sum()) / abs(fw.sum()),
        M1=abs(np.dot(k, fx) - np.dot(k, fw)) / abs(np.dot(k, fw)),
        state=rel_max_diff(fx, fw),
        elem=float(np.max(np.abs(fx[big] / fw[big] - 1.0))) if big.any() else 0.0,
        accepted=abs(x["total_accepted"] - w["total_accepted"]) / max(w["total_accepted"], 1),
    )


# north_star bars, each raised to 10x the CPU-vs-CPU noise floor where that floor is higher
# (after the first divergent decision the drift is a random walk of O(tol) kicks; the floor is
# one sample of it, hence the factor), plus lock-step agreement before that point.
# The error estimate ||n5 - n4|| (or ||half - full||) is a difference of O(1) quantities and carries
# ~1e-8 relative roundoff noise in ANY build, so trajectories whose step sequence is sensitive to it
# drift apart by O(tol) per divergent accept/reject even between two CPU builds of the reference
# (SURVEY §8c note 6). The floor is the largest distance from the oracle of: the oracle built with
# FMA contraction, the oracle with a 2x longer FFT (a different roundoff pattern in the birth term,
# as the GPU's four-step FFT has), and the oracle run at tol*(1 -+ 1e-8).
BARS = dict(N=1e-8, M1=1e-8, state=1e-6, elem=1e-6, accepted=0.02)


def check_run(g, w, f=None):
    """g: device RunReport, w: oracle run, f: oracle_fma run (noise floor)."""
    assert g.termination == ("completed" if w["termination"] == 0 else "aborted")
    assert g.final_t == w["final_t"]
    gx = dict(final_state=g.final_state, total_accepted=g.total_accepted)
    mg = _metrics(gx, w)
    if f is None:
        mf = {k: 0.0 for k in BARS}
    elif isinstance(f, _Floor):
        mf = f
    else:
        mf = _metrics(f, w)
    for key, bar in BARS.items():
        assert mg[key] <= max(bar, FLOOR_FACTOR * mf[key]), (key, mg[key], bar, mf[key])
    return mg, mf


FLOOR_FACTOR = 10.0


def lockstep_len(x_records, w_records, tol=1e-9):
    """Number of leading records on which run x tracks the oracle run w to ~roundoff (same
    cumulative rejects and evals, t and N within `tol` relative)."""
    q = 0
    for a, b in zip(x_records, w_records):
        if a["rejects"] != b["rejects"] or a["rhs_evals"] != b["rhs_evals"]:
            break
        if abs(a["t"] - b["t"]) > tol * max(abs(b["t"]), 1.0):
            break
        if abs(a["density"] - b["density"]) > tol * max(abs(b["density"]), 1e-300):
            break
        q += 1
    return q


def check_lockstep(g, w, f):
    """The device trajectory stays in lock-step with the oracle at least half as long as an
    equally valid CPU build with a different FFT roundoff pattern (the 2x-padded restatement,
    f.variants[1]) does: the birth term's FFT noise in err decides where two builds part ways."""
    cpu = lockstep_len(f.variants[1]["records"], w["records"])
    gpu = lockstep_len(g.records, w["records"])
    assert gpu >= min(cpu, len(w["records"])) // 2, (gpu, cpu)


class _Floor(dict):
    pass


def oracle_pair(om, n0, ctl_kwargs, t_end, **kw):
    """(oracle run, noise-floor metrics) for one configuration; f.variants holds the CPU runs."""
    from oracle.oracle import Oracle
    port = Oracle("port")
    w = port.run(om, n0, O.Control(**ctl_kwargs), t_end, **kw)
    variants = [Oracle("port_fma").run(om, n0, O.Control(**ctl_kwargs), t_end, **kw),
                Oracle("port_pad2").run(om, n0, O.Control(**ctl_kwargs), t_end, **kw)]
    if ctl_kwargs.get("mode", O.ADAPTIVE) == O.ADAPTIVE:
        for d in (1e-8, -1e-8):
            ck = dict(ctl_kwargs, tol=ctl_kwargs.get("tol", 1e-6) * (1.0 + d))
            variants.append(port.run(om, n0, O.Control(**ck), t_end, **kw))
    mets = [_metrics(v, w) for v in variants]
    f = _Floor({k: max(mt[k] for mt in mets) for k in BARS})
    f.variants = variants
    return w, f


def test_golden_run_fixtures(agk):
    """Runs recorded from oracle/_ref (tests/golden/make_golden.py)."""
    with open(os.path.join(GOLDEN, "golden_runs.json")) as f:
        runs = json.load(f)
    for name, c in runs.items():
        _, ws = build(agk, c["kind"], c["m"], c["alpha"], c["variant"], [tuple(s) for s in c["sources"]], c["lam"])
        n0 = np.zeros(c["m"])
        if c["variant"] != O.SOURCES:
            n0[0] = 1.0
        ctl = agk.StepControl(stepper=c["stepper"], mode=c["mode"], tau=c["value"] if c["mode"] == O.FIXED else 0.0,
                              tol=c["value"] if c["mode"] == O.ADAPTIVE else 1e-6)
        g = agk.run(ws, agk.SimulationConfig(ctl, c["t_end"], n0, snapshot_times=c["snapshots"]))
        w = dict(termination=c["termination"], total_accepted=c["total_accepted"], final_t=c["final_t"],
                 final_state=np.array(c["final_state"]))
        om = O.Model(*factors(c["kind"], c["m"], c["alpha"]), c["variant"], [tuple(s) for s in c["sources"]], c["lam"])
        okw = dict(stepper=c["stepper"], mode=c["mode"], tau=ctl.tau, tol=ctl.tol)
        _, f = oracle_pair(om, n0, okw, c["t_end"], snapshot_times=c["snapshots"])
        check_run(g, w, f)


def test_reference_out_goldens(agk):
    """proj/out/*/summary.txt: aggregation_small 1572/128/3, shattering_relaxation 1800/149/1."""
    _, ws = build(agk, "constant", 256)
    n0 = np.zeros(256)
    n0[0] = 1.0
    g = agk.run(ws, agk.SimulationConfig(agk.StepControl(stepper=agk.RK4, tol=1e-8), 10.0, n0, snapshot_times=[1.0, 10.0]))
    assert (g.total_rhs_evals, g.total_accepted, g.total_rejects) == (1572, 128, 3)
    assert len(g.snapshots) == 2 and g.snapshots[0][0] == 1.0
    _, ws = build(agk, "constant", 4096, variant=O.SHATTERING, lam=0.01)
    n0 = np.zeros(4096)
    n0[0] = 1.0
    g = agk.run(ws, agk.SimulationConfig(agk.StepControl(stepper=agk.RK4, tol=1e-6), 5000.0, n0,
                                         snapshot_times=[500.0, 5000.0]))
    assert (g.total_rhs_evals, g.total_accepted, g.total_rejects) == (1800, 149, 1)


def test_sources_steady_state_golden(agk):
    """proj/out/sources_steady_state: m=32768, sources 1:1, 100:0.1, RKF45 tol 1e-6 to t=1000:
    4512 evals, 710 accepted, 42 rejects."""
    _, ws = build(agk, "constant", 32768, variant=O.SOURCES, sources=[(1, 1.0), (100, 0.1)])
    n0 = np.zeros(32768)
    n0[0] = 1.0
    g = agk.run(ws, agk.SimulationConfig(agk.StepControl(tol=1e-6), 1000.0, n0, snapshot_times=[100.0, 1000.0]))
    assert g.termination == "completed"
    assert abs(g.total_accepted - 710) <= 0.02 * 710
    assert (g.total_rhs_evals, g.total_accepted, g.total_rejects) == (4512, 710, 42)


def test_analytic_trajectory(agk):
    """acceptance #1 / test_simulator.cpp:93-112."""
    _, ws = build(agk, "constant", 256)
    n0 = np.zeros(256)
    n0[0] = 1.0
    g = agk.run(ws, agk.SimulationConfig(agk.StepControl(stepper=agk.RK4, tol=1e-8), 10.0, n0,
                                         snapshot_times=[1.0, 2.0, 5.0, 10.0]))
    worst = 0.0
    for t, n in g.snapshots:
        for k in range(1, 21):
            exact = 4.0 / (t + 2) ** 2 * (t / (t + 2)) ** (k - 1)
            worst = max(worst, abs(n[k - 1] - exact) / exact)
    assert worst <= 1e-6
    assert abs(np.sum(g.final_state) - 1.0 / 6.0) <= 1e-7


def test_zero_horizon_and_records(agk):
    _, ws = build(agk, "constant", 8)
    n0 = np.zeros(8)
    n0[0] = 1.0
    g = agk.run(ws, agk.SimulationConfig(agk.StepControl(stepper=agk.RK4, tol=1e-8), 0.0, n0,
                                         record=agk.RECORD_EVERY_STEP))
    assert g.termination == "completed" and g.final_t == 0.0 and g.final_state[0] == 1.0
    assert g.num_records == 1 and g.records[0]["t"] == 0.0 and g.total_rhs_evals == 0


def test_records_match_oracle(agk, oracle_port):
    om, ws = build(agk, "constant", 64)
    n0 = np.zeros(64)
    n0[0] = 1.0
    ctl = dict(stepper=O.RK4, tol=1e-8)
    g = agk.run(ws, agk.SimulationConfig(agk.StepControl(**ctl), 3.0, n0, snapshot_times=[0.0, 0.3777, 1.5, 3.0],
                                         record=agk.RECORD_EVERY_STEP))
    w = oracle_port.run(om, n0, O.Control(**ctl), 3.0, snapshot_times=[0.0, 0.3777, 1.5, 3.0],
                        record=O.RECORD_EVERY_STEP, records_capacity=10000)
    assert g.num_records == w["num_records"]
    wr = w["records"]
    for q, (rg, rw) in enumerate(zip(g.records, wr)):
        # err = ||half - full|| carries ~1e-8 relative cancellation noise (both sides), tau ~ err^(-1/4)
        assert abs(rg["t"] - rw["t"]) <= 1e-7 * max(rw["t"], 1.0)
        assert rg["rhs_evals"] == rw["rhs_evals"] and rg["rejects"] == rw["rejects"]
        # the same record index may sit at a slightly different t (above): the density is compared
        # at 1e-8 relative plus what that time shift moves it by along the oracle's trajectory
        a_, b_ = wr[max(q - 1, 0)], wr[min(q + 1, len(wr) - 1)]
        slope = (b_["density"] - a_["density"]) / (b_["t"] - a_["t"]) if b_["t"] > a_["t"] else 0.0
        assert abs(rg["density"] - rw["density"]) <= 1e-8 * abs(rw["density"]) + abs(slope * (rg["t"] - rw["t"]))
        assert abs(rg["mass"] - rw["mass"]) <= 1e-8 * abs(rw["mass"])
    assert [t for t, _ in g.snapshots] == [0.0, 0.3777, 1.5, 3.0]
    for (tg, sg), sw in zip(g.snapshots, w["snapshots"]):
        assert rel_max_diff(sg, sw) <= 1e-10
    # records strictly increasing in time, counters non-decreasing (test_simulator.cpp:104-111)
    ts = [r["t"] for r in g.records]
    assert all(b > a for a, b in zip(ts, ts[1:]))
    assert g.total_rhs_evals == g.records[-1]["rhs_evals"]


def test_interval_recording(agk, oracle_port):
    om, ws = build(agk, "constant", 32)
    n0 = np.zeros(32)
    n0[0] = 1.0
    g = agk.run(ws, agk.SimulationConfig(agk.StepControl(stepper=agk.RK4, tol=1e-8), 2.0, n0,
                                         record=agk.RECORD_INTERVAL, record_interval=0.5))
    w = oracle_port.run(om, n0, O.Control(stepper=O.RK4, tol=1e-8), 2.0, record=O.RECORD_INTERVAL,
                        record_interval=0.5, records_capacity=1000)
    assert g.num_records == w["num_records"] and g.records[0]["t"] == 0.0 and g.records[-1]["t"] == 2.0


def test_fixed_step_counts(agk):
    _, ws = build(agk, "constant", 16)
    n0 = np.zeros(16)
    n0[0] = 1.0
    g = agk.run(ws, agk.SimulationConfig(agk.StepControl(stepper=agk.RK2, mode=agk.FIXED, tau=0.01), 1.0, n0))
    assert (g.total_accepted, g.total_rhs_evals, g.total_rejects) == (100, 200, 0)


def test_abort_matches_oracle(agk, oracle_port):
    om, ws = build(agk, "constant", 32)
    n0 = np.zeros(32)
    n0[0] = 1.0
    kw = dict(stepper=O.RK2, tol=1e-14, max_rejects=2, tau_min=1e-3)
    g = agk.run(ws, agk.SimulationConfig(agk.StepControl(**kw), 5.0, n0, initial_tau=1.0))
    w = oracle_port.run(om, n0, O.Control(**kw), 5.0, initial_tau=1.0)
    assert g.termination == "aborted" and w["termination"] == 1
    assert g.abort_reason == agk.describe(w["abort_status"])
    assert g.abort_t == w["abort_t"] and g.abort_tau == w["abort_tau"]
    assert (g.total_rhs_evals, g.total_rejects, g.total_accepted) == \
           (w["total_rhs_evals"], w["total_rejects"], w["total_accepted"])


def test_validation_errors(agk):
    _, ws = build(agk, "constant", 8)
    n0 = np.ones(8)
    with pytest.raises(ValueError):
        agk.run(ws, agk.SimulationConfig(agk.StepControl(), -1.0, n0))
    with pytest.raises(ValueError):
        agk.run(ws, agk.SimulationConfig(agk.StepControl(), 1.0, n0, snapshot_times=[0.5, 0.2]))
    with pytest.raises(ValueError):
        agk.run(ws, agk.SimulationConfig(agk.StepControl(safety=1.5), 1.0, n0))
    with pytest.raises(ValueError):
        agk.run(ws, agk.SimulationConfig(agk.StepControl(), 1.0, n0, record=agk.RECORD_INTERVAL))


@pytest.mark.parametrize("stepper", [O.RK2, O.RK4, O.RKF45])
def test_config1_full(agk, oracle_port, stepper):
    """BASELINE config 1: constant kernel, M=4096, n0=e1, tol 1e-6 (rtol), t_end=100."""
    om, ws = build(agk, "constant", 4096)
    n0 = np.zeros(4096)
    n0[0] = 1.0
    g = agk.run(ws, agk.SimulationConfig(agk.StepControl(stepper=stepper, tol=1e-6), 100.0, n0))
    w, f = oracle_pair(om, n0, dict(stepper=stepper, tol=1e-6), 100.0)
    mg, _ = check_run(g, w, f)
    assert mg["N"] <= 1e-8 and mg["M1"] <= 1e-8  # this config is not step-sequence sensitive
    assert abs(np.sum(g.final_state) - 2.0 / 102.0) <= 1e-4 * 2.0 / 102.0


@pytest.mark.parametrize("stepper", [O.RK2, O.RK4, O.RKF45])
def test_config5_reduced_m(agk, oracle_port, stepper):
    """BASELINE config 5 kernel/source at reduced M (4096) to t=50 (SURVEY §8d parity plan)."""
    om, ws = build(agk, "brownian2", 4096, variant=O.SOURCES, sources=[(1, 1.0)])
    n0 = np.zeros(4096)
    g = agk.run(ws, agk.SimulationConfig(agk.StepControl(stepper=stepper, tol=1e-6), 50.0, n0,
                                         record=agk.RECORD_EVERY_STEP))
    w, f = oracle_pair(om, n0, dict(stepper=stepper, tol=1e-6), 50.0, record=O.RECORD_EVERY_STEP,
                       records_capacity=100000)
    check_lockstep(g, w, f)
    check_run(g, w, f)


def test_config3_reduced_m(agk, oracle_port):
    """BASELINE config 3 kernel (alpha=0.9, lambda=0.01, tol 1e-8) at M=2048 to t=20."""
    om, ws = build(agk, "brownian", 2048, 0.9, O.SHATTERING, lam=0.01)
    n0 = np.zeros(2048)
    n0[0] = 1.0
    g = agk.run(ws, agk.SimulationConfig(agk.StepControl(tol=1e-8), 20.0, n0, record=agk.RECORD_EVERY_STEP))
    w, f = oracle_pair(om, n0, dict(tol=1e-8), 20.0, record=O.RECORD_EVERY_STEP, records_capacity=100000)
    check_lockstep(g, w, f)
    check_run(g, w, f)


def test_record_stream_past_ring(agk, oracle_port):
    """More records than the device ring holds (1 << 16): the run pauses to drain the ring and
    every record comes back, identical in count and order to the reference's RunReport
    (simulator.cpp:130-145, 209-222). Fixed RK2 steps: the same decisions on both sides."""
    om, ws = build(agk, "constant", 64)
    n0 = np.zeros(64)
    n0[0] = 1.0
    ctl = dict(stepper=O.RK2, mode=O.FIXED, tau=1e-3)
    g = agk.run(ws, agk.SimulationConfig(agk.StepControl(**ctl), 150.0, n0, snapshot_times=[75.0],
                                         record=agk.RECORD_EVERY_STEP))
    w = oracle_port.run(om, n0, O.Control(**ctl), 150.0, snapshot_times=[75.0], record=O.RECORD_EVERY_STEP,
                        records_capacity=200000)
    assert g.num_records == w["num_records"] == len(g.records) > 140000
    assert [r["rhs_evals"] for r in g.records] == [r["rhs_evals"] for r in w["records"]]
    gt = np.array([r["t"] for r in g.records])
    wt = np.array([r["t"] for r in w["records"]])
    assert np.max(np.abs(gt - wt) / np.maximum(wt, 1.0)) <= 1e-12
    gd = np.array([r["density"] for r in g.records])
    wd = np.array([r["density"] for r in w["records"]])
    assert np.max(np.abs(gd / wd - 1.0)) <= 1e-9
    assert len(g.snapshots) == 1 and g.snapshots[0][0] == 75.0
