"""Byte compatibility of paper_2407_16559_b200/report_io.py with the reference's writers
(report_io.cpp:32-98, analysis.cpp:76-118, bench.cpp:100-171), compiled from the reference's own
sources into oracle/_ref (skipped where the reference is not present). The run reports come from
the CPU oracle here; on the GPU box the same writer serves agk.run's reports (test at the end)."""
import ctypes as C
import os
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_16559_b200 import report_io as R


def read_dir(d):
    return {f: open(os.path.join(d, f), "rb").read() for f in sorted(os.listdir(d))}


def as_report(rep, snapshot_times, abort_reason, wall):
    """An oracle run dict in the shape of agk.RunReport."""
    return SimpleNamespace(
        termination="completed" if rep["termination"] == 0 else "aborted", abort_reason=abort_reason,
        abort_t=rep["abort_t"], abort_tau=rep["abort_tau"], final_t=rep["final_t"],
        snapshots=[(float(t), rep["snapshots"][q]) for q, t in enumerate(snapshot_times[:len(rep["snapshots"])])],
        records=rep["records"], total_rhs_evals=rep["total_rhs_evals"], total_accepted=rep["total_accepted"],
        total_rejects=rep["total_rejects"], wall_seconds=wall)


def ref_write(ref, rep, m, snapshot_times, abort_reason, wall, d):
    recs = (O._Record * max(len(rep.records), 1))()
    for q, r in enumerate(rep.records):
        recs[q] = O._Record(r["t"], r["tau"], r["density"], r["mass"], r["m2"], r["error_estimate"],
                            r["rhs_evals"], r["rejects"])
    snaps = np.ascontiguousarray(np.array([n for _, n in rep.snapshots] or [np.zeros(m)]), dtype=np.float64)
    st = np.ascontiguousarray(snapshot_times if len(snapshot_times) else [0.0], dtype=np.float64)
    c = O._Report()
    c.termination = 0 if rep.termination == "completed" else 1
    c.abort_t, c.abort_tau, c.final_t = rep.abort_t, rep.abort_tau, rep.final_t
    c.total_rhs_evals, c.total_accepted, c.total_rejects = rep.total_rhs_evals, rep.total_accepted, rep.total_rejects
    c.final_state = None
    c.snapshots = snaps.ctypes.data_as(O._dp)
    c.num_snapshots_taken = len(rep.snapshots)
    c.records = recs
    c.records_capacity = len(rep.records)
    c.num_records = len(rep.records)
    fn = ref.lib.ref_write_run_outputs
    fn.restype = C.c_int
    assert fn(C.byref(c), C.c_size_t(m), st.ctypes.data_as(O._dp), abort_reason.encode(), C.c_double(wall),
              d.encode()) == 0


@pytest.mark.parametrize("case", ["records", "interval_snapshots", "aborted", "oscillating"])
def test_run_outputs_byte_identical(oracle_port, oracle_ref, tmp_path, case):
    m = 96
    u, v = O.constant_factors(m)
    model = O.Model(u, v)
    n0 = np.zeros(m)
    n0[0] = 1.0
    snaps = [0.5, 1.0, 3.0]
    abort_reason = ""
    if case == "records":
        rep = oracle_port.run(model, n0, O.Control(tol=1e-8), 4.0, snapshot_times=snaps,
                              record=O.RECORD_EVERY_STEP, records_capacity=10000)
    elif case == "interval_snapshots":
        rep = oracle_port.run(model, n0, O.Control(stepper=O.RK4, tol=1e-7), 3.0, snapshot_times=snaps,
                              record=O.RECORD_INTERVAL, record_interval=0.25, records_capacity=10000)
    elif case == "aborted":
        rep = oracle_port.run(model, n0, O.Control(tol=1e-8, tau_min=1.0), 4.0, snapshot_times=snaps,
                              record=O.RECORD_EVERY_STEP, records_capacity=10000)
        assert rep["termination"] == 1
        abort_reason = "step size underflow"
    else:
        # a damped oscillation of >= 100 records exercises detect_oscillations in summary.txt
        t = np.linspace(0.0, 20.0, 400)
        rep = dict(termination=0, abort_t=0.0, abort_tau=0.0, final_t=20.0, total_rhs_evals=2400,
                   total_accepted=400, total_rejects=3, snapshots=[],
                   records=[dict(t=float(x), tau=0.05, density=float(1 + np.exp(-x / 10) * np.sin(2 * x)),
                                 mass=1.0, m2=float(1 + x), error_estimate=1e-9, rhs_evals=6 * q, rejects=0)
                            for q, x in enumerate(t)])
    wall = 0.123456789
    r = as_report(rep, snaps, abort_reason, wall)
    R.write_run_outputs(r, str(tmp_path / "py"))
    ref_write(oracle_ref, r, m, snaps, abort_reason, wall, str(tmp_path / "ref"))
    a, b = read_dir(tmp_path / "py"), read_dir(tmp_path / "ref")
    assert a.keys() == b.keys()
    for k in a:
        assert a[k] == b[k], k
    if case == "oscillating":
        assert b"density_cycles" in a["summary.txt"]


def test_bench_outputs_byte_identical(oracle_ref, tmp_path):
    schemes = [O.RK2, O.RK4, O.RKF45]
    cells = [R.BenchCell(R.FIXED, 0.01), R.BenchCell(R.ADAPTIVE, 1e-4), R.BenchCell(R.ADAPTIVE, 1e-8)]
    rng = np.random.default_rng(5)
    results = []
    for s in schemes:
        for c in cells:
            ok = not (s == O.RK2 and c.value == 1e-8)
            results.append(R.BenchResult(s, c, int(rng.integers(1, 10 ** 6)), int(rng.integers(1, 10 ** 5)),
                                         int(rng.integers(0, 100)), float(rng.random() * 100), ok,
                                         "" if ok else "too many rejected trials at t=3.25"))
    R.write_bench_outputs(schemes, cells, results, str(tmp_path / "py"))
    ns, nc = len(schemes), len(cells)
    arr = lambda xs, t: (t * len(xs))(*xs)  # noqa: E731
    notes = (C.c_char_p * (ns * nc))(*[r.note.encode() for r in results])
    fn = oracle_ref.lib.ref_write_bench_outputs
    fn.restype = C.c_int
    assert fn(arr(schemes, C.c_int), C.c_size_t(ns), arr([c.mode for c in cells], C.c_int),
              arr([c.value for c in cells], C.c_double), C.c_size_t(nc),
              arr([r.rhs_evals for r in results], C.c_uint64), arr([r.accepted for r in results], C.c_uint64),
              arr([r.rejected for r in results], C.c_uint64), arr([r.wall_seconds for r in results], C.c_double),
              arr([int(r.completed) for r in results], C.c_int), notes, str(tmp_path / "ref").encode()) == 0
    a, b = read_dir(tmp_path / "py"), read_dir(tmp_path / "ref")
    assert a.keys() == b.keys()
    for k in a:
        assert a[k] == b[k], k


def test_format_full_specials():
    assert R.format_full(1.0) == "1.0000000000000000e+00"
    assert R.format_full(-2.5e-300) == "-2.5000000000000000e-300"
    assert R.format_full(float("inf")) == "inf" and R.format_full(float("nan")) == "nan"
    assert R.snapshot_filename(0.1) == "snapshot_0.10000000000000001.csv"


@pytest.mark.gpu
def test_device_run_report_and_bench_grid(agk, tmp_path):
    """The writers on agk.run's device reports, and run_bench's grid on the GPU."""
    m = 128
    u, v = O.constant_factors(m)
    ws = agk.RhsWorkspace(agk.Model(u, v))
    n0 = np.zeros(m)
    n0[0] = 1.0
    rep = agk.run(ws, agk.SimulationConfig(agk.StepControl(tol=1e-8), 4.0, n0, snapshot_times=[1.0, 4.0],
                                           record=agk.RECORD_EVERY_STEP))
    R.write_run_outputs(rep, str(tmp_path / "run"))
    files = read_dir(tmp_path / "run")
    assert set(files) == {"observables.csv", "summary.txt", "snapshot_1.csv", "snapshot_4.csv"}
    assert files["observables.csv"].count(b"\n") == len(rep.records) + 1
    res = R.run_bench(ws, 2.0, n0, [agk.RK2, agk.RKF45], [R.BenchCell(R.FIXED, 0.05), R.BenchCell(R.ADAPTIVE, 1e-6)])
    assert all(r.completed for r in res) and res[0].rhs_evals == 40 * 2   # 40 fixed RK2 steps
    R.write_bench_outputs([agk.RK2, agk.RKF45], [R.BenchCell(R.FIXED, 0.05), R.BenchCell(R.ADAPTIVE, 1e-6)], res,
                          str(tmp_path / "bench"))
    assert b"adaptive tol=1e-06" in read_dir(tmp_path / "bench")["bench_table.txt"]
