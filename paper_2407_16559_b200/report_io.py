"""Output formats of the reference's run and bench drivers over the device run loop (SURVEY §8f
item 2), byte-compatible with the reference:

  write_run_outputs   report_io.cpp:32-98   observables.csv, snapshot_<t>.csv, summary.txt,
                                            aborted.marker
  detect_oscillations analysis.cpp:76-118   density cycles / mean period in summary.txt
  run_bench           bench.cpp:27-98       (scheme x cell) grid of full runs with recording off;
                                            every cell is a device-resident run on the GPU
  format_bench_table  bench.cpp:100-134
  write_bench_outputs bench.cpp:136-171     bench_table.txt, bench_results.csv, bench_{evals,seconds}.csv

tests/test_report_io.py checks the files byte for byte against the reference's own writers
(oracle/_ref, compiled from the reference's sources).
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

STEPPER_NAMES = {0: "rk2", 1: "rk4", 2: "rkf45"}  # to_string(StepperKind), config.cpp:96-106
FIXED, ADAPTIVE = 0, 1


def format_full(x: float) -> str:
    """format_full (report_io.cpp:19-23): printf("%.16e")."""
    x = float(x)
    if math.isnan(x):
        return "-nan" if math.copysign(1.0, x) < 0 else "nan"
    if math.isinf(x):
        return "-inf" if x < 0 else "inf"
    return "%.16e" % x


def snapshot_filename(t: float) -> str:
    """snapshot_filename (report_io.cpp:25-29): snapshot_<%.17g>.csv."""
    return "snapshot_" + ("%.17g" % float(t)) + ".csv"


@dataclass
class OscillationSummary:
    peak_times: List[float] = field(default_factory=list)
    periods: List[float] = field(default_factory=list)
    amplitudes: List[float] = field(default_factory=list)
    cycle_count: int = 0


def detect_oscillations(t: Sequence[float], value: Sequence[float], prominence_fraction: float = 0.01):
    """detect_oscillations (analysis.cpp:76-118): strict local maxima whose topographic prominence
    is at least prominence_fraction of the series range."""
    t = np.asarray(t, dtype=np.float64)
    v = np.asarray(value, dtype=np.float64)
    if t.size != v.size:
        raise ValueError("time and value sizes differ")
    if t.size < 100:
        raise ValueError("need at least 100 records")
    if not np.all(t[1:] > t[:-1]):
        raise ValueError("times must be strictly increasing")
    out = OscillationSummary()
    rng = float(v.max() - v.min())
    if rng <= 0.0:
        return out
    min_prom = prominence_fraction * rng
    peaks = []
    n = v.size
    for i in range(1, n - 1):
        if not (v[i] > v[i - 1] and v[i] > v[i + 1]):
            continue
        left = v[i]
        for j in range(i - 1, -1, -1):
            if v[j] > v[i]:
                break
            left = min(left, v[j])
        right = v[i]
        for j in range(i + 1, n):
            if v[j] > v[i]:
                break
            right = min(right, v[j])
        if v[i] - max(left, right) >= min_prom:
            peaks.append(i)
    for p, i in enumerate(peaks):
        out.peak_times.append(float(t[i]))
        end = peaks[p + 1] if p + 1 < len(peaks) else n
        trough = v[i]
        for j in range(i + 1, end):
            trough = min(trough, v[j])
        out.amplitudes.append(float(v[i] - trough))
        if p > 0:
            out.periods.append(float(t[i] - t[peaks[p - 1]]))
    out.cycle_count = len(peaks) - 1 if peaks else 0
    return out


def write_run_outputs(report, directory: str) -> None:
    """write_run_outputs (report_io.cpp:32-98) for an agk.RunReport (or any object with the same
    fields: records as dicts, snapshots as (t, n) pairs)."""
    os.makedirs(directory, exist_ok=True)
    with open(os.path.join(directory, "observables.csv"), "w", newline="\n") as f:
        f.write("t,tau,N,M1,M2,err,rhs_evals,rejects\n")
        for r in report.records:
            f.write(",".join(format_full(r[k]) for k in ("t", "tau", "density", "mass", "m2", "error_estimate")))
            f.write(f",{int(r['rhs_evals'])},{int(r['rejects'])}\n")
    for t, n in report.snapshots:
        with open(os.path.join(directory, snapshot_filename(t)), "w", newline="\n") as f:
            f.write("k,n_k\n")
            f.write("".join(f"{k},{format_full(x)}\n" for k, x in enumerate(np.asarray(n), start=1)))
    completed = report.termination == "completed"
    with open(os.path.join(directory, "summary.txt"), "w", newline="\n") as f:
        f.write(f"termination = {'completed' if completed else 'aborted'}\n")
        if not completed:
            f.write(f"abort_reason = {report.abort_reason}\n")
            f.write(f"abort_t = {format_full(report.abort_t)}\n")
            f.write(f"abort_tau = {format_full(report.abort_tau)}\n")
        f.write(f"final_t = {format_full(report.final_t)}\n")
        f.write(f"total_rhs_evals = {int(report.total_rhs_evals)}\n")
        f.write(f"total_accepted = {int(report.total_accepted)}\n")
        f.write(f"total_rejects = {int(report.total_rejects)}\n")
        if len(report.records) >= 100:
            osc = detect_oscillations([r["t"] for r in report.records], [r["density"] for r in report.records])
            f.write(f"density_cycles = {osc.cycle_count}\n")
            if osc.cycle_count > 0:
                mean = 0.0
                for p in osc.periods:
                    mean += p
                mean /= len(osc.periods)
                f.write(f"density_mean_period = {format_full(mean)}\n")
        f.write(f"wall_seconds = {format_full(report.wall_seconds)}\n")
    if not completed:
        with open(os.path.join(directory, "aborted.marker"), "w", newline="\n") as f:
            f.write(f"{report.abort_reason} at t = {format_full(report.abort_t)}, tau = {format_full(report.abort_tau)}\n")


@dataclass
class BenchCell:
    """BenchCell (config.hpp:21-26): a fixed step tau or an adaptive tolerance."""
    mode: int = ADAPTIVE
    value: float = 0.0


@dataclass
class BenchResult:
    """BenchResult (bench.hpp:13-22)."""
    scheme: int
    cell: BenchCell
    rhs_evals: int = 0
    accepted: int = 0
    rejected: int = 0
    wall_seconds: float = 0.0
    completed: bool = False
    note: str = ""


def _cell_label(cell: BenchCell) -> str:
    return ("fixed tau=" if cell.mode == FIXED else "adaptive tol=") + ("%g" % cell.value)


def run_bench(ws, t_end: float, initial, schemes: Sequence[int], cells: Sequence[BenchCell],
              initial_tau: float = 0.0, base_control=None) -> List[BenchResult]:
    """run_bench (bench.cpp:27-98): every (scheme, cell) as a full run with recording off and
    no snapshots; an aborted or failing cell is reported in place. The reference spreads cells
    over host threads; here each cell is one device-resident run (agk.run) on the workspace's
    GPU, and bench.py / replicas.py spread independent grids over GPUs."""
    import paper_2407_16559_b200 as agk
    if not schemes or not cells:
        raise ValueError("bench mode needs bench_schemes and bench_cells")
    out = []
    for sch in schemes:
        for cell in cells:
            res = BenchResult(sch, cell)
            kw = dict(base_control.__dict__) if base_control is not None else {}
            kw.update(stepper=sch, mode=cell.mode)
            if cell.mode == FIXED:
                kw.update(tau=cell.value, tol=0.0)
            else:
                kw.update(tol=cell.value, tau=0.0)
            try:
                rep = agk.run(ws, agk.SimulationConfig(agk.StepControl(**kw), t_end, initial, initial_tau))
                res.rhs_evals, res.accepted, res.rejected = rep.total_rhs_evals, rep.total_accepted, rep.total_rejects
                res.wall_seconds = rep.wall_seconds
                res.completed = rep.termination == "completed"
                if not res.completed:
                    res.note = rep.abort_reason + (" at t=%g" % rep.abort_t)
            except (ValueError, RuntimeError) as e:
                res.completed = False
                res.note = str(e)
            out.append(res)
    return out


def format_bench_table(schemes: Sequence[int], cells: Sequence[BenchCell], results: Sequence[BenchResult]) -> str:
    """format_bench_table (bench.cpp:100-134): rows = schemes, columns = cells, 'seconds / evals'."""
    headers = ["scheme"] + [_cell_label(c) for c in cells]
    rows = []
    for r, sch in enumerate(schemes):
        row = [STEPPER_NAMES[sch]]
        for c in range(len(cells)):
            res = results[r * len(cells) + c]
            row.append("%.3f / %d" % (res.wall_seconds, res.rhs_evals) if res.completed else "aborted: " + res.note)
        rows.append(row)
    widths = [max([len(headers[c])] + [len(row[c]) for row in rows]) for c in range(len(headers))]
    lines = []
    for row in [headers] + rows:
        lines.append("".join(x + " " * (widths[c] - len(x) + 2) for c, x in enumerate(row)) + "\n")
    return "".join(lines)


def write_bench_outputs(schemes: Sequence[int], cells: Sequence[BenchCell], results: Sequence[BenchResult],
                        directory: str) -> None:
    """write_bench_outputs (bench.cpp:136-171)."""
    os.makedirs(directory, exist_ok=True)
    with open(os.path.join(directory, "bench_table.txt"), "w", newline="\n") as f:
        f.write(format_bench_table(schemes, cells, results))
    with open(os.path.join(directory, "bench_results.csv"), "w", newline="\n") as f:
        f.write("scheme,mode,value,rhs_evals,accepted,rejected,wall_seconds,status\n")
        for res in results:
            f.write(f"{STEPPER_NAMES[res.scheme]},{'fixed' if res.cell.mode == FIXED else 'adaptive'},"
                    f"{format_full(res.cell.value)},{res.rhs_evals},{res.accepted},{res.rejected},"
                    f"{format_full(res.wall_seconds)},{'completed' if res.completed else 'aborted: ' + res.note}\n")
    for which in ("evals", "seconds"):
        with open(os.path.join(directory, f"bench_{which}.csv"), "w", newline="\n") as f:
            f.write("scheme" + "".join("," + _cell_label(c) for c in cells) + "\n")
            for r, sch in enumerate(schemes):
                f.write(STEPPER_NAMES[sch])
                for c in range(len(cells)):
                    res = results[r * len(cells) + c]
                    f.write(",")
                    if not res.completed:
                        f.write("aborted")
                    elif which == "evals":
                        f.write(str(res.rhs_evals))
                    else:
                        f.write(format_full(res.wall_seconds))
                f.write("\n")
