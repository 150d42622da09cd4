#!/usr/bin/env python3
"""bench.py — RHS evaluations/s of the low-rank Smoluchowski operator on B200 (BASELINE config 4).

Workload (BASELINE.json configs[3], the configuration the headline metric is quoted on):
random positive low-rank kernel, R = 16, M = 2^20, fp64, seeded synthetic inputs
(paper_2407_16559_b200/configs.py). One "step" = one eval_rhs over the state vector.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

* value: K evaluations per rank on device-resident inputs, device time from CUDA events on the
  handle's stream around captured graphs of 10 chained evaluations (max over ranks); U/V exceed the
  126 MB L2, so every evaluation streams them from HBM (no flush needed).
* e2e: the same metric through the public C ABI (agk_rhs_eval) with pinned HOST buffers: the
  H2D copy of n and the D2H copy of S(n) are inside the timed region every step; `callers` host
  threads (default 4: copies in both directions overlap the other callers' kernels), each with its
  own workspace, call concurrently, at least 60 calls in all (the reference's bench runs
  cells on threads too), so copies overlap kernels; the one-caller figure is reported beside it.
* roofline: the dominant kernel's algorithmic bytes per launch / its event-timed duration.
* cpu_baseline: the reference compiled from its own sources (oracle/_ref), single thread, on a
  bounded sample (2 evaluations) on rank 0.
* adaptive: the metric's time-to-t_end half, live: config 5 (M = 2^20, Brownian + source) RKF45
  on the device to t = 200 (a prefix of t_end = 1e5; full horizons in profiles/runs_*.json).
* --impl reference: the reference's CPU implementation on all host cores (one independent
  evaluation per thread, as the reference's own bench runs cells on std::threads).
* N > 1: replicas only (the path does not shard): one independent workload per GPU,
  no data-path collective; torch.distributed is used only for the barrier and max-over-ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RHS evals/s + HBM GB/s (M=2^20,R=16,fp64); adaptive solve time to t_end"
UNIT = "RHS evals/s"
M, R = 1 << 20, 16


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-callers", type=int, default=4)
    ap.add_argument("--ref-budget-s", type=float, default=240.0)
    ap.add_argument("--adaptive-horizon", type=float, default=200.0,
                    help="config-5 RKF45 adaptive solve to this t (0: skip); t_end is 1e5")
    ap.add_argument("--no-t-end", action="store_true", help="skip the time-to-t_end legs (configs 1, 2)")
    return ap.parse_args()


def spawn_replicas(args):
    """--gpus N without a torchrun environment: launch the N replicas ourselves (one process per
    GPU, the same torch.distributed.run command the driver uses) and pass their exit code on."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ------------------------------------------------------------------ distributed plumbing
# replicas only (paper_2407_16559_b200/replicas.py): barrier + max over ranks, no data exchange

def dist_setup():
    from paper_2407_16559_b200 import replicas
    return replicas.setup("nccl" if int(os.environ.get("WORLD_SIZE", "1")) > 1 else None)


def barrier(world):
    from paper_2407_16559_b200 import replicas
    replicas.barrier(world)


def max_over_ranks(x, world, local):
    from paper_2407_16559_b200 import replicas
    return replicas.max_over_ranks(x, world, local)


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ algorithmic counts

def survey_bytes(m, r, rf):
    """SURVEY §8d two-pass model bytes_alg = M (88 + 16R + 72R_f) and the compulsory 8M(2R+2)."""
    return m * (88 + 16 * r + 72 * rf), 8 * m * (2 * r + 2)


def survey_flops(m, rf):
    p = 1
    while p < 2 * m:
        p *= 2
    lg = p.bit_length() - 1
    return 5 * p * lg * (rf + 0.5) + 18 * p * rf


def kernel_counts(cls, m, r, rf, plan, first, g):
    """Algorithmic HBM bytes and fp64 flops of ONE launch of a fast-path kernel class at P = 2^21
    (DESIGN.md §3): the bytes each kernel must move at minimum, the flops of 5 N log2 N per
    transform plus the pointwise work."""
    log2p, n1, n2, gs = plan
    p = 1 << log2p
    l1, l2 = n1.bit_length() - 1, n2.bit_length() - 1
    if cls == "transpose":
        return 8 * m + 8 * (p // 2), 0
    if cls == "col_fwd":  # n grid + (U, V) columns + Y write, per rank in the group
        return 8 * (p // 2) + 16 * (p // 2) * g + 16 * p * g, g * (5 * p * l1 + 6 * p)
    if cls == "row":  # Y read + accumulator rows (+ read when not the first group); last: inverse rows
        acc = 16 * (n1 // 2 + 1) * n2
        return 16 * p * g + acc * (1 if first else 2), g * (5 * p * l2 + 9 * p) + 5 * (p // 2) * l2
    if cls == "dvec":  # U^T rows, n, D
        return 8 * m * r + 16 * m, 2 * m * r
    if cls == "col_inv":  # G half rows, D, S
        return 16 * (n1 // 2 + 1) * n2 + 16 * m, 5 * (p // 2) * l1
    return 8 * m * (2 * r + 2), survey_flops(m, rf)


def load_ncu_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return {}


# ------------------------------------------------------------------ arms

def cpu_baseline_sample(U, V, n, evals=2):
    from oracle.oracle import Model, Oracle
    try:
        o, kind = Oracle("reference"), "reference"
    except FileNotFoundError:
        o, kind = Oracle("port"), "port"
    md = Model(U, V)
    t0 = time.perf_counter()
    for _ in range(evals):
        o.eval_rhs(md, n)
    dt = time.perf_counter() - t0
    return {"value": evals / dt, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{evals} eval_rhs at M=2^20, R=16 (config 4), single thread, {dt:.1f} s"}


def run_reference(args, world, rank):
    """The reference's own CPU eval_rhs (oracle/_ref) on all host threads."""
    if rank != 0:
        return None
    from paper_2407_16559_b200.configs import random_config4
    from oracle.oracle import Model, Oracle
    try:
        o, kind = Oracle("reference"), "reference"
    except FileNotFoundError:
        o, kind = Oracle("port"), "port"
    U, V, n = random_config4(M, R)
    md = Model(U, V)
    cores = os.cpu_count() or 1

    def one_round():
        ths = [threading.Thread(target=o.eval_rhs, args=(md, n)) for _ in range(cores)]
        t0 = time.perf_counter()
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return time.perf_counter() - t0

    for _ in range(max(1, min(args.warmup, 1))):
        one_round()
    times = []
    t_start = time.perf_counter()
    for _ in range(args.steps):
        times.append(one_round())
        if time.perf_counter() - t_start > args.ref_budget_s:
            break
    total = sum(times)
    value = cores * len(times) / total
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "steps_timed": len(times), "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config4: low-rank RHS M=2^20 R=16 random kernel (seed 0x5eed5eed)",
                   "m": M, "r": R, "threads": cores},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{cores} concurrent eval_rhs per step (one per host thread), "
                                   f"{len(times)} step(s) timed"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def run_b200(args, world, rank, local):
    import torch
    import paper_2407_16559_b200 as agk
    from paper_2407_16559_b200.configs import random_config4

    torch.cuda.set_device(local)
    U, V, n = random_config4(M, R)
    ws = agk.RhsWorkspace(agk.Model(U, V), device=local)
    rf = ws.unique_ranks()
    n_dev = torch.from_numpy(n).to(f"cuda:{local}")
    out_dev = torch.empty_like(n_dev)
    launches = ws.launches_per_eval()

    agk.eval_rhs_timed(ws, n_dev, out_dev, max(args.warmup, 3))  # warm-up (graph capture inside)
    with ClockSampler(local) as clk:
        # keep the GPU under this same load until the sampler reports, so the clocks recorded
        # bracket the timed region (which alone is shorter than nvidia-smi's sampling period)
        t_load = time.perf_counter()
        while time.perf_counter() - t_load < 0.6 or (not clk.lines and time.perf_counter() - t_load < 5):
            agk.eval_rhs_timed(ws, n_dev, out_dev, 50)
        barrier(world)
        torch.cuda.synchronize()
        ms = agk.eval_rhs_timed(ws, n_dev, out_dev, args.steps)
        torch.cuda.synchronize()
        barrier(world)
        agk.eval_rhs_timed(ws, n_dev, out_dev, 200)
    ms = max_over_ranks(ms, world, local)
    sec = ms * 1e-3
    value = world * args.steps / sec

    # end to end through the public API with pinned host buffers: `callers` host threads, each
    # with its own workspace (the reference's one-workspace-per-concurrent-caller rule,
    # rhs.hpp:42-44), every call = H2D of n + the RHS + D2H of S(n) + sync, so one caller's copies
    # run on the copy engines while another's kernels run. value = all calls / wall time.
    lib = agk.load_library()
    callers = max(1, args.e2e_callers)
    wss = [ws] + [agk.RhsWorkspace(agk.Model(U, V), device=local) for _ in range(callers - 1)]
    h_in = [torch.from_numpy(n).pin_memory() for _ in wss]
    h_out = [torch.empty(M, dtype=torch.float64).pin_memory() for _ in wss]

    def calls(q, count):
        torch.cuda.set_device(local)
        for _ in range(count):
            agk._check(lib.agk_rhs_eval(wss[q].handle, h_in[q].data_ptr(), h_out[q].data_ptr(), agk.MEM_HOST),
                       wss[q].handle)

    def timed_calls(count_per_caller):
        ths = [threading.Thread(target=calls, args=(q, count_per_caller)) for q in range(len(wss))]
        t0 = time.perf_counter()
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return time.perf_counter() - t0

    timed_calls(2)
    calls(0, 2)
    barrier(world)
    t0 = time.perf_counter()
    calls(0, args.steps)
    single_sec = max_over_ranks(time.perf_counter() - t0, world, local)
    barrier(world)
    per = max(1, max(args.steps, 60) // callers)
    e2e_sec = max_over_ranks(timed_calls(per), world, local)
    for extra in wss[1:]:
        extra.close()
    e2e = {"value": world * per * callers / e2e_sec, "unit": UNIT, "h2d_bytes_per_step": 8 * M,
           "d2h_bytes_per_step": 8 * M, "callers": callers,
           "single_caller_value": world * args.steps / single_sec}

    # per-kernel roofline of the dominant kernel
    prof, plan = agk.profile_rhs(ws, n_dev, out_dev, reps=5)
    by_cls = {}
    first_row = True
    g = plan[3]
    per_launch = []
    for cls, kms in prof:
        first = first_row if cls == "row" else True
        if cls == "row":
            first_row = False
        b, f = kernel_counts(cls, M, R, rf, plan, first, g)
        per_launch.append((cls, kms, b, f))
        d = by_cls.setdefault(cls, {"ms": 0.0, "bytes": 0, "flops": 0, "launches": 0})
        d["ms"] += kms
        d["bytes"] += b
        d["flops"] += f
        d["launches"] += 1
    total_ms = sum(d["ms"] for d in by_cls.values())
    dom = max(by_cls, key=lambda c: by_cls[c]["ms"])
    dd = by_cls[dom]
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
        hbm_peak, hbm_src = float(peaks["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    except Exception:
        hbm_peak, hbm_src = 6650.0, "B200_PROFILING.md fallback"
    fp64_peak = 33.8  # TFLOP/s, DFMA microbenchmark on this pool (profiles/probe_r01.txt)
    avg_ms = dd["ms"] / dd["launches"]
    ach_gbs = dd["bytes"] / dd["launches"] / (avg_ms * 1e-3) / 1e9
    ach_tf = dd["flops"] / dd["launches"] / (avg_ms * 1e-3) / 1e12
    traffic = load_ncu_traffic().get(dom)
    b_alg, b_comp = survey_bytes(M, R, rf)
    per_rhs_s = sec / args.steps * world
    roofline = {
        "bound": "hbm", "kernel": dom, "achieved": ach_gbs, "peak": hbm_peak, "unit": "GB/s",
        "frac": ach_gbs / hbm_peak, "traffic": traffic, "peak_source": hbm_src,
        "share_of_step": dd["ms"] / total_ms, "avg_launch_ms": avg_ms, "launches_per_step": dd["launches"],
        "alg_bytes_per_launch": dd["bytes"] / dd["launches"],
        "fp64": {"achieved_tflops": ach_tf, "peak_tflops": fp64_peak, "frac": ach_tf / fp64_peak,
                 "alg_flops_per_launch": dd["flops"] / dd["launches"],
                 "peak_source": "DFMA microbenchmark, profiles/probe_r01.txt"},
        "per_class_ms": {c: by_cls[c]["ms"] for c in by_cls},
        "per_class": {c: {"ms": d["ms"], "alg_bytes": d["bytes"], "gbs": d["bytes"] / (d["ms"] * 1e-3) / 1e9,
                          "hbm_frac": d["bytes"] / (d["ms"] * 1e-3) / 1e9 / hbm_peak,
                          "fp64_frac": d["flops"] / (d["ms"] * 1e-3) / 1e12 / fp64_peak}
                      for c, d in by_cls.items() if d["ms"] > 0},
        "whole_rhs": {"bytes_alg_survey": b_alg, "bytes_compulsory": b_comp, "flops_alg": survey_flops(M, rf),
                      "gbs_survey_model": b_alg / per_rhs_s / 1e9,
                      "frac_survey_model": b_alg / per_rhs_s / 1e9 / hbm_peak,
                      "frac_compulsory": b_comp / per_rhs_s / 1e9 / hbm_peak,
                      "fp64_frac": survey_flops(M, rf) / per_rhs_s / 1e12 / fp64_peak},
    }
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config4: low-rank RHS M=2^20 R=16 random kernel (seed 0x5eed5eed)",
                   "m": M, "r": R, "unique_ranks": rf, "plan": {"log2p": plan[0], "n1": plan[1], "n2": plan[2],
                                                               "ranks_per_group": plan[3]},
                   "l2": "inputs (U,V 256 MiB) larger than the 126 MB L2; no flush", "parallelism": f"replicas{world}"},
        "e2e": e2e, "roofline": roofline, "gpu_launches": launches * args.steps,
        "clocks": clk.summary(),
    }
    ws.close()
    if args.adaptive_horizon > 0:
        res["adaptive"] = adaptive_leg(args, world, local)
    if not args.no_t_end:
        res["t_end"] = t_end_legs(args, world, rank, local)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline_sample(U, V, n)
    return res


def adaptive_leg(args, world, local):
    """The metric's second half, measured live: a device-resident adaptive solve of BASELINE
    config 5 (Brownian kernel + monomer source, M = 2^20, R = 3, n0 = 0, RKF45, tol 1e-6) to
    t = --adaptive-horizon, a prefix of its t_end = 1e5 (the full horizons are tools/runs.py runs,
    profiles/runs_*.json). Wall time around agk.run (graph build excluded: built by a first short
    run), accepted steps/s and the in-run time per RHS evaluation."""
    import torch
    import paper_2407_16559_b200 as agk
    from paper_2407_16559_b200.configs import baseline_config
    cfg = baseline_config(5)
    ws = agk.RhsWorkspace(agk.Model(cfg["u"], cfg["v"], cfg["variant"], cfg["sources"], cfg["lam"]), device=local)
    ctl = agk.StepControl(stepper=agk.RKF45, tol=cfg["tol"])
    agk.run(ws, agk.SimulationConfig(ctl, 1.0, cfg["n0"]))  # builds and instantiates the step graph
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = agk.run(ws, agk.SimulationConfig(ctl, args.adaptive_horizon, cfg["n0"]))
    wall = max_over_ranks(time.perf_counter() - t0, world, local)
    ws.close()
    return {"workload": f"config5 RKF45 tol 1e-6, M=2^20 R=3, t in [0, {args.adaptive_horizon:g}] (t_end 1e5)",
            "termination": rep.termination, "final_t": rep.final_t, "wall_s": wall,
            "accepted": rep.total_accepted, "rejects": rep.total_rejects, "rhs_evals": rep.total_rhs_evals,
            "accepted_steps_per_s": world * rep.total_accepted / wall,
            "us_per_rhs_in_run": 1e6 * wall / max(rep.total_rhs_evals, 1)}


def t_end_legs(args, world, rank, local):
    """Time to t_end (the metric's second half) on full BASELINE configs, each beside the
    reference's own CPU run() on this box's host (oracle/_ref, one core: run() is single-threaded):
      * config 1 (M=4096, constant kernel, t_end=100) with each of the three schemes: GPU and CPU
        both measured in full;
      * config 2 (M=2^16, Brownian+2 with a monomer source, n0=0, t_end=1e4) RKF45: GPU in full;
        the CPU time is EXTRAPOLATED as (measured CPU seconds per RHS at this shape) x (the run's
        RHS count), since the full CPU run takes hours.
    GPU wall time is around agk.run (graph built by a first short run), device-resident."""
    import torch
    import paper_2407_16559_b200 as agk
    from paper_2407_16559_b200.configs import baseline_config
    try:
        from oracle.oracle import Control as OC, Model as OM, Oracle
        ref = Oracle("reference")
    except Exception:
        ref = None
    legs = []
    for idx, schemes in ((1, (agk.RK2, agk.RK4, agk.RKF45)), (2, (agk.RKF45,))):
        cfg = baseline_config(idx)
        ws = agk.RhsWorkspace(agk.Model(cfg["u"], cfg["v"], cfg["variant"], cfg["sources"], cfg["lam"]),
                              device=local)
        for st in schemes:
            ctl = agk.StepControl(stepper=st, tol=cfg["tol"])
            agk.run(ws, agk.SimulationConfig(ctl, min(cfg["t_end"], 1e-3), cfg["n0"]))  # graph build
            barrier(world)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep = agk.run(ws, agk.SimulationConfig(ctl, cfg["t_end"], cfg["n0"]))
            wall = max_over_ranks(time.perf_counter() - t0, world, local)
            leg = {"config": idx, "scheme": ("rk2", "rk4", "rkf45")[st], "t_end": cfg["t_end"],
                   "m": int(cfg["n0"].size), "termination": rep.termination, "final_t": rep.final_t,
                   "gpu_wall_s": wall, "accepted": rep.total_accepted, "rejects": rep.total_rejects,
                   "rhs_evals": rep.total_rhs_evals, "accepted_steps_per_s": world * rep.total_accepted / wall,
                   "us_per_rhs_in_run": 1e6 * wall / max(rep.total_rhs_evals, 1)}
            if ref is not None and rank == 0:
                md = OM(cfg["u"], cfg["v"], cfg["variant"], list(cfg["sources"]), cfg["lam"])
                if idx == 1:
                    t0 = time.perf_counter()
                    w = ref.run(md, cfg["n0"], OC(stepper=st, tol=cfg["tol"]), cfg["t_end"])
                    cpu = time.perf_counter() - t0
                    leg["cpu_reference"] = {"wall_s": cpu, "kind": "measured", "cores": 1,
                                            "accepted": w["total_accepted"], "rhs_evals": w["total_rhs_evals"]}
                else:
                    k = 20
                    x = np.abs(np.random.default_rng(1).standard_normal(cfg["n0"].size)) * 1e-3
                    ref.eval_rhs(md, x)
                    t0 = time.perf_counter()
                    for _ in range(k):
                        ref.eval_rhs(md, x)
                    per = (time.perf_counter() - t0) / k
                    leg["cpu_reference"] = {"wall_s": per * rep.total_rhs_evals, "kind": "extrapolated", "cores": 1,
                                            "s_per_rhs": per, "sample": f"{k} eval_rhs at this shape x the GPU "
                                                                        "run's RHS count"}
                leg["speedup_vs_cpu"] = leg["cpu_reference"]["wall_s"] / wall
            legs.append(leg)
        ws.close()
    return legs


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_replicas(args))
    world, rank, local = dist_setup()
    if world != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; reporting the true rank count",
              file=sys.stderr)
    if args.impl == "reference":
        res = run_reference(args, world, rank)
    else:
        res = run_b200(args, world, rank, local)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)
    from paper_2407_16559_b200 import replicas
    replicas.teardown(world)


if __name__ == "__main__":
    main()
