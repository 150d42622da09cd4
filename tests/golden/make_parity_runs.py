"""Full-integration parity goldens from the REFERENCE itself (oracle/_ref), TEST INFRASTRUCTURE.

SURVEY §8d's parity plan (VERDICT r1 "Next round" item 1): full-shape prefixes and reduced-M full
horizons of BASELINE configs 1, 2, 3 and 5, run by the reference's own run() (simulator.cpp:
112-229, compiled from /root/reference sources by oracle/Makefile), plus the same case run by a
second, equally valid CPU build (the C restatement with FMA contraction, or with a 2x-padded FFT)
whose distance from the reference is the CPU-vs-CPU noise floor reported beside every GPU number.

Run here (where /root/reference exists), one process per case (they are single-threaded):

    python tests/golden/make_parity_runs.py --list
    python tests/golden/make_parity_runs.py CASE [--floor port_fma]
    python tests/golden/make_parity_runs.py CASE --which floor --floor port_pad2 --leg floor2

(a second floor build, the restatement with a 2x-padded FFT, i.e. a different FFT roundoff pattern:
the floor of a case is the larger of its floor legs)

Writes tests/golden/parity/CASE__ref.npz and CASE__floor.npz. The state is stored compactly: the head of the final state
up to the last index with n_s > 1e-13 max n (everything that can move the normwise or element-wise
bars) and the max |n_s| of the tail beyond it.
"""
import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402

OUT = os.path.join(HERE, "parity")
HEAD_REL = 1e-13

# BASELINE.json configs: (kernel, variant, sources, lambda, initial, tol)
CONFIG = {
    1: ("constant", O.AGGREGATION, [], 0.0, "mono", 1e-6),
    2: ("brownian2", O.SOURCES, [(1, 1.0)], 0.0, "zero", 1e-6),
    3: ("brownian0.9", O.SHATTERING, [], 0.01, "mono", 1e-8),
    5: ("brownian2", O.SOURCES, [(1, 1.0)], 0.0, "zero", 1e-6),
}
STEPPERS = {"rk2": O.RK2, "rk4": O.RK4, "rkf45": O.RKF45}

# name -> (config, m, stepper, t_end)
CASES = {}
for s in STEPPERS:
    CASES[f"c1_full_{s}"] = (1, 4096, s, 100.0)                 # config 1, full shape and horizon
    CASES[f"c2_m4096_{s}"] = (2, 4096, s, 1e4)                  # config 2 full horizon, reduced M
    CASES[f"c5_m4096_{s}"] = (5, 4096, s, 1e5)                  # config 5 full horizon, reduced M
    CASES[f"c5_full_t2_{s}"] = (5, 1 << 20, s, 2.0)             # config 5 full shape, prefix
CASES["c3_m2048_rkf45"] = (3, 2048, "rkf45", 5000.0)            # config 3 full horizon, reduced M
CASES["c3_full_t1_rkf45"] = (3, 1 << 17, "rkf45", 1.0)          # config 3 full shape, prefix
CASES["c2_full_rkf45"] = (2, 1 << 16, "rkf45", 1e4)             # config 2 full shape and horizon


def model_for(cfg, m):
    kind, var, srcs, lam, init, tol = CONFIG[cfg]
    if kind == "constant":
        u, v = O.constant_factors(m)
    elif kind == "brownian2":
        u, v = O.brownian_plus2_factors(m)
    else:
        u, v = O.brownian_factors(m, float(kind[len("brownian"):]))
    n0 = np.zeros(m)
    if init == "mono":
        n0[0] = 1.0
    return O.Model(u, v, var, list(srcs), lam), n0, tol


def case_inputs(name):
    cfg, m, st, t_end = CASES[name]
    md, n0, tol = model_for(cfg, m)
    ctl = O.Control(stepper=STEPPERS[st], mode=O.ADAPTIVE, tol=tol)
    return md, n0, ctl, t_end


def summarize(r):
    x = np.asarray(r["final_state"])
    k = np.arange(1, x.size + 1, dtype=np.float64)
    mx = float(np.max(np.abs(x))) if x.size else 0.0
    sig = np.nonzero(np.abs(x) > HEAD_REL * mx)[0]
    head = int(sig[-1]) + 1 if sig.size else 0
    out = dict(termination=int(r["termination"]), final_t=float(r["final_t"]),
               accepted=int(r["total_accepted"]), rejects=int(r["total_rejects"]),
               rhs_evals=int(r["total_rhs_evals"]), N=float(x.sum()), M1=float(np.dot(k, x)),
               M2=float(np.dot(k * k, x)), n1=float(x[0]), maxn=mx,
               head=x[:head].copy(), tail_maxabs=float(np.max(np.abs(x[head:]))) if head < x.size else 0.0)
    return compact(out)


def compact(out, keep=1 << 17, every=16):
    """Heads longer than `keep` (the full-shape M = 2^20 prefixes, whose far tail is FFT noise of
    +-1e-8 down to the last size) keep their first `keep` entries and every `every`-th entry
    beyond (sample_idx / sample_val), so a golden stays ~1 MB; the normwise distance is then
    taken over the kept entries (tests/test_gpu_parity_runs.py)."""
    h = np.asarray(out["head"])
    if h.size <= keep:
        return out
    idx = np.arange(keep, h.size, every, dtype=np.int64)
    out = dict(out)
    out["sample_idx"], out["sample_val"] = idx, h[idx].copy()
    out["head_len"] = np.array(h.size)
    out["head"] = h[:keep].copy()
    return out


def run_one(which, name):
    md, n0, ctl, t_end = case_inputs(name)
    t0 = time.time()
    r = O.Oracle(which).run(md, n0, ctl, t_end, record=O.RECORD_NONE)
    s = summarize(r)
    s["wall_s"] = time.time() - t0
    return s


def fluctuation(name, frac=0.01, nsnap=40):
    """How much the REFERENCE's own trajectory moves about its final state: the reference is
    restarted from its golden final state (the system is autonomous) and run a further `frac` of
    the horizon with every step recorded and `nsnap` snapshots. At a steady state held at the
    controller's stability limit, N(t) and n_s(t) wander step to step by far more than 1e-8 (config 5
    at M = 4096 with RK2: 8e-5 in N), so where a run ends inside that band is decided by roundoff:
    a final value cannot be pinned tighter than this band. Written to CASE__fluct.npz."""
    z = np.load(os.path.join(OUT, f"{name}__ref.npz"))
    cfg, m, st, t_end = CASES[name]
    x0 = np.zeros(m)
    head = np.asarray(z["head"], dtype=np.float64)
    x0[: head.size] = head
    if "sample_idx" in z.files:
        x0[np.asarray(z["sample_idx"])] = np.asarray(z["sample_val"])
    md, _, ctl, _ = case_inputs(name)
    dt = frac * t_end
    snaps = np.linspace(dt / nsnap, dt, nsnap)
    r = O.Oracle("reference").run(md, x0, ctl, dt, snapshot_times=snaps, record=O.RECORD_EVERY_STEP,
                                  records_capacity=4000000)
    k = np.arange(1, m + 1, dtype=np.float64)
    n0, m10, mx = x0.sum(), float(np.dot(k, x0)), float(np.max(np.abs(x0)))
    N = np.array([q["density"] for q in r["records"]])
    M1 = np.array([q["mass"] for q in r["records"]])
    S = np.asarray(r["snapshots"])
    big = x0 > 1e-9 * mx
    out = dict(N=float(np.max(np.abs(N - n0)) / abs(n0)), M1=float(np.max(np.abs(M1 - m10)) / abs(m10)),
               state=float(np.max(np.abs(S - x0)) / mx),
               elem=float(np.max(np.abs(S[:, big] / x0[big] - 1.0))) if big.any() else 0.0,
               window=dt, steps=int(r["total_accepted"]), rejects=int(r["total_rejects"]))
    print(name, "fluct", out, flush=True)
    np.savez_compressed(os.path.join(OUT, f"{name}__fluct.npz"), **{k2: np.asarray(v) for k2, v in out.items()})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case", nargs="?")
    ap.add_argument("--list", action="store_true")
    ap.add_argument("--floor", default="port_fma", help="second CPU build for the noise floor ('' = none)")
    ap.add_argument("--which", default="both", choices=["both", "ref", "floor"])
    ap.add_argument("--fluct", action="store_true",
                    help="write CASE__fluct.npz: the reference trajectory's own fluctuation about its final state")
    ap.add_argument("--leg", default="floor", help="file suffix of the floor leg (floor, floor2: a second floor build)")
    a = ap.parse_args()
    if a.list or not a.case:
        print("\n".join(CASES))
        return
    os.makedirs(OUT, exist_ok=True)
    cfg, m, st, t_end = CASES[a.case]
    if a.fluct:
        fluctuation(a.case)
        return
    legs = []
    if a.which in ("both", "ref"):
        legs.append(("ref", "reference"))
    if a.which in ("both", "floor") and a.floor:
        legs.append((a.leg, a.floor))
    for key, which in legs:
        s = run_one(which, a.case)
        out = dict(config=np.array(cfg), m=np.array(m), stepper=np.array(st), t_end=np.array(t_end),
                   build=np.array(which))
        out.update({k: np.asarray(v) for k, v in s.items()})
        print(a.case, key, which, {k: v for k, v in s.items() if k != "head"}, flush=True)
        np.savez_compressed(os.path.join(OUT, f"{a.case}__{key}.npz"), **out)

if __name__ == "__main__":
    main()
