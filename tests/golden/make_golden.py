"""Generate the golden fixtures from the REFERENCE itself (oracle/_ref, compiled from the
reference's own sources by oracle/Makefile). Run here, where /root/reference exists:

    make -C oracle all ref && python tests/golden/make_golden.py

Writes tests/golden/golden_rhs.npz and tests/golden/golden_runs.json. The fixtures travel with
the repo; the GPU box never needs /root/reference.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402

KERNELS = [("constant", 0.0), ("brownian", 1.0 / 3.0), ("brownian", 0.95), ("brownian2", 0.0)]
VARIANTS = [O.AGGREGATION, O.SOURCES, O.SHATTERING]


def factors(kind, m, alpha):
    if kind == "constant":
        return O.constant_factors(m)
    if kind == "brownian":
        return O.brownian_factors(m, alpha)
    return O.brownian_plus2_factors(m)


def rhs_cases():
    ref = O.Oracle("reference")
    rng = np.random.Generator(np.random.MT19937(0x5EED5EED))
    out = {}
    idx = 0
    for m in (2, 3, 17, 64, 96, 256, 1000, 4096):
        for kind, alpha in KERNELS:
            for var in VARIANTS:
                u, v = factors(kind, m, alpha)
                srcs = [(1, 1.0), (min(m, 10), 0.1)] if var == O.SOURCES else []
                md = O.Model(u, v, var, srcs, 0.01 if var == O.SHATTERING else 0.0)
                n = rng.random(m)
                s = ref.eval_rhs(md, n)
                out[f"c{idx}_meta"] = np.array([m, var, KERNELS.index((kind, alpha))], dtype=np.float64)
                out[f"c{idx}_n"] = n
                out[f"c{idx}_S"] = s
                idx += 1
    out["count"] = np.array([idx])
    np.savez_compressed(os.path.join(HERE, "golden_rhs.npz"), **out)
    return idx


def dense_cases():
    """DenseKernel (free-molecular, kernels.cpp:49-51) RHS goldens: the reference's dense branches
    (rhs.cpp:37-45, 153-159, 197-205) on seeded states."""
    ref = O.Oracle("reference")
    rng = np.random.Generator(np.random.MT19937(0x5EED5EED + 1))
    out = {}
    idx = 0
    for m in (2, 3, 17, 64, 257, 1000):
        k = O.free_molecular_dense(m)
        for var in VARIANTS:
            srcs = [(1, 1.0), (min(m, 10), 0.1)] if var == O.SOURCES else []
            md = O.Model(None, None, var, srcs, 0.01 if var == O.SHATTERING else 0.0, k=k)
            n = rng.random(m)
            out[f"c{idx}_meta"] = np.array([m, var], dtype=np.float64)
            out[f"c{idx}_n"] = n
            out[f"c{idx}_S"] = ref.eval_rhs(md, n)
            out[f"c{idx}_bound"] = np.array([ref.euler_stability_bound(md, n, 0.25)])
            idx += 1
    out["count"] = np.array([idx])
    np.savez_compressed(os.path.join(HERE, "golden_dense.npz"), **out)
    return idx


RUNS = [
    # (name, kernel, alpha, m, variant, sources, lambda, stepper, mode, tol/tau, t_end, snapshots)
    ("agg_const_rk4_m256", "constant", 0.0, 256, O.AGGREGATION, [], 0.0, O.RK4, O.ADAPTIVE, 1e-8, 10.0, [1.0, 10.0]),
    ("agg_const_rkf45_m256", "constant", 0.0, 256, O.AGGREGATION, [], 0.0, O.RKF45, O.ADAPTIVE, 1e-8, 10.0, [1.0]),
    ("agg_const_rk2_m128", "constant", 0.0, 128, O.AGGREGATION, [], 0.0, O.RK2, O.ADAPTIVE, 1e-6, 5.0, []),
    ("src_brown_rkf45_m512", "brownian2", 0.0, 512, O.SOURCES, [(1, 1.0)], 0.0, O.RKF45, O.ADAPTIVE, 1e-6, 20.0, [5.0]),
    ("shat_brown_rk4_m256", "brownian", 0.95, 256, O.SHATTERING, [], 0.01, O.RK4, O.ADAPTIVE, 1e-6, 20.0, []),
    ("fixed_rk2_m64", "constant", 0.0, 64, O.AGGREGATION, [], 0.0, O.RK2, O.FIXED, 0.01, 1.0, []),
    ("fixed_rkf45_m64", "brownian", 1.0 / 3.0, 64, O.SOURCES, [(1, 1.0), (10, 0.1)], 0.0, O.RKF45, O.FIXED, 0.05, 2.0, []),
]


def run_cases():
    ref = O.Oracle("reference")
    res = {}
    for name, kind, alpha, m, var, srcs, lam, stepper, mode, val, t_end, snaps in RUNS:
        u, v = factors(kind, m, alpha)
        md = O.Model(u, v, var, srcs, lam)
        n0 = np.zeros(m)
        if var != O.SOURCES:
            n0[0] = 1.0
        ctl = O.Control(stepper=stepper, mode=mode, tau=val if mode == O.FIXED else 0.0,
                        tol=val if mode == O.ADAPTIVE else 1e-6)
        r = ref.run(md, n0, ctl, t_end, snapshot_times=snaps, record=O.RECORD_EVERY_STEP,
                    records_capacity=200000)
        res[name] = dict(kind=kind, alpha=alpha, m=m, variant=var, sources=srcs, lam=lam, stepper=stepper, mode=mode,
                         value=val, t_end=t_end, snapshots=snaps, termination=r["termination"],
                         total_rhs_evals=r["total_rhs_evals"], total_accepted=r["total_accepted"],
                         total_rejects=r["total_rejects"], final_t=r["final_t"],
                         final_state=[float(x) for x in r["final_state"]],
                         num_records=r["num_records"],
                         last_record=r["records"][-1] if r["records"] else None)
    with open(os.path.join(HERE, "golden_runs.json"), "w") as f:
        json.dump(res, f, indent=1)
    return len(res)


if __name__ == "__main__" and "--dense-only" in sys.argv:
    print("dense cases:", dense_cases())
    sys.exit(0)

if __name__ == "__main__":
    print("rhs cases", rhs_cases())
    print("dense cases", dense_cases())
    print("run cases", run_cases())
