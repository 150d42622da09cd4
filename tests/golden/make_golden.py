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


# Config texts for the front end's parser (aggkin.parse_config_text vs config.cpp:131-438): valid
# ones exercising every key, and one case per error path (messages compared verbatim).
BASE = "model = aggregation\nkernel = constant\nm = 64\nstepper = rk4\nmode = adaptive\ntol = 1e-8\nt_end = 2\n"
CONFIG_TEXTS = [
    BASE,
    BASE + "snapshots = 2, 0.5, 1, 0.5\nrecord = interval\nrecord_interval = 0.25\n",
    "# comment line\nmodel = shattering   # trailing comment\nkernel = brownian\nalpha = 0.95\nm = 8192\n"
    "lambda = 0.01\ninitial = monodisperse\nstepper = rk2\nmode = adaptive\ntol = 1e-6\nt_end = 250\n"
    "record = every_step\noutput = out/x\n",
    "model = sources\nkernel = constant\nm = 4096\nsources = 100:0.1, 1:1\nstepper = rkf45\nmode = fixed\n"
    "tau = 0.01\nt_end = 1000\nbench_schemes = rk2, rk4, rkf45\nbench_cells = fixed:0.01, adaptive:1e-4, "
    "adaptive:1e-6\nrecord = none\nseed = 42\n",
    "model = aggregation\nkernel = free_molecular\nm = 128\ninitial = exponential\ninitial_scale = 5\n"
    "stepper = rkf45\nmode = adaptive\ntol = 1e-7\ntau0 = 0.001\nsafety = 0.8\ngrowth_max = 3\n"
    "shrink_min = 0.2\ntau_min = 1e-14\nmax_rejects = 7\nerror_norm = relative\nt_end = 0x1p3\n",
    "model = aggregation\nkernel = factors\nfactors_path = /tmp/f.txt\nm = 16\nstepper = rk2\nmode = fixed\n"
    "tau = .5\nt_end = 1.\n",
    "  model=aggregation\r\nkernel=constant\r\nm=8\r\nstepper=rk2\r\nmode=fixed\r\ntau=1E-2\r\nt_end=+3\r\n",
    BASE.replace("tol = 1e-8", "tol = inf"),
    # errors
    BASE + "bogus = 1\n",
    BASE + "m = 3\n",
    BASE + "no equals sign\n",
    BASE + " = 4\n",
    BASE + "alpha =\n",
    BASE.replace("model = aggregation", "model = growth"),
    BASE.replace("kernel = constant", "kernel = linear"),
    BASE.replace("stepper = rk4", "stepper = euler"),
    BASE.replace("mode = adaptive", "mode = both"),
    BASE.replace("m = 64", "m = -4"),
    BASE.replace("m = 64", "m = 1"),
    BASE.replace("m = 64", "m = 12abc"),
    BASE.replace("tol = 1e-8", "tol = 1e-8x"),
    BASE.replace("tol = 1e-8", "tol = 1e999"),
    BASE.replace("tol = 1e-8", "tol = 0"),
    BASE.replace("kernel = constant", "kernel = brownian"),
    BASE.replace("kernel = constant", "kernel = brownian\nalpha = -1"),
    BASE.replace("kernel = constant", "kernel = factors"),
    BASE.replace("model = aggregation", "model = sources"),
    BASE.replace("model = aggregation", "model = sources\nsources = 1-2"),
    BASE.replace("model = aggregation", "model = sources\nsources = 65:1"),
    BASE.replace("model = aggregation", "model = sources\nsources = 1:-1"),
    BASE.replace("model = aggregation", "model = shattering"),
    BASE.replace("model = aggregation", "model = shattering\nlambda = -0.5"),
    BASE + "tau0 = -1\n",
    BASE + "safety = 1\n",
    BASE + "growth_max = 0.9\n",
    BASE + "tau_min = 0\n",
    BASE + "max_rejects = 0\n",
    BASE.replace("mode = adaptive\ntol = 1e-8", "mode = fixed"),
    BASE.replace("mode = adaptive\ntol = 1e-8", "mode = fixed\ntau = -0.1"),
    BASE + "initial = exponential\n",
    BASE + "initial = gaussian\n",
    BASE + "record = interval\n",
    BASE + "record = sometimes\n",
    BASE + "error_norm = weighted\n",
    BASE.replace("t_end = 2", "t_end = nan"),
    BASE + "snapshots = 0.5, 3\n",
    BASE + "bench_cells = fixed 0.1\n",
    BASE + "bench_cells = sometimes:0.1\n",
    BASE + "bench_cells = adaptive:0\n",
    BASE + "bench_schemes = rk3\n",
    "model = aggregation\n",
    "",
]


def frontend_cases():
    """The reference's own parser, kernel_entry and fits (oracle/ref_shim.cpp) on fixed inputs, and
    run_text counts of small configs (the reference's run over to_simulation_config)."""
    import ctypes as C
    lib = C.CDLL(os.path.join(os.path.dirname(os.path.dirname(HERE)), "oracle", "_ref", "libaggkin_ref.so"))
    buf = C.create_string_buffer(1 << 16)
    cfgs = []
    for text in CONFIG_TEXTS:
        rc = lib.ref_parse_config(text.encode(), buf, len(buf))
        cfgs.append(dict(text=text, rc=rc, out=buf.value.decode()))
    ents = []
    lib.ref_kernel_entry.argtypes = [C.c_int, C.c_double, C.c_size_t, C.c_size_t, C.POINTER(C.c_double)]
    for var, alpha in ((0, 0.0), (1, 1.0 / 3.0), (1, 0.95), (2, 0.0)):
        for i, j in ((1, 1), (1, 2), (2, 1), (3, 7), (100, 1), (4096, 17), (1 << 20, 3)):
            v = C.c_double()
            lib.ref_kernel_entry(var, alpha, i, j, C.byref(v))
            ents.append(dict(variant=var, alpha=alpha, i=i, j=j, value=v.value))
    fits = []
    lib.ref_fit.argtypes = [C.POINTER(C.c_double), C.c_size_t, C.c_double, C.c_int, C.c_size_t, C.c_size_t,
                            C.POINTER(C.c_double)]
    k = np.arange(1, 2049, dtype=np.float64)
    rng = np.random.Generator(np.random.MT19937(7))
    series = [k ** -1.5, k ** -1.5 * np.exp(-1e-4 * k), k ** -2.2 * rng.uniform(0.9, 1.1, k.size)]
    series[2][100:140] = 0.0
    for si, n in enumerate(series):
        for lam, cut, lo, hi in ((0.0, 0, 10, 2000), (0.01, 1, 10, 2000), (0.0, 0, 1, 2048), (0.02, 1, 50, 500)):
            res = (C.c_double * 6)()
            a = np.ascontiguousarray(n)
            rc = lib.ref_fit(a.ctypes.data_as(C.POINTER(C.c_double)), a.size, lam, cut, lo, hi, res)
            fits.append(dict(series=si, lam=lam, cutoff=cut, k_lo=lo, k_hi=hi, rc=rc, res=list(res)))
    with open(os.path.join(HERE, "config_cases.json"), "w") as f:
        json.dump(dict(configs=cfgs, kernel_entries=ents, fits=fits), f, indent=1)
    return len(cfgs), len(ents), len(fits)


if __name__ == "__main__" and "--frontend-only" in sys.argv:
    print("frontend cases:", frontend_cases())
    sys.exit(0)

if __name__ == "__main__" and "--dense-only" in sys.argv:
    print("dense cases:", dense_cases())
    sys.exit(0)

if __name__ == "__main__":
    print("rhs cases", rhs_cases())
    print("dense cases", dense_cases())
    print("run cases", run_cases())
    print("frontend cases", frontend_cases())
