"""Drive every device code path once (a coverage driver for memory / race checkers).

Usage (on the GPU box):  python tools/sanitize.py [--quick]
(meant to run under compute-sanitizer memcheck / racecheck / synccheck; the tool is closed on
this GPU pool, so the repo's own out-of-bounds check is tests/test_gpu_guards.py, and this
driver's plain run is recorded in profiles/path_coverage_r01k.log)

Paths driven (rhs.cu rhs_make_plan): the single-kernel small path (P <= 4096), the four-step
mid-size path (configs 2 and 3 shapes), the M = 2^20 warp path with the transpose / dvec launches
(config 4, all three variants), the dense-kernel path, the device steppers (RK2 / RK4 doubling,
RKF45 embedded, fixed steps) and the device run loop (WHILE graph, snapshots, records).
`--quick` drops the M = 2^20 cases (racecheck instruments every shared-memory access).
This is a memory / race checker driver, not a parity test: parity lives in tests/ (against the
oracle); here each result is only checked for finiteness and run-to-run determinism.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_16559_b200 as agk  # noqa: E402
from paper_2407_16559_b200 import configs  # noqa: E402


def check(name, x):
    x = np.asarray(x)
    assert np.all(np.isfinite(x)), name
    print(f"  {name}: ok (max |x| {np.max(np.abs(x)):.3e})", flush=True)


def rhs_case(name, model, n):
    ws = agk.RhsWorkspace(model, device=0)
    a = agk.eval_rhs(ws, n)
    b = agk.eval_rhs(ws, n)
    assert np.array_equal(a, b), f"{name}: not deterministic"
    check(f"{name} eval_rhs", a)
    return ws


def step_cases(name, ws, n0, tau, tol):
    for st in (agk.RK2, agk.RK4, agk.RKF45):
        o = agk.advance(ws, n0, tau, agk.StepControl(stepper=st, tol=tol))
        check(f"{name} advance stepper={st} status={o.status} rejects={o.rejects}", o.state)
    check(f"{name} rk4_step", agk.rk4_step(ws, n0, tau))


def run_case(name, ws, n0, t_end, tol, stepper=agk.RKF45):
    cfg = agk.SimulationConfig(agk.StepControl(stepper=stepper, tol=tol), t_end, n0,
                               snapshot_times=[t_end / 2], record=1, record_interval=t_end / 4)
    rep = agk.run(ws, cfg)
    assert rep.termination == "completed", rep.abort_reason
    check(f"{name} run stepper={stepper} accepted={rep.total_accepted} records={rep.num_records}", rep.final_state)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()

    print("small path: config 1 shape (M = 2048, constant kernel)", flush=True)
    u, v = configs.constant_factors(2048)
    n0 = configs.monodisperse(2048)
    ws = rhs_case("c1", agk.Model(u, v), n0)
    step_cases("c1", ws, n0, 0.05, 1e-6)
    run_case("c1", ws, n0, 2.0, 1e-6)

    print("four-step path: config 2 shape (M = 2^16, Brownian+2, sources)", flush=True)
    u, v = configs.brownian_plus2_factors(1 << 16)
    n0 = np.zeros(1 << 16)
    ws = rhs_case("c2", agk.Model(u, v, agk.AGGREGATION_SOURCES, [(1, 1.0)]), n0 + 1e-3)
    step_cases("c2", ws, n0, 0.01, 1e-6)
    run_case("c2", ws, n0, 0.5, 1e-6, agk.RK2)

    print("four-step path: config 3 shape (M = 2^17, alpha 0.9, shattering)", flush=True)
    u, v = configs.brownian_factors(1 << 17, 0.9)
    n0 = configs.monodisperse(1 << 17)
    ws = rhs_case("c3", agk.Model(u, v, agk.AGGREGATION_SHATTERING, [], 0.01), n0)
    run_case("c3", ws, n0, 0.05, 1e-8)

    print("dense path (M = 1024)", flush=True)
    i = np.arange(1, 1025, dtype=np.float64)
    k = (np.cbrt(i)[:, None] + np.cbrt(i)[None, :]) ** 2
    rhs_case("dense", agk.Model(None, None, k=k), np.exp(-i / 100.0))

    if not args.quick:
        print("warp path: config 4 shape (M = 2^20, R = 16)", flush=True)
        U, V, n = configs.random_config4()
        for var, src, lam in ((agk.AGGREGATION, [], 0.0), (agk.AGGREGATION_SOURCES, [(1, 1.0), (3, 0.5)], 0.0),
                              (agk.AGGREGATION_SHATTERING, [], 0.01)):
            rhs_case(f"c4 variant={var}", agk.Model(U, V, var, src, lam), n)
        print("warp path: config 5 shape (M = 2^20, Brownian+2, sources), short run", flush=True)
        u, v = configs.brownian_plus2_factors(1 << 20)
        n0 = np.zeros(1 << 20)
        ws = agk.RhsWorkspace(agk.Model(u, v, agk.AGGREGATION_SOURCES, [(1, 1.0)]), device=0)
        run_case("c5", ws, n0, 0.05, 1e-6)
    print("SANITIZE DRIVER DONE", flush=True)


if __name__ == "__main__":
    main()
