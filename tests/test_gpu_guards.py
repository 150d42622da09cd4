"""Guard-band bounds checks of every device RHS path and the device stepper, through the C ABI
with DEVICE pointers (agk_rhs_eval / agk_rhs_eval_timed / agk_advance, include/agk/agk.h).

n and out are views into larger device buffers whose guard bands hold a sentinel: after the
call the guards must be bit-for-bit unchanged (no store outside [out, out + m)), and a NaN
guard around n must not leak into the result (no load outside [n, n + m) feeds the RHS). The
result must equal the host-pointer path bit for bit (same kernels, same order). Paths: the
single-kernel small path, the four-step mid-size path, the M = 2^20 warp path (transpose and
dvec launches) for all three variants, the dense-kernel path. (compute-sanitizer is not
available on the GPU pool; these guards are the repo's own out-of-bounds check.)
"""
import ctypes as C

import numpy as np
import pytest

from tests.helpers import config4_inputs, factors

pytestmark = pytest.mark.gpu

G = 4096  # guard elements on each side (32 KiB)
SENTINEL = -1.2345678901234567e300


def _guarded(torch, m, fill):
    buf = torch.full((m + 2 * G,), fill, dtype=torch.float64, device="cuda:0")
    return buf, buf[G:G + m]


def _check_guards(torch, buf, m, fill):
    lo, hi = buf[:G], buf[G + m:]
    if np.isnan(fill):
        assert bool(torch.isnan(lo).all()) and bool(torch.isnan(hi).all())
    else:
        assert bool((lo == fill).all()) and bool((hi == fill).all())


def _cases(agk):
    u, v = factors("constant", 2048)
    yield "small c1-shape", agk.Model(u, v), np.random.default_rng(1).random(2048)
    u, v = factors("brownian2", 1 << 16)
    yield "four-step c2-shape", agk.Model(u, v, agk.AGGREGATION_SOURCES, [(1, 1.0), (7, 0.25)]), \
        np.random.default_rng(2).random(1 << 16)
    u, v = factors("brownian", 1 << 17, 0.9)
    yield "four-step c3-shape", agk.Model(u, v, agk.AGGREGATION_SHATTERING, [], 0.01), \
        np.random.default_rng(3).random(1 << 17)
    U, V, n = config4_inputs()
    yield "warp c4 aggregation", agk.Model(U, V), n
    yield "warp c4 sources", agk.Model(U, V, agk.AGGREGATION_SOURCES, [(1, 1.0), (1 << 20, 0.5)]), n
    yield "warp c4 shattering", agk.Model(U, V, agk.AGGREGATION_SHATTERING, [], 0.01), n
    i = np.arange(1, 1025, dtype=np.float64)
    yield "dense", agk.Model(None, None, k=(np.cbrt(i)[:, None] + np.cbrt(i)[None, :]) ** 2), np.exp(-i / 100.0)


def test_rhs_guard_bands(agk):
    import torch
    lib = agk.load_library()
    for name, model, n in _cases(agk):
        m = n.size
        ws = agk.RhsWorkspace(model, device=0)
        want = agk.eval_rhs(ws, n)
        nbuf, nd = _guarded(torch, m, float("nan"))
        nd.copy_(torch.from_numpy(n))
        obuf, od = _guarded(torch, m, SENTINEL)
        rc = lib.agk_rhs_eval(ws.handle, nd.data_ptr(), od.data_ptr(), agk.MEM_DEVICE)
        assert rc == 0, (name, agk.describe(rc))
        torch.cuda.synchronize()
        _check_guards(torch, obuf, m, SENTINEL)
        _check_guards(torch, nbuf, m, float("nan"))
        got = od.cpu().numpy()
        assert np.array_equal(got, want), name
        # back-to-back evaluations through the captured per-RHS graph
        od.fill_(0.0)
        ms = C.c_float()
        rc = lib.agk_rhs_eval_timed(ws.handle, nd.data_ptr(), od.data_ptr(), 3, C.byref(ms))
        assert rc == 0, (name, agk.describe(rc))
        torch.cuda.synchronize()
        _check_guards(torch, obuf, m, SENTINEL)
        assert np.array_equal(od.cpu().numpy(), want), name


@pytest.mark.parametrize("stepper", ["RK2", "RK4", "RKF45"])
@pytest.mark.parametrize("m", [2048, 1 << 16])
def test_advance_guard_bands(agk, stepper, m):
    import torch
    u, v = factors("brownian2", m)
    ws = agk.RhsWorkspace(agk.Model(u, v, agk.AGGREGATION_SOURCES, [(1, 1.0)]), device=0)
    n0 = np.random.default_rng(m).random(m) * 1e-3
    ctl = agk.StepControl(stepper=getattr(agk, stepper), tol=1e-6)
    want = agk.advance(ws, n0, 0.01, ctl)
    nbuf, nd = _guarded(torch, m, float("nan"))
    nd.copy_(torch.from_numpy(n0))
    sbuf, sd = _guarded(torch, m, SENTINEL)
    o = agk._Outcome()
    cc = ctl.c()
    rc = agk.load_library().agk_advance(ws.handle, nd.data_ptr(), C.c_double(0.01), C.byref(cc), C.byref(o),
                                        sd.data_ptr(), agk.MEM_DEVICE)
    assert rc == 0, agk.describe(rc)
    torch.cuda.synchronize()
    _check_guards(torch, nbuf, m, float("nan"))
    _check_guards(torch, sbuf, m, SENTINEL)
    assert o.status == want.status == 0
    assert o.rejects == want.rejects and o.rhs_evals == want.rhs_evals
    assert np.array_equal(sd.cpu().numpy(), want.state)
