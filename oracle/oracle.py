"""ctypes front end for the CPU oracle — TEST INFRASTRUCTURE ONLY.

Two interchangeable backends with one API:
  * ``Oracle("port")``      -> oracle/liboracle.so, the C restatement (agk_oracle.c)
  * ``Oracle("reference")`` -> oracle/_ref/libaggkin_ref.so, the reference compiled from its
                               own sources (oracle/Makefile) behind ref_shim.cpp
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this module; the
product path (paper_2407_16559_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "port": (os.path.join(HERE, "liboracle.so"), "ora_"),
    "reference": (os.path.join(HERE, "_ref", "libaggkin_ref.so"), "ref_"),
    # the restatement built with FMA contraction: the CPU-vs-CPU noise floor for trajectories
    "port_fma": (os.path.join(HERE, "liboracle_fma.so"), "ora_"),
    # the restatement with a 2x longer FFT (different roundoff, same algebra)
    "port_pad2": (os.path.join(HERE, "liboracle_pad2.so"), "ora_"),
}

AGGREGATION, SOURCES, SHATTERING = 0, 1, 2
RHS_MODEL, RHS_DECAY, RHS_STILL, RHS_DRAIN, RHS_BURST_INF, RHS_BURST_NAN = range(6)
RK2, RK4, RKF45 = 0, 1, 2
FIXED, ADAPTIVE = 0, 1
STEP_OK, STEP_NONFINITE, STEP_TOO_MANY_REJECTS, STEP_TAU_UNDERFLOW = range(4)
RECORD_EVERY_STEP, RECORD_INTERVAL, RECORD_NONE = 0, 1, 2

_dp = C.POINTER(C.c_double)


class _Model(C.Structure):
    _fields_ = [("m", C.c_size_t), ("r", C.c_size_t), ("u", _dp), ("v", _dp), ("variant", C.c_int),
                ("source_k", C.POINTER(C.c_uint64)), ("source_rate", _dp),
                ("num_sources", C.c_size_t), ("shatter_rate", C.c_double), ("k", _dp)]


class _Control(C.Structure):
    _fields_ = [("stepper", C.c_int), ("mode", C.c_int), ("tau", C.c_double), ("tol", C.c_double),
                ("safety", C.c_double), ("growth_max", C.c_double), ("shrink_min", C.c_double),
                ("tau_min", C.c_double), ("max_rejects", C.c_int), ("relative_error", C.c_int)]


class _Outcome(C.Structure):
    _fields_ = [("tau_used", C.c_double), ("tau_next", C.c_double), ("error_estimate", C.c_double),
                ("rejects", C.c_int), ("rhs_evals", C.c_int), ("status", C.c_int)]


class _Rhs(C.Structure):
    _fields_ = [("kind", C.c_int), ("param", C.c_double), ("model", C.POINTER(_Model)),
                ("evals", C.c_uint64)]


class _RunDesc(C.Structure):
    _fields_ = [("control", _Control), ("t_end", C.c_double), ("initial", _dp),
                ("initial_tau", C.c_double), ("snapshot_times", _dp), ("num_snapshots", C.c_size_t),
                ("record", C.c_int), ("record_interval", C.c_double)]


class _Record(C.Structure):
    _fields_ = [("t", C.c_double), ("tau", C.c_double), ("density", C.c_double),
                ("mass", C.c_double), ("m2", C.c_double), ("error_estimate", C.c_double),
                ("rhs_evals", C.c_uint64), ("rejects", C.c_uint64)]


class _Report(C.Structure):
    _fields_ = [("termination", C.c_int), ("abort_status", C.c_int), ("abort_t", C.c_double),
                ("abort_tau", C.c_double), ("final_t", C.c_double),
                ("total_rhs_evals", C.c_uint64), ("total_accepted", C.c_uint64),
                ("total_rejects", C.c_uint64), ("final_state", _dp), ("snapshots", _dp),
                ("num_snapshots_taken", C.c_size_t), ("records", C.POINTER(_Record)),
                ("records_capacity", C.c_size_t), ("num_records", C.c_size_t)]


def _p(a):
    return a.ctypes.data_as(_dp)


@dataclass
class Model:
    """Model in the reference's layouts (kernels.hpp:26-43, rhs.hpp:32-40): low-rank factors
    u (m, r) and v (r, m), or a DenseKernel `k` (m, m) — then u and v may be None."""
    u: np.ndarray           # (m, r) row-major
    v: np.ndarray           # (r, m) row-major
    variant: int = AGGREGATION
    sources: list = field(default_factory=list)   # [(k, rate)], 1-based k
    shatter_rate: float = 0.0
    k: np.ndarray = None    # dense kernel (m, m) row-major, K(i,j) = k[i-1, j-1]

    def __post_init__(self):
        if self.k is not None:
            self.k = np.ascontiguousarray(self.k, dtype=np.float64)
            m = self.k.shape[0]
            if self.u is None:
                self.u = np.zeros((m, 1))
            if self.v is None:
                self.v = np.zeros((1, m))
        self.u = np.ascontiguousarray(self.u, dtype=np.float64)
        self.v = np.ascontiguousarray(self.v, dtype=np.float64)
        if self.u.ndim == 1:
            self.u = self.u.reshape(-1, 1)
        if self.v.ndim == 1:
            self.v = self.v.reshape(1, -1)
        self._sk = np.array([k for k, _ in self.sources] or [0], dtype=np.uint64)
        self._sr = np.array([r for _, r in self.sources] or [0.0], dtype=np.float64)

    @property
    def m(self):
        return self.u.shape[0]

    @property
    def r(self):
        return self.u.shape[1]

    def c(self):
        return _Model(self.m, self.r, _p(self.u), _p(self.v), self.variant,
                      self._sk.ctypes.data_as(C.POINTER(C.c_uint64)), _p(self._sr),
                      len(self.sources), float(self.shatter_rate),
                      _p(self.k) if self.k is not None else None)


class OracleError(ValueError):
    pass


@dataclass
class Control:
    stepper: int = RKF45
    mode: int = ADAPTIVE
    tau: float = 0.0
    tol: float = 1e-6
    safety: float = 0.0
    growth_max: float = 2.0
    shrink_min: float = 0.5
    tau_min: float = 1e-12
    max_rejects: int = 40
    relative_error: bool = False

    def c(self):
        return _Control(self.stepper, self.mode, self.tau, self.tol, self.safety, self.growth_max,
                        self.shrink_min, self.tau_min, self.max_rejects, int(self.relative_error))


class Oracle:
    def __init__(self, which: str = "port"):
        path, prefix = LIBS[which]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (run `make -C oracle all ref`)")
        self.which = which
        self.lib = C.CDLL(path)
        self.pre = prefix

    def _fn(self, name):
        return getattr(self.lib, self.pre + name)

    # ---- RHS
    def _rhs_call(self, name, model: Model, n, *extra):
        n = np.ascontiguousarray(n, dtype=np.float64)
        out = np.zeros(model.m)
        cm = model.c()
        rc = self._fn(name)(C.byref(cm), _p(n), *extra, _p(out))
        if rc != 0:
            raise OracleError(f"{name} rejected its arguments")
        return out

    def eval_rhs(self, model, n):
        return self._rhs_call("eval_rhs", model, n)

    def birth_term(self, model, n):
        return self._rhs_call("birth_term", model, n)

    def death_term(self, model, n):
        return self._rhs_call("death_term", model, n)

    def shattering_terms(self, model, n, lam):
        return self._rhs_call("shattering_terms", model, n, C.c_double(lam))

    def eval_rhs_dense(self, model, n):
        return self._rhs_call("eval_rhs_dense", model, n)

    def eval_rhs_truth(self, model, n):
        """Long-double evaluation of the same algorithm (port library only)."""
        return self._rhs_call("eval_rhs_truth", model, n)

    def euler_stability_bound(self, model, n, a):
        n = np.ascontiguousarray(n, dtype=np.float64)
        cm = model.c()
        out = C.c_double()
        if self._fn("euler_stability_bound")(C.byref(cm), _p(n), C.c_double(a), C.byref(out)):
            raise OracleError("euler_stability_bound rejected its arguments")
        return out.value

    # ---- steppers
    def _rhs_struct(self, model, kind, param):
        cm = model.c() if model is not None else None
        f = _Rhs(kind, param, C.pointer(cm) if cm is not None else None, 0)
        return f, cm

    def rk_step(self, stepper, n, tau, model=None, kind=RHS_MODEL, param=0.0):
        n = np.ascontiguousarray(n, dtype=np.float64)
        m = n.size
        out, out5, err = np.zeros(m), np.zeros(m), C.c_double(np.nan)
        f, _keep = self._rhs_struct(model, kind, param)
        self._fn("rk_step").argtypes = None
        rc = self._fn("rk_step")(C.byref(f), stepper, C.c_size_t(m), _p(n), C.c_double(tau), _p(out),
                                 _p(out5), C.byref(err))
        if rc:
            raise OracleError("rk_step rejected its arguments")
        return out, out5, err.value, f.evals

    def advance(self, n, tau, control: Control, model=None, kind=RHS_MODEL, param=0.0):
        n = np.ascontiguousarray(n, dtype=np.float64)
        m = n.size
        state = np.zeros(m)
        o = _Outcome()
        f, _keep = self._rhs_struct(model, kind, param)
        cc = control.c()
        rc = self._fn("advance")(C.byref(f), C.c_size_t(m), _p(n), C.c_double(tau), C.byref(cc),
                                 C.byref(o), _p(state))
        if rc:
            raise OracleError("advance rejected its arguments")
        return dict(state=state, tau_used=o.tau_used, tau_next=o.tau_next,
                    error_estimate=o.error_estimate, rejects=o.rejects, rhs_evals=o.rhs_evals,
                    status=o.status, evals_counted=f.evals)

    def run(self, model, initial, control: Control, t_end, initial_tau=0.0, snapshot_times=(),
            record=RECORD_NONE, record_interval=0.0, records_capacity=0):
        initial = np.ascontiguousarray(initial, dtype=np.float64)
        m = initial.size
        snaps_t = np.ascontiguousarray(snapshot_times, dtype=np.float64).reshape(-1)
        snaps_t_buf = snaps_t if snaps_t.size else np.zeros(1)
        final = np.zeros(m)
        snaps = np.zeros((max(snaps_t.size, 1), m))
        recs = (_Record * max(records_capacity, 1))()
        d = _RunDesc(control.c(), float(t_end), _p(initial), float(initial_tau), _p(snaps_t_buf),
                     snaps_t.size, record, float(record_interval))
        rep = _Report()
        rep.final_state = _p(final)
        rep.snapshots = _p(snaps)
        rep.records = recs
        rep.records_capacity = records_capacity
        f, _keep = self._rhs_struct(model, RHS_MODEL, 0.0)
        rc = self._fn("run")(C.byref(f), C.c_size_t(m), C.byref(d), C.byref(rep))
        if rc:
            raise OracleError("run rejected its arguments")
        nrec = min(rep.num_records, records_capacity)
        records = [dict(t=r.t, tau=r.tau, density=r.density, mass=r.mass, m2=r.m2,
                        error_estimate=r.error_estimate, rhs_evals=r.rhs_evals, rejects=r.rejects)
                   for r in recs[:nrec]]
        return dict(termination=rep.termination, abort_status=rep.abort_status,
                    abort_t=rep.abort_t, abort_tau=rep.abort_tau, final_t=rep.final_t,
                    total_rhs_evals=rep.total_rhs_evals, total_accepted=rep.total_accepted,
                    total_rejects=rep.total_rejects, final_state=final,
                    snapshots=snaps[:rep.num_snapshots_taken].copy(), records=records,
                    num_records=rep.num_records)


# ---- kernel factor builders (kernels.cpp:59-101 and BASELINE.json configs)

def constant_factors(m):
    """K = 1 (kernels.cpp:64-69)."""
    return np.ones((m, 1)), np.ones((1, m))


def brownian_factors(m, alpha):
    """(i/j)^a + (j/i)^a with bitwise-reciprocal columns (kernels.cpp:74-85)."""
    i = np.arange(1, m + 1, dtype=np.float64)
    p = np.power(i, alpha)
    u = np.stack([p, 1.0 / p], axis=1)
    v = np.stack([1.0 / p, p], axis=0)
    return u, v


def free_molecular_dense(m):
    """DenseKernel of the free-molecular kernel (kernels.cpp:49-51, build_dense 103-): K(x,y) =
    (cbrt x + cbrt y)^2 sqrt(1/x + 1/y), x, y = 1..m."""
    x = np.arange(1, m + 1, dtype=np.float64)
    c = np.cbrt(x)
    s = c[:, None] + c[None, :]
    return s * s * np.sqrt(1.0 / x[:, None] + 1.0 / x[None, :])


def brownian_plus2_factors(m):
    """Config 2/5 kernel (i/j)^(1/3) + (j/i)^(1/3) + 2, R=3 (SURVEY §8c note 4)."""
    i = np.arange(1, m + 1, dtype=np.float64)
    p = np.power(i, 1.0 / 3.0)
    s2 = np.sqrt(2.0)
    u = np.stack([p, 1.0 / p, np.full(m, s2)], axis=1)
    v = np.stack([1.0 / p, p, np.full(m, s2)], axis=0)
    return u, v
