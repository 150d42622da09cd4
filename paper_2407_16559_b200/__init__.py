"""B200-native low-rank Smoluchowski RHS + adaptive Runge–Kutta hot path (arXiv 2407.16559).

Host-side mirror of the reference ``aggkin`` operator API for this path, over the C ABI in
``include/agk/agk.h`` (``libagk_b200.so``, built in-tree for sm_100a):

    reference (C++, /root/reference/proj)          this package
    --------------------------------------         ----------------------------------------
    ModelSpec + LowRankFactors (rhs.hpp:32-40)      Model
    RhsWorkspace (rhs.hpp:45-70)                    RhsWorkspace  (owns the device handle)
    eval_rhs / birth_term / death_term /            eval_rhs / birth_term / death_term /
      shattering_terms (rhs.hpp:75-90)                shattering_terms
    euler_stability_bound (rhs.hpp:99)              euler_stability_bound
    StepControl / StepOutcome (steppers.hpp)        StepControl / StepOutcome
    rk2_step / rk4_step / rkf45_step / fixed_step   rk2_step / rk4_step / rkf45_step / fixed_step
    advance (steppers.hpp:109)                      advance
    SimulationConfig / RunReport / run              SimulationConfig / RunReport / run
    RhsFn fakes of the stepper tests                fake_rhs(kind, m, param)

Argument errors raise ``ValueError`` where the reference throws ``std::invalid_argument``.
There is no CPU fallback: without the built library or without a B200 every call raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AGK_LIB") or os.path.join(_HERE, "libagk_b200.so")  # AGK_LIB: A/B experiments

# enums mirrored from include/agk/agk.h
AGGREGATION, AGGREGATION_SOURCES, AGGREGATION_SHATTERING = 0, 1, 2
RHS_MODEL, RHS_DECAY, RHS_STILL, RHS_DRAIN, RHS_BURST_INF, RHS_BURST_NAN = range(6)
RK2, RK4, RKF45 = 0, 1, 2
FIXED, ADAPTIVE = 0, 1
STEP_OK, STEP_NONFINITE, STEP_TOO_MANY_REJECTS, STEP_TAU_UNDERFLOW = range(4)
RECORD_EVERY_STEP, RECORD_INTERVAL, RECORD_NONE = 0, 1, 2
MEM_HOST, MEM_DEVICE = 0, 1
AGK_OK, AGK_ERR_INVALID_ARGUMENT, AGK_ERR_NO_DEVICE, AGK_ERR_CUDA, AGK_ERR_OUT_OF_MEMORY = range(5)

_dp = C.POINTER(C.c_double)


class _ModelDesc(C.Structure):
    _fields_ = [("m", C.c_size_t), ("r", C.c_size_t), ("u", _dp), ("v", _dp), ("variant", C.c_int),
                ("source_k", C.POINTER(C.c_uint64)), ("source_rate", _dp), ("num_sources", C.c_size_t),
                ("shatter_rate", C.c_double), ("device", C.c_int), ("k", _dp)]


class _Control(C.Structure):
    _fields_ = [("stepper", C.c_int), ("mode", C.c_int), ("tau", C.c_double), ("tol", C.c_double),
                ("safety", C.c_double), ("growth_max", C.c_double), ("shrink_min", C.c_double),
                ("tau_min", C.c_double), ("max_rejects", C.c_int), ("relative_error", C.c_int)]


class _Outcome(C.Structure):
    _fields_ = [("tau_used", C.c_double), ("tau_next", C.c_double), ("error_estimate", C.c_double),
                ("rejects", C.c_int), ("rhs_evals", C.c_int), ("status", C.c_int)]


class _RunDesc(C.Structure):
    _fields_ = [("control", _Control), ("t_end", C.c_double), ("initial", _dp), ("initial_tau", C.c_double),
                ("snapshot_times", _dp), ("num_snapshots", C.c_size_t), ("record", C.c_int),
                ("record_interval", C.c_double)]


class _Record(C.Structure):
    _fields_ = [("t", C.c_double), ("tau", C.c_double), ("density", C.c_double), ("mass", C.c_double),
                ("m2", C.c_double), ("error_estimate", C.c_double), ("rhs_evals", C.c_uint64),
                ("rejects", C.c_uint64)]


_RecordSink = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(_Record), C.c_size_t)
RECORD_DTYPE = np.dtype([("t", "<f8"), ("tau", "<f8"), ("density", "<f8"), ("mass", "<f8"), ("m2", "<f8"),
                         ("error_estimate", "<f8"), ("rhs_evals", "<u8"), ("rejects", "<u8")])


class _Report(C.Structure):
    _fields_ = [("termination", C.c_int), ("abort_status", C.c_int), ("abort_t", C.c_double),
                ("abort_tau", C.c_double), ("final_t", C.c_double), ("total_rhs_evals", C.c_uint64),
                ("total_accepted", C.c_uint64), ("total_rejects", C.c_uint64), ("wall_seconds", C.c_double),
                ("final_state", _dp), ("snapshots", _dp), ("num_snapshots_taken", C.c_size_t),
                ("records", C.POINTER(_Record)), ("records_capacity", C.c_size_t), ("num_records", C.c_size_t),
                ("record_sink", _RecordSink), ("sink_user", C.c_void_p)]


# exported symbols and their signatures (must match include/agk/agk.h)
_SIGS = {
    "agk_rhs_create": (C.c_int, [C.POINTER(_ModelDesc), C.POINTER(C.c_void_p)]),
    "agk_rhs_create_fake": (C.c_int, [C.c_int, C.c_size_t, C.c_double, C.c_int, C.POINTER(C.c_void_p)]),
    "agk_rhs_destroy": (None, [C.c_void_p]),
    "agk_rhs_size": (C.c_size_t, [C.c_void_p]),
    "agk_rhs_unique_ranks": (C.c_size_t, [C.c_void_p]),
    "agk_rhs_eval": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    "agk_rhs_eval_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "agk_birth_term": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    "agk_death_term": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    "agk_shattering_terms": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_int]),
    "agk_euler_stability_bound": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double, _dp, C.c_int]),
    "agk_rhs_evals": (C.c_uint64, [C.c_void_p]),
    "agk_rhs_reset_evals": (None, [C.c_void_p]),
    "agk_control_defaults": (None, [C.POINTER(_Control)]),
    "agk_control_validate": (C.c_int, [C.POINTER(_Control)]),
    "agk_rk_step": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, _dp, C.c_int]),
    "agk_advance": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double, C.POINTER(_Control), C.POINTER(_Outcome),
                              C.c_void_p, C.c_int]),
    "agk_run": (C.c_int, [C.c_void_p, C.POINTER(_RunDesc), C.POINTER(_Report)]),
    "agk_last_error": (C.c_char_p, [C.c_void_p]),
    "agk_describe_status": (C.c_char_p, [C.c_int]),
    "agk_rhs_eval_timed": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_float)]),
    "agk_rhs_launches_per_eval": (C.c_int, [C.c_void_p]),
    "agk_rhs_profile": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, _dp, C.POINTER(C.c_int), C.c_int,
                                  C.POINTER(C.c_int), C.POINTER(C.c_int)]),
}

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libagk_b200.so (raises if it has not been built: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `make -C paper_2407_16559_b200` "
                          "(or __graft_entry__.build()); the B200 path has no CPU fallback")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols():
    return sorted(_SIGS)


def _check(rc, handle=None):
    if rc == AGK_OK:
        return
    msg = load_library().agk_last_error(handle).decode(errors="replace")
    if rc == AGK_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    raise RuntimeError(f"agk error {rc}: {msg}")


def describe(status: int) -> str:
    """describe(StepStatus) (simulator.cpp:98-110)."""
    return load_library().agk_describe_status(status).decode()


# ---------------------------------------------------------------------------- arrays

class _Arr:
    """Host numpy or CUDA torch array as (pointer, where, keepalive).

    CUDA tensors: torch's current stream is synchronized first, so a tensor whose producing kernel
    (or, for outputs, whose previous user) is still queued is complete before the handle's stream
    touches it (the handle's stream is only ordered after the legacy default stream, agk.h)."""

    def __init__(self, x, m, writable=False):
        if hasattr(x, "is_cuda") and x.is_cuda:
            import torch
            if x.dtype != torch.float64 or not x.is_contiguous() or x.numel() != m:
                raise ValueError("device arrays must be contiguous float64 of size m")
            torch.cuda.current_stream(x.device).synchronize()
            self.ptr, self.where, self.obj = x.data_ptr(), MEM_DEVICE, x
        else:
            a = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1))
            if a.size != m:
                raise ValueError(f"state size {a.size} does not match model size {m}")
            self.ptr, self.where, self.obj = a.ctypes.data, MEM_HOST, a


def _out_like(x, m):
    if hasattr(x, "is_cuda") and x.is_cuda:
        import torch
        return torch.empty(m, dtype=torch.float64, device=x.device)
    return np.empty(m, dtype=np.float64)


# ---------------------------------------------------------------------------- model / workspace

@dataclass
class Model:
    """ModelSpec, reference layouts: LowRankFactors u (m, r), v (r, m) (kernels.hpp:26-35), or a
    DenseKernel k (m, m) (kernels.hpp:38-43; then u and v may be None)."""
    u: Optional[np.ndarray]
    v: Optional[np.ndarray]
    variant: int = AGGREGATION
    sources: Sequence = field(default_factory=list)  # [(k, rate)], 1-based k (SourceTerm)
    shatter_rate: float = 0.0
    k: Optional[np.ndarray] = None  # dense K(i,j) = k[i-1, j-1]

    def __post_init__(self):
        if self.k is not None:
            self.k = np.ascontiguousarray(self.k, dtype=np.float64)
            mk = self.k.shape[0]
            if self.k.shape != (mk, mk):
                raise ValueError("dense kernel must be m x m")
            if self.u is None:
                self.u = np.zeros((mk, 1))
            if self.v is None:
                self.v = np.zeros((1, mk))
        self.u = np.ascontiguousarray(self.u, dtype=np.float64)
        self.v = np.ascontiguousarray(self.v, dtype=np.float64)
        if self.u.ndim == 1:
            self.u = self.u.reshape(-1, 1)
        if self.v.ndim == 1:
            self.v = self.v.reshape(1, -1)

    @property
    def m(self):
        return self.u.shape[0]

    @property
    def r(self):
        return self.u.shape[1]


class RhsWorkspace:
    """RhsWorkspace + ModelSpec on the device (one per concurrent caller, rhs.hpp:42-44)."""

    def __init__(self, model: Optional[Model] = None, device: int = -1, *, fake: Optional[int] = None,
                 m: Optional[int] = None, param: float = 0.0):
        lib = load_library()
        self._h = C.c_void_p()
        if fake is not None:
            _check(lib.agk_rhs_create_fake(fake, m, param, device, C.byref(self._h)))
            self.m = m
            self.model = None
            return
        if model.v.shape != (model.r, model.m):
            raise ValueError("kernel size does not match m")
        sk = np.array([k for k, _ in model.sources] or [0], dtype=np.uint64)
        sr = np.array([rt for _, rt in model.sources] or [0.0], dtype=np.float64)
        d = _ModelDesc(model.m, model.r, model.u.ctypes.data_as(_dp), model.v.ctypes.data_as(_dp), model.variant,
                       sk.ctypes.data_as(C.POINTER(C.c_uint64)), sr.ctypes.data_as(_dp), len(model.sources),
                       float(model.shatter_rate), device,
                       model.k.ctypes.data_as(_dp) if model.k is not None else None)
        _check(lib.agk_rhs_create(C.byref(d), C.byref(self._h)))
        self.m = model.m
        self.model = model

    @property
    def handle(self):
        return self._h

    def evals(self) -> int:
        return int(load_library().agk_rhs_evals(self._h))

    def reset_evals(self):
        load_library().agk_rhs_reset_evals(self._h)

    def unique_ranks(self) -> int:
        return int(load_library().agk_rhs_unique_ranks(self._h))

    def launches_per_eval(self) -> int:
        return int(load_library().agk_rhs_launches_per_eval(self._h))

    def close(self):
        if getattr(self, "_h", None):
            load_library().agk_rhs_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def fake_rhs(kind: int, m: int, param: float = 0.0, device: int = -1) -> RhsWorkspace:
    """Injected RhsFn of the reference stepper tests, evaluated on the device."""
    return RhsWorkspace(fake=kind, m=m, param=param, device=device)


def _call_vec(fn, ws, n, *extra):
    a = _Arr(n, ws.m)
    out = _out_like(n, ws.m)
    o = _Arr(out, ws.m, writable=True)
    _check(fn(ws.handle, a.ptr, *extra, o.ptr, a.where), ws.handle)
    return out


def eval_rhs(ws: RhsWorkspace, n):
    """eval_rhs (rhs.cpp:212-235): S(n); counts one evaluation on the workspace."""
    return _call_vec(load_library().agk_rhs_eval, ws, n)


def birth_term(ws: RhsWorkspace, n):
    return _call_vec(load_library().agk_birth_term, ws, n)


def death_term(ws: RhsWorkspace, n):
    return _call_vec(load_library().agk_death_term, ws, n)


def shattering_terms(ws: RhsWorkspace, n, lam: float):
    a = _Arr(n, ws.m)
    out = _out_like(n, ws.m)
    o = _Arr(out, ws.m)
    _check(load_library().agk_shattering_terms(ws.handle, a.ptr, C.c_double(lam), o.ptr, a.where), ws.handle)
    return out


def euler_stability_bound(ws: RhsWorkspace, n, a: float) -> float:
    x = _Arr(n, ws.m)
    out = C.c_double()
    _check(load_library().agk_euler_stability_bound(ws.handle, x.ptr, C.c_double(a), C.byref(out), x.where),
           ws.handle)
    return out.value


# ---------------------------------------------------------------------------- steppers

@dataclass
class StepControl:
    """StepControl (steppers.hpp:18-36), reference defaults."""
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
        return _Control(self.stepper, self.mode, float(self.tau), float(self.tol), float(self.safety),
                        float(self.growth_max), float(self.shrink_min), float(self.tau_min),
                        int(self.max_rejects), int(bool(self.relative_error)))

    def validate(self):
        cc = self.c()
        if load_library().agk_control_validate(C.byref(cc)) != AGK_OK:
            raise ValueError("invalid step control")

    def effective_safety(self):
        if self.safety > 0.0:
            return self.safety
        return 0.9 if self.stepper == RKF45 else 0.25


@dataclass
class StepOutcome:
    state: Optional[np.ndarray]
    tau_used: float
    tau_next: float
    error_estimate: float
    rejects: int
    rhs_evals: int
    status: int

    def ok(self):
        return self.status == STEP_OK


def advance(ws: RhsWorkspace, n, tau: float, control: StepControl) -> StepOutcome:
    """advance (steppers.cpp:293-300); the trial loop and the controller run on the device."""
    a = _Arr(n, ws.m)
    state = _out_like(n, ws.m)
    s = _Arr(state, ws.m)
    o = _Outcome()
    cc = control.c()
    _check(load_library().agk_advance(ws.handle, a.ptr, C.c_double(tau), C.byref(cc), C.byref(o), s.ptr, a.where),
           ws.handle)
    return StepOutcome(state if o.status == STEP_OK else None, o.tau_used, o.tau_next, o.error_estimate,
                       o.rejects, o.rhs_evals, o.status)


def fixed_step(ws, n, tau, kind):
    return advance(ws, n, tau, StepControl(stepper=kind, mode=FIXED, tau=tau))


def step_doubling_adaptive(ws, n, tau, control: StepControl):
    if control.stepper not in (RK2, RK4):
        raise ValueError("step doubling applies to rk2 and rk4 only")
    return advance(ws, n, tau, control)


def fehlberg_adaptive(ws, n, tau, control: StepControl):
    if control.stepper != RKF45:
        raise ValueError("the embedded-pair rule applies to rkf45 only")
    return advance(ws, n, tau, control)


def _rk(ws, kind, n, tau, want5=False):
    a = _Arr(n, ws.m)
    out = _out_like(n, ws.m)
    o = _Arr(out, ws.m)
    out5 = _out_like(n, ws.m) if want5 else None
    p5 = _Arr(out5, ws.m).ptr if want5 else None
    err = C.c_double(math.nan)
    _check(load_library().agk_rk_step(ws.handle, kind, a.ptr, C.c_double(tau), o.ptr, p5, C.byref(err), a.where),
           ws.handle)
    return out, out5, err.value


def rk2_step(ws, n, tau):
    return _rk(ws, RK2, n, tau)[0]


def rk4_step(ws, n, tau):
    return _rk(ws, RK4, n, tau)[0]


def rkf45_step(ws, n, tau):
    """Returns (n4, n5, ||n5 - n4||_2) (steppers.cpp:124-159)."""
    return _rk(ws, RKF45, n, tau, want5=True)


# ---------------------------------------------------------------------------- run loop

@dataclass
class SimulationConfig:
    """SimulationConfig (simulator.hpp:24-37) with a custom initial state; the model is the workspace's."""
    control: StepControl
    t_end: float
    initial: np.ndarray
    initial_tau: float = 0.0
    snapshot_times: Sequence[float] = ()
    record: int = RECORD_NONE
    record_interval: float = 0.0


@dataclass
class RunReport:
    termination: str
    abort_reason: str
    abort_t: float
    abort_tau: float
    final_t: float
    final_state: np.ndarray
    snapshots: list
    records: list
    num_records: int
    total_rhs_evals: int
    total_accepted: int
    total_rejects: int
    wall_seconds: float


def run(ws: RhsWorkspace, cfg: SimulationConfig) -> RunReport:
    """run (simulator.cpp:112-229) as one device-resident CUDA graph."""
    m = ws.m
    init = np.ascontiguousarray(cfg.initial, dtype=np.float64).reshape(-1)
    if init.size != m:
        raise ValueError("custom initial state size does not match m")
    st = np.ascontiguousarray(cfg.snapshot_times, dtype=np.float64).reshape(-1)
    st_buf = st if st.size else np.zeros(1)
    final = np.zeros(m)
    snaps = np.zeros((max(st.size, 1), m))
    d = _RunDesc(cfg.control.c(), float(cfg.t_end), init.ctypes.data_as(_dp), float(cfg.initial_tau),
                 st_buf.ctypes.data_as(_dp), st.size, cfg.record, float(cfg.record_interval))
    rep = _Report()
    rep.final_state = final.ctypes.data_as(_dp)
    rep.snapshots = snaps.ctypes.data_as(_dp)
    # every record streams through the sink (the device drains its record ring between segments)
    chunks = []

    def _sink(_user, recs, n):
        chunks.append(np.ctypeslib.as_array(C.cast(recs, C.POINTER(C.c_uint8)), shape=(n * RECORD_DTYPE.itemsize,))
                      .view(RECORD_DTYPE).copy())

    sink = _RecordSink(_sink)
    if cfg.record != RECORD_NONE:
        rep.record_sink = sink
    _check(load_library().agk_run(ws.handle, C.byref(d), C.byref(rep)), ws.handle)
    arr = np.concatenate(chunks) if chunks else np.zeros(0, dtype=RECORD_DTYPE)
    records = [dict(zip(RECORD_DTYPE.names, row)) for row in arr.tolist()]
    snapshots = [(float(st[q]), snaps[q].copy()) for q in range(rep.num_snapshots_taken)]
    return RunReport("completed" if rep.termination == 0 else "aborted",
                     "" if rep.termination == 0 else describe(rep.abort_status), rep.abort_t, rep.abort_tau,
                     rep.final_t, final, snapshots, records, rep.num_records, rep.total_rhs_evals,
                     rep.total_accepted, rep.total_rejects, rep.wall_seconds)


KERNEL_CLASSES = ("small", "col_fwd", "row", "col_inv", "transpose", "dvec", "row_inv", "dense_rows", "dense_birth")


def eval_rhs_timed(ws: RhsWorkspace, n_dev, out_dev, count: int) -> float:
    """Device milliseconds for `count` back-to-back evaluations on device tensors (CUDA events
    on the workspace's stream around the captured per-RHS graph)."""
    ms = C.c_float()
    _check(load_library().agk_rhs_eval_timed(ws.handle, n_dev.data_ptr(), out_dev.data_ptr(), count, C.byref(ms)),
           ws.handle)
    return ms.value


def profile_rhs(ws: RhsWorkspace, n_dev, out_dev, reps: int = 5):
    """Per-launch device times of one evaluation: [(class, ms)], plus (log2P, N1, N2, group)."""
    cap = 256
    ms = (C.c_double * cap)()
    cls = (C.c_int * cap)()
    nk = C.c_int()
    plan = (C.c_int * 4)()
    _check(load_library().agk_rhs_profile(ws.handle, n_dev.data_ptr(), out_dev.data_ptr(), reps, ms, cls, cap,
                                          C.byref(nk), plan), ws.handle)
    return [(KERNEL_CLASSES[cls[i]], ms[i]) for i in range(nk.value)], tuple(plan)


def moments(n, orders=(0, 1, 2)):
    """moments (simulator.cpp:53-68) — host helper for reports and tests."""
    n = np.asarray(n, dtype=np.float64)
    k = np.arange(1, n.size + 1, dtype=np.float64)
    return tuple(float(np.sum(k ** p * n)) for p in orders)
