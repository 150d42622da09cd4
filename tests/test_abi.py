"""CPU-side checks of the C-ABI library: it loads, exports every entry point include/agk/agk.h
declares, the Python mirror binds them all, and without a B200 it refuses to run (no fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "agk", "agk.h")
LIB = os.path.join(ROOT, "paper_2407_16559_b200", "libagk_b200.so")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(agk_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("agk_rhs_create", "agk_rhs_eval", "agk_advance", "agk_run", "agk_birth_term",
                 "agk_death_term", "agk_shattering_terms", "agk_euler_stability_bound", "agk_rhs_evals"):
        assert must in names


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build libagk_b200.so first (make -C paper_2407_16559_b200)"
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_mirror_binds_every_symbol():
    import paper_2407_16559_b200 as agk
    assert set(agk.exported_symbols()) == set(declared_functions())
    agk.load_library()


def test_control_defaults_and_validation():
    import paper_2407_16559_b200 as agk
    c = agk._Control()
    agk.load_library().agk_control_defaults(ctypes.byref(c))
    assert (c.stepper, c.mode, c.tol, c.growth_max, c.shrink_min, c.tau_min, c.max_rejects) == \
           (agk.RKF45, agk.ADAPTIVE, 1e-6, 2.0, 0.5, 1e-12, 40)      # steppers.hpp:18-36
    agk.StepControl().validate()
    with pytest.raises(ValueError):
        agk.StepControl(safety=1.5).validate()
    with pytest.raises(ValueError):
        agk.StepControl(mode=agk.FIXED, tau=0.0).validate()
    with pytest.raises(ValueError):
        agk.StepControl(growth_max=0.9).validate()
    assert agk.describe(agk.STEP_TAU_UNDERFLOW) == "step size underflow"   # simulator.cpp:98-110


def test_no_cpu_fallback_without_gpu():
    from tests.conftest import has_gpu
    if has_gpu():
        pytest.skip("a GPU is present")
    import paper_2407_16559_b200 as agk
    with pytest.raises(RuntimeError, match="no CUDA device"):
        agk.RhsWorkspace(agk.Model(np.ones((8, 1)), np.ones((1, 8))))
    with pytest.raises(RuntimeError):
        agk.fake_rhs(agk.RHS_DECAY, 4)
