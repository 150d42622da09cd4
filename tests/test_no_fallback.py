"""The product path has no CPU fallback: a missing library and a missing GPU both fail loudly
(never route through the oracle or any host computation)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(code, env_extra):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                          timeout=300)


def test_missing_library_raises():
    code = ("import numpy as np, paper_2407_16559_b200 as agk\n"
            "try:\n"
            "    agk.RhsWorkspace(agk.Model(np.ones((8, 1)), np.ones((1, 8))))\n"
            "except ImportError as e:\n"
            "    print('RAISED', e)\n")
    r = _run(code, {"AGK_LIB": "/nonexistent/libagk_b200.so"})
    assert r.returncode == 0, r.stderr
    assert "RAISED" in r.stdout and "no CPU fallback" in r.stdout


def test_no_gpu_raises_instead_of_computing():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    if not os.path.exists(os.path.join(ROOT, "paper_2407_16559_b200", "libagk_b200.so")):
        pytest.skip("library not built")
    code = ("import numpy as np, paper_2407_16559_b200 as agk\n"
            "try:\n"
            "    ws = agk.RhsWorkspace(agk.Model(np.ones((8, 1)), np.ones((1, 8))), device=0)\n"
            "    print('COMPUTED', agk.eval_rhs(ws, np.ones(8)))\n"
            "except Exception as e:\n"
            "    print('RAISED', type(e).__name__, e)\n")
    r = _run(code, {})
    assert r.returncode == 0, r.stderr
    assert "RAISED" in r.stdout and "COMPUTED" not in r.stdout, r.stdout


def test_production_library_reads_no_experiment_knobs():
    """the AGK_* experiment switches (tools/ab.sh) exist only in the
    -DAGK_EXPERIMENTS build (libagk_b200_exp.so); the production library cannot see them, so no
    stray environment variable can change a plan or skip work in a timed or parity run."""
    blob = open(os.path.join(ROOT, "paper_2407_16559_b200", "libagk_b200.so"), "rb").read()
    for knob in (b"AGK_DBG", b"AGK_PFD", b"AGK_FAST", b"AGK_RANK_GROUP", b"AGK_PDL", b"AGK_VARIANT", b"AGK_MVAR",
                 b"AGK_FUSE_STAGES", b"AGK_DVEC_MODE"):
        assert knob not in blob, knob
