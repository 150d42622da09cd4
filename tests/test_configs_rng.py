"""the synthetic inputs are std::mt19937_64(0x5eed5eed) draws, so a C++ caller
regenerates them. configs.Mt19937_64 is checked bit for bit against the C++ standard library
(g++ here), over enough draws to cross many 312-word twists."""
import os
import subprocess

import numpy as np
import pytest

from paper_2407_16559_b200.configs import Mt19937_64, random_config4

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def cxx_draws(tmp_path_factory):
    exe = tmp_path_factory.mktemp("rng") / "config4_inputs"
    try:
        subprocess.run(["g++", "-std=c++17", "-O2", "-o", str(exe), os.path.join(HERE, "cpp", "config4_inputs.cpp")],
                       check=True, capture_output=True)
    except (OSError, subprocess.CalledProcessError) as e:
        pytest.skip(f"no C++ compiler: {e}")
    out = subprocess.run([str(exe), "16", "5000"], check=True, capture_output=True, text=True).stdout.split()
    return np.array([int(x, 16) for x in out], dtype=np.uint64).view(np.float64)


def test_draws_bitwise(cxx_draws):
    g = Mt19937_64()
    mine = []
    for _ in range(16):
        mine += [g.uniform(0.5, 1.5), g.uniform(0.5, 1.5), g.uniform(-0.5, 0.5)]
    mine = np.concatenate([np.array(mine), g.uniform(0.9, 1.1, 5000)])
    assert np.array_equal(mine.view(np.uint64), cxx_draws.view(np.uint64))


def test_config4_uses_the_draws(cxx_draws):
    U, V, n = random_config4(5000, 16)
    d = cxx_draws[:48].reshape(16, 3)
    i = np.arange(1, 5001, dtype=np.float64)
    # U_ia = u_a i^p_a, V_aj = v_a j^-p_a, n_s = exp(-s/1000) U(0.9, 1.1): the draws are bitwise
    # the C++ ones; pow/exp may differ from a C++ libm by an ulp (numpy's SIMD transcendental paths)
    assert np.allclose(U, d[:, 0][None, :] * i[:, None] ** d[:, 2][None, :], rtol=4e-16, atol=0)
    assert np.allclose(V, d[:, 1][:, None] * i[None, :] ** (-d[:, 2][:, None]), rtol=4e-16, atol=0)
    assert np.allclose(n, np.exp(-i / 1000.0) * cxx_draws[48:], rtol=4e-16, atol=0)
