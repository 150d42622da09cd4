"""Shared test helpers: the reference's error metric and model builders."""
import numpy as np

from oracle import oracle as O


def rel_max_diff(got, want):
    """Normwise relative error max|got-want| / max|want| (test_rhs.cpp:21-28)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    num = np.max(np.abs(got - want)) if got.size else 0.0
    den = np.max(np.abs(want)) if want.size else 0.0
    return num / den if den > 0 else num


def random_state(rng, m):
    return rng.random(m)


def factors(kind, m, alpha=0.0):
    if kind == "constant":
        return O.constant_factors(m)
    if kind == "brownian":
        return O.brownian_factors(m, alpha)
    if kind == "brownian2":
        return O.brownian_plus2_factors(m)
    raise ValueError(kind)


def config4_inputs(m=1 << 20, r=16):
    """BASELINE config 4 inputs (paper_2407_16559_b200/configs.py, seed 0x5eed5eed)."""
    from paper_2407_16559_b200.configs import random_config4
    return random_config4(m, r)
