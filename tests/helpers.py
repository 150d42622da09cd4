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


def config4_inputs(m=1 << 20, r=16, seed=0x5EED5EED):
    """BASELINE config 4: U_ia = u_a i^p_a, V_aj = v_a j^-p_a, n_s = exp(-s/1000) U(0.9,1.1)
    (SURVEY §8d draw order: u_a, v_a then p_a per rank, then n)."""
    rng = np.random.Generator(np.random.MT19937(seed))
    u = np.empty(r)
    v = np.empty(r)
    p = np.empty(r)
    for a in range(r):
        u[a] = rng.uniform(0.5, 1.5)
        v[a] = rng.uniform(0.5, 1.5)
        p[a] = rng.uniform(-0.5, 0.5)
    i = np.arange(1, m + 1, dtype=np.float64)
    U = np.ascontiguousarray((u[None, :] * i[:, None] ** p[None, :]))
    V = np.ascontiguousarray((v[:, None] * i[None, :] ** (-p[:, None])))
    s = np.arange(1, m + 1, dtype=np.float64)
    n = np.exp(-s / 1000.0) * rng.uniform(0.9, 1.1, size=m)
    return U, V, n
