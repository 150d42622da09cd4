"""Kernel factor builders and the BASELINE.json workloads (synthetic, seeded).

Factor layouts are the reference's (kernels.hpp:26-35): U is m x r row-major, V is r x m.
  constant          K = 1, R = 1                          (kernels.cpp:64-69)
  brownian(alpha)   (i/j)^a + (j/i)^a, R = 2, bitwise-reciprocal columns (kernels.cpp:74-85)
  brownian_plus2    (i/j)^(1/3) + (j/i)^(1/3) + 2, R = 3   (BASELINE configs 2 and 5)
  random_config4    U_ia = u_a i^p_a, V_aj = v_a j^-p_a, R = 16 (BASELINE config 4)
Inputs are generated on the host from numpy's MT19937 seeded with 0x5eed5eed (the reference's
verify seed, verify.cpp:19); the same arrays feed the GPU path and the CPU oracle.
"""
from __future__ import annotations

import numpy as np

SEED = 0x5EED5EED


def constant_factors(m):
    return np.ones((m, 1)), np.ones((1, m))


def brownian_factors(m, alpha):
    i = np.arange(1, m + 1, dtype=np.float64)
    p = np.power(i, alpha)
    return np.stack([p, 1.0 / p], axis=1), np.stack([1.0 / p, p], axis=0)


def brownian_plus2_factors(m):
    i = np.arange(1, m + 1, dtype=np.float64)
    p = np.power(i, 1.0 / 3.0)
    s2 = np.sqrt(2.0)
    return (np.stack([p, 1.0 / p, np.full(m, s2)], axis=1),
            np.stack([1.0 / p, p, np.full(m, s2)], axis=0))


def random_config4(m=1 << 20, r=16, seed=SEED):
    """BASELINE config 4: draws u_a, v_a ~ U(0.5,1.5) then p_a ~ U(-0.5,0.5) per rank, then
    n_s = exp(-s/1000) * U(0.9,1.1)."""
    rng = np.random.Generator(np.random.MT19937(seed))
    u = np.empty(r)
    v = np.empty(r)
    p = np.empty(r)
    for a in range(r):
        u[a] = rng.uniform(0.5, 1.5)
        v[a] = rng.uniform(0.5, 1.5)
        p[a] = rng.uniform(-0.5, 0.5)
    i = np.arange(1, m + 1, dtype=np.float64)
    U = np.ascontiguousarray(u[None, :] * i[:, None] ** p[None, :])
    V = np.ascontiguousarray(v[:, None] * i[None, :] ** (-p[:, None]))
    n = np.exp(-i / 1000.0) * rng.uniform(0.9, 1.1, size=m)
    return U, V, n


def monodisperse(m):
    n = np.zeros(m)
    n[0] = 1.0
    return n


def baseline_config(idx: int):
    """BASELINE.json configs[idx-1] as a dict: factors, variant, sources, lambda, initial state,
    tol, t_end. (rtol maps to the reference's absolute-L2 tol; atol has no reference
    counterpart, SURVEY §8c note 1.)"""
    if idx == 1:
        u, v = constant_factors(4096)
        return dict(u=u, v=v, variant=0, sources=[], lam=0.0, n0=monodisperse(4096), tol=1e-6, t_end=100.0)
    if idx == 2:
        u, v = brownian_plus2_factors(1 << 16)
        return dict(u=u, v=v, variant=1, sources=[(1, 1.0)], lam=0.0, n0=np.zeros(1 << 16), tol=1e-6, t_end=1e4)
    if idx == 3:
        u, v = brownian_factors(1 << 17, 0.9)
        return dict(u=u, v=v, variant=2, sources=[], lam=0.01, n0=monodisperse(1 << 17), tol=1e-8, t_end=5000.0)
    if idx == 4:
        U, V, n = random_config4()
        return dict(u=U, v=V, variant=0, sources=[], lam=0.0, n0=n, tol=None, t_end=None)
    if idx == 5:
        u, v = brownian_plus2_factors(1 << 20)
        return dict(u=u, v=v, variant=1, sources=[(1, 1.0)], lam=0.0, n0=np.zeros(1 << 20), tol=1e-6, t_end=1e5)
    raise ValueError(idx)
