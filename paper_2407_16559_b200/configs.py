"""Kernel factor builders and the BASELINE.json workloads (synthetic, seeded).

Factor layouts are the reference's (kernels.hpp:26-35): U is m x r row-major, V is r x m.
  constant          K = 1, R = 1                          (kernels.cpp:64-69)
  brownian(alpha)   (i/j)^a + (j/i)^a, R = 2, bitwise-reciprocal columns (kernels.cpp:74-85)
  brownian_plus2    (i/j)^(1/3) + (j/i)^(1/3) + 2, R = 3   (BASELINE configs 2 and 5)
  random_config4    U_ia = u_a i^p_a, V_aj = v_a j^-p_a, R = 16 (BASELINE config 4)
Inputs are generated on the host by std::mt19937_64 seeded with 0x5eed5eed (the reference's
verify seed, verify.cpp:19) and libstdc++'s uniform_real_distribution<double>, restated below in
numpy (Mt19937_64), so a C++ caller regenerates bit-identical arrays (
tests/test_configs_rng.py checks it against the C++ standard library). The same arrays feed the GPU
path and the CPU oracle.
"""
from __future__ import annotations

import numpy as np

SEED = 0x5EED5EED


class Mt19937_64:
    """std::mt19937_64 (64-bit Mersenne Twister, the C++ standard's parameters) with
    std::uniform_real_distribution<double>(a, b) as libstdc++ computes it: generate_canonical
    draws ONE 64-bit word x (53 digits <= 64 bits) and returns double(x) / 2^64 (nextafter(1, 0)
    if that rounds to 1), then a + u (b - a)."""
    NN, MM = 312, 156
    MATRIX_A = np.uint64(0xB5026F5AA96619E9)
    UM, LM = np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)

    def __init__(self, seed=SEED):
        mt = [int(seed) & 0xFFFFFFFFFFFFFFFF]
        for i in range(1, self.NN):
            prev = mt[-1]
            mt.append((6364136223846793005 * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF)
        self.mt = np.array(mt, dtype=np.uint64)
        self.idx = self.NN

    def _twist(self):
        mt, N, M = self.mt, self.NN, self.MM
        one = np.uint64(1)

        def mix(cur, nxt, far):
            x = (cur & self.UM) | (nxt & self.LM)
            return far ^ (x >> one) ^ np.where((x & one) != 0, self.MATRIX_A, np.uint64(0))

        mt[:N - M] = mix(mt[:N - M], mt[1:N - M + 1], mt[M:N])                 # far words not yet updated
        mt[N - M:N - 1] = mix(mt[N - M:N - 1], mt[N - M + 1:N], mt[0:M - 1])  # far words already new
        mt[N - 1:N] = mix(mt[N - 1:N], mt[0:1], mt[M - 1:M])
        self.idx = 0

    def raw(self, n):
        out = np.empty(n, dtype=np.uint64)
        k = 0
        while k < n:
            if self.idx >= self.NN:
                self._twist()
            take = min(n - k, self.NN - self.idx)
            y = self.mt[self.idx:self.idx + take].copy()
            y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
            y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
            y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
            y ^= y >> np.uint64(43)
            out[k:k + take] = y
            self.idx += take
            k += take
        return out

    def uniform(self, a, b, n=None):
        cnt = 1 if n is None else n
        u = self.raw(cnt).astype(np.float64) / 18446744073709551616.0  # round-to-nearest, then / 2^64
        u = np.where(u >= 1.0, np.nextafter(1.0, 0.0), u)
        x = u * (b - a) + a
        return float(x[0]) if n is None else x


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
    rng = Mt19937_64(seed)
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
    n = np.exp(-i / 1000.0) * rng.uniform(0.9, 1.1, m)
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
