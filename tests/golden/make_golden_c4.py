"""Config-4 golden (TEST INFRASTRUCTURE): the REFERENCE's own eval_rhs (oracle/_ref) on BASELINE
config 4 (M = 2^20, R = 16 random low-rank kernel, std::mt19937_64 inputs, configs.py), stored
compactly for smoke() and the GPU tests on boxes without /root/reference:
  idx: 8192 sampled sizes (the first 1024, then spread over the rest), S: S(n) there,
  maxabs: max |S| over all sizes (the normwise denominator), sum: sum of S.

    make -C oracle ref && python tests/golden/make_golden_c4.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402
from paper_2407_16559_b200.configs import random_config4  # noqa: E402


def main():
    U, V, n = random_config4()
    m = n.size
    S = O.Oracle("reference").eval_rhs(O.Model(U, V), n)
    idx = np.unique(np.concatenate([np.arange(1024), np.linspace(1024, m - 1, 7168).astype(np.int64)]))
    np.savez_compressed(os.path.join(HERE, "golden_c4.npz"), idx=idx, S=S[idx], maxabs=np.max(np.abs(S)),
                        sum=np.sum(S), n_checksum=np.sum(n))
    print("config 4 golden:", idx.size, "samples, max|S|", np.max(np.abs(S)))


if __name__ == "__main__":
    main()
