"""N > 1 path on CPU: two gloo ranks run independent replica workloads (the oracle RHS on
different seeds), the timed region is bracketed by barriers and reduced with max-over-ranks —
the same plumbing bench.py uses under torchrun with nccl."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2407_16559_b200 import replicas
    from oracle.oracle import Model, Oracle, constant_factors
    w, r, local = replicas.setup("gloo")
    u, v = constant_factors(512)
    n = np.random.default_rng(r).random(512)
    replicas.barrier(w)
    out = Oracle("port").eval_rhs(Model(u, v), n)      # replica workload, no data exchange
    my_time = 0.5 + r                                   # deterministic per-rank "device time"
    mx = replicas.max_over_ranks(my_time, w, local)
    replicas.barrier(w)
    rate = replicas.aggregate_rate(10, mx, w)
    q.put((r, mx, rate, float(out.sum())))
    replicas.teardown(w)


def test_two_gloo_replicas():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [x[1] for x in res] == [1.5, 1.5]           # max over ranks
    assert all(abs(x[2] - 2 * 10 / 1.5) < 1e-12 for x in res)
    assert res[0][3] != res[1][3]                       # independent workloads


def test_single_rank_is_identity():
    from paper_2407_16559_b200 import replicas
    assert replicas.setup() == (1, 0, 0)
    assert replicas.max_over_ranks(3.0, 1) == 3.0
    assert replicas.aggregate_rate(20, 2.0, 1) == 10.0
