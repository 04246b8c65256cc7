"""Multi-rank logic on CPU: world_size 2 over gloo. Each rank evaluates its
shard of a candidate batch with the (pinned) oracle standing in for the GPU
evaluator, and the single all-gather + lexicographic merge must reproduce
the single-process numpy.argmin of the whole batch on every rank."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import instance_doc
from paper_2308_00127_b200.dist import merge_best, shard_range

INF = float("inf")


def test_shard_ranges_cover_exactly():
    for n in (0, 1, 7, 100, 101, 4097):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def test_merge_best_semantics():
    assert merge_best([(3.0, 5), (1.0, 9), (1.0, 2)]) == (1.0, 2)
    assert merge_best([(INF, 4), (INF, 1)]) == (INF, 1)
    assert merge_best([(INF, -1), (2.0, 8)]) == (2.0, 8)
    assert merge_best([]) == (INF, -1)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, genes, out):
    import torch.distributed as dist
    from oracle import hs_oracle as O
    from paper_2308_00127_b200.dist import sharded_best
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tb = O.build_tables(O.Instance.from_doc(instance_doc("ws30")), 1)

    def ev(lo, hi):
        ms, _ = O.fitness_np(tb, genes[lo:hi])
        c, k = O.argmin_first(ms)
        return c, lo + k

    out[rank] = sharded_best(len(genes), ev)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_argmin(world):
    from oracle import hs_oracle as O
    tb = O.build_tables(O.Instance.from_doc(instance_doc("ws30")), 1)
    genes = np.random.default_rng(3).integers(3, size=(3001, tb.V),
                                              dtype=np.uint8)
    genes[2000] = genes[17]  # a tie across the shard boundary
    ms, _ = O.fitness_np(tb, genes)
    want = O.argmin_first(ms)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _port(), genes, out),
                       nprocs=world, join=True, start_method="fork")
    assert dict(out) == {r: want for r in range(world)}
