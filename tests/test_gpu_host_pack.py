"""hs_eval_host's host-side packing (csrc/host_pack.cpp): uint8 genomes in
the reference's layout, packed to 2 bits per gene by the host thread pool
chunk by chunk while the GPU works, must give exactly the unpacked path's
makespans, statuses and best -- including a chunk that holds an
out-of-range gene (sent unpacked, flagged status 5 by the kernel), strided
rows and a ragged last chunk."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import instance_doc

import paper_2308_00127_b200 as hs
from paper_2308_00127_b200 import _native as N
from paper_2308_00127_b200.plan import get_plan

pytestmark = pytest.mark.gpu


def _host(plan, genes, monkeypatch, pack):
    monkeypatch.setenv("HS_HOST_PACK", "1" if pack else "0")  # forced either way
    n = len(genes)
    ms = np.empty(n, np.float64)
    st = np.empty(n, np.uint8)
    b = N.Best()
    plan.eval_host(genes, ms, st, b)
    return ms, st, (b.cost, b.index)


@pytest.mark.parametrize("name", ["ws200", "ws30", "rn50f"])
def test_host_pack_equals_unpacked(name, monkeypatch):
    g, hw, t = hs.load_instance(instance_doc(name))
    plan = get_plan(g, hw, t, 1)
    rng = np.random.default_rng(11)
    n = (1 << 20) + 12345  # ragged last chunk
    genes = rng.integers(plan.K, size=(n, plan.V), dtype=np.uint8)
    a = _host(plan, genes, monkeypatch, True)
    b = _host(plan, genes, monkeypatch, False)
    assert np.array_equal(a[0].view(np.uint64), b[0].view(np.uint64))
    assert np.array_equal(a[1], b[1]) and a[2] == b[2]


def test_host_pack_bad_gene_and_stride(monkeypatch):
    g, hw, t = hs.load_instance(instance_doc("ws200"))
    plan = get_plan(g, hw, t, 1)
    rng = np.random.default_rng(12)
    n = 700_001
    wide = rng.integers(3, size=(n, plan.V + 9), dtype=np.uint8)
    wide[600_000, 17] = 3  # gene >= K in the second chunk
    genes = wide[:, :plan.V]  # row stride V + 9
    a = _host(plan, genes, monkeypatch, True)
    b = _host(plan, np.ascontiguousarray(genes), monkeypatch, False)
    assert a[1][600_000] == N.ST_GENE
    assert np.array_equal(a[1], b[1])
    ok = a[1] < N.ST_MISSING
    assert np.array_equal(a[0][ok].view(np.uint64), b[0][ok].view(np.uint64))
    assert a[2] == b[2]
