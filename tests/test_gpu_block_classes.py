"""Node-block link classes in the specialised evaluator (jit.cpp,
`block_classes`): on full-mesh multi-server platforms whose link class is
(same device, same node, other node) with nodes as blocks of consecutive
sorted devices -- the paper's transformer case study -- the class is
computed from the genes instead of looked up. Differential test against
the plan-walking AOT kernel (pinned to the reference's goldens, which use
the class tables) on random graphs, node counts, node sizes and
bandwidths, plus the golden transformer cases through the block path."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import case_genes, fhex, instance_doc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2308_00127_b200 as hs  # noqa: E402
from paper_2308_00127_b200.core import (Device, DnnGraph,  # noqa: E402
                                        HardwareSystem, LatencyTable,
                                        TaskNode)
from paper_2308_00127_b200.plan import Plan  # noqa: E402


def _instance(seed):
    rng = np.random.default_rng(seed)
    nodes = int(rng.integers(2, 7))
    per = int(rng.integers(2, 6))
    devs = [f"n{a:02d}_d{b}" for a in range(nodes) for b in range(per)]
    # one intra-node and one inter-node bandwidth (the block structure)
    bi, bo = float(rng.uniform(1e6, 1e7)), float(rng.uniform(1e4, 1e5))
    hw = HardwareSystem([Device(d, 1e12, (1, 2)) for d in devs],
                        {(u, v): bi if u[:3] == v[:3] else bo
                         for u in devs for v in devs if u != v})
    V = int(rng.integers(20, 120))
    ids = [f"t{k:03d}" for k in range(V)]
    tasks = [TaskNode(i, float(rng.uniform(0, 10)), float(rng.uniform(0, 5)),
                      float(rng.uniform(0, 1e5)) * (rng.random() < 0.9))
             for i in ids]
    edges = [(ids[a], ids[b]) for a in range(V)
             for b in range(a + 1, min(V, a + 12)) if rng.random() < 0.25]
    g = DnnGraph(tasks, edges)
    table = LatencyTable({(i, d, b): float(rng.uniform(0.5, 20.0)) * b
                          for i in ids for d in devs for b in (1, 2)})
    return g, hw, table


def _eval(plan, genes):
    d = torch.from_numpy(genes).cuda()
    ms = torch.empty(len(genes), dtype=torch.float64, device="cuda")
    st = torch.empty(len(genes), dtype=torch.uint8, device="cuda")
    plan.eval(d, ms, st, None)
    return ms.cpu().numpy(), st.cpu().numpy()


@pytest.mark.parametrize("seed", range(8))
def test_block_classes_equal_table_classes(seed):
    g, hw, t = _instance(seed)
    for L in (1, 2):
        jit = Plan(g, hw, t, L)
        src = jit.specialized_source(128)
        assert "BCL[" not in src and ">> " in src  # block path emitted
        jit.specialize()
        aot = Plan(g, hw, t, L)
        rng = np.random.default_rng(100 + seed)
        genes = rng.integers(jit.K, size=(50_000, jit.pref_ld),
                             dtype=np.uint8)
        a = _eval(jit, genes)
        b = _eval(aot, genes)
        assert np.array_equal(a[1], b[1])
        assert np.array_equal(a[0].view(np.uint64), b[0].view(np.uint64))


def test_transformer_golden_through_block_path():
    doc = instance_doc("tf96")
    g, hw, t = hs.load_instance(doc)
    for case in doc["cases"]:
        plan = Plan(g, hw, t, case["L"])
        assert "BCL[" not in plan.specialized_source(128)
        plan.specialize()
        genes = case_genes(case)
        rows = np.zeros((len(genes), plan.pref_ld), np.uint8)
        rows[:, :plan.V] = genes
        ms, st = _eval(plan, rows)
        got = ["GraphError" if s >= 4 else fhex(v) for v, s in zip(ms, st)]
        assert got == case["expected"]
