"""Module detection (csrc/decomp.cpp through hs_bridges_articulation /
hs_k_edge_components) against what the reference returned
(tests/golden/decomp.json, made by make_golden_r2.py from
splitting.py:36-81 and :178-219 with networkx's k_edge_components): the
bridges in edge order, the articulation set, connectivity, and for c = 1, 2,
3 the modules in the reference's lexicographic topological order with the
cut edges per module pair in edge order. Host-only: runs without a GPU."""
from __future__ import annotations

import json

import pytest

from conftest import INSTANCES, golden, instance_doc

import paper_2308_00127_b200 as hs
from paper_2308_00127_b200.core import GraphError, load_graph


def _entries():
    return golden("decomp")


def _graph(e):
    if "graph" in e:
        return load_graph(json.dumps(e["graph"]))
    return hs.load_instance(instance_doc(e["name"]))[0]


def _check(g, e):
    bridges, artic, conn = hs.find_bridges_and_articulation_points(g)
    assert [list(x) for x in bridges] == e["bridges"]
    assert sorted(artic) == e["articulation"]
    assert conn == e["connected"]
    for c, want in e["k_edge"].items():
        d = hs.k_edge_components(g, int(c))
        assert [sorted(m) for m in d.modules] == want["modules"], c
        got_cuts = [[a, b, [list(x) for x in es]]
                    for (a, b), es in d.cut_edges.items()]
        assert sorted(got_cuts) == sorted(want["cuts"]), c
        # per module pair the edges keep the graph's edge order
        assert {(a, b): es for a, b, es in got_cuts} == \
            {(a, b): es for a, b, es in want["cuts"]}
        assert d.is_chain == want["is_chain"]
        assert d.channels == int(c)
        assert sorted(t for m in d.modules for t in m) == sorted(g.tasks)


@pytest.mark.parametrize("name", INSTANCES)
def test_decomposition_instances(name):
    e = next(x for x in _entries() if x["name"] == name)
    _check(_graph(e), e)


def test_decomposition_random_graphs():
    extra = [e for e in _entries() if "graph" in e]
    assert len(extra) >= 90
    for e in extra:
        _check(_graph(e), e)


def test_decomposition_json_round_trip():
    g = hs.load_instance(instance_doc("ws_stack_10x20"))[0]
    d = hs.k_edge_components(g, 1)
    d2 = hs.ModuleDecomposition.from_json(d.to_json())
    assert d2.modules == d.modules and d2.cut_edges == d.cut_edges
    assert len(d.modules) == 10 and d.is_chain and d.max_cut_width() == 1
    with pytest.raises(GraphError):
        hs.ModuleDecomposition.from_json('{"modules": []}')


def test_decomposition_rejects_bad_budget():
    g = hs.load_instance(instance_doc("ws30"))[0]
    with pytest.raises(GraphError):
        hs.k_edge_components(g, 0)


def test_decomposition_matches_live_reference():
    """Random DAGs beyond the fixture, against the reference itself when it
    is importable (this container, or oracle/_ref on the GPU box)."""
    import sys

    import numpy as np
    from oracle import ref
    if ref.import_reference() is None:
        pytest.skip("reference not importable")
    RS = sys.modules["hetsched.splitting"]
    RC = sys.modules["hetsched.core"]
    for seed in range(40):
        rng = np.random.default_rng(1000 + seed)
        n = int(rng.integers(2, 30))
        p = float(rng.uniform(0.05, 0.5))
        ids = [f"v{int(x):03d}" for x in rng.permutation(n * 2)[:n]]
        edges = [(ids[a], ids[b]) for a in range(n) for b in range(a + 1, n)
                 if rng.random() < p]
        rg = RC.DnnGraph([RC.TaskNode(id=i) for i in ids], edges)
        g = load_graph(RC.save_graph(rg))
        rb, ra, rc = RS.find_bridges_and_articulation_points(rg)
        b, a, c = hs.find_bridges_and_articulation_points(g)
        assert (b, a, c) == (rb, ra, rc)
        for k in (1, 2, 3):
            rd, d = RS.k_edge_components(rg, k), hs.k_edge_components(g, k)
            assert d.modules == rd.modules and d.cut_edges == rd.cut_edges
            assert d.is_chain == rd.is_chain
