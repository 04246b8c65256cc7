"""Lower-bound building blocks on the GPU against the reference's recorded
critical paths, dep/pre closures and subgraph_cap=0 lower bounds
(tests/golden/bounds.json)."""
from __future__ import annotations

import pytest

from conftest import fhex, golden, instance_doc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2308_00127_b200 as hs  # noqa: E402


class _Decomp:
    def __init__(self, doc):
        self.modules = [frozenset(m) for m in doc["modules"]]
        self.cut_edges = {(c["from"], c["to"]): [tuple(e) for e in c["edges"]]
                          for c in doc["cuts"]}


@pytest.mark.parametrize("k", range(5))
def test_bounds(k):
    entries = golden("bounds")
    if k >= len(entries):
        pytest.skip("no entry")
    e = entries[k]
    g, hw, t = hs.load_instance(instance_doc(e["instance"]))
    vals = hs.critical_path_bounds(g, hw, t, [c["tasks"] for c in
                                              e["critical_path"]])
    assert [fhex(v) for v in vals] == [c["value"] for c in e["critical_path"]]
    assert fhex(hs.critical_path_bound(g, hw, t,
                                       e["critical_path"][0]["tasks"])) == \
        e["critical_path"][0]["value"]
    for r in e["reach"]:
        assert sorted(hs.dep_subgraph(g, r["u"], r["T"])) == r["dep"]
        assert sorted(hs.pre_subgraph(g, r["u"], r["T"])) == r["pre"]
    d = _Decomp(e["decomposition"])
    for lb in e["lower_bound_cap0"]:
        rep = hs.lower_bound(g, hw, t, lb["L"], d, subgraph_cap=0)
        assert fhex(rep.lower_bound_ms) == lb["lower_bound_ms"]
        assert fhex(rep.throughput_upper_bound) == lb["throughput_upper_bound"]
        assert rep.terms == lb["terms"]


def test_critical_path_known_answers():
    T = hs.TaskNode
    g = hs.DnnGraph([T("a"), T("b")], [("a", "b")])
    hw = hs.HardwareSystem([hs.Device("d0", 1e9, (1,)),
                            hs.Device("d1", 1e9, (1,))],
                           {("d0", "d1"): 1.0, ("d1", "d0"): 1.0})
    t = hs.LatencyTable({(i, u, 1): (2.0 if i == "a" else 3.0) *
                         (1.0 if u == "d0" else 2.0)
                         for i in "ab" for u in ("d0", "d1")})
    assert hs.critical_path_bound(g, hw, t, {"a", "b"}) == 5.0  # bounds:46-53
    assert hs.critical_path_bound(g, hw, t, set()) == 0.0
    missing = hs.LatencyTable({("a", "d0", 1): 1.0})
    with pytest.raises(hs.GraphError):
        hs.critical_path_bound(g, hw, missing, {"a"})


def test_transitive_closure():
    doc = instance_doc("er_stack_10x10")
    g, _, _ = hs.load_instance(doc)
    tc = hs.transitive_closure(g)
    for u in list(g.tasks)[:20]:
        seen, stack = set(), [u]
        while stack:
            for w in g.succ[stack.pop()]:
                if w not in seen:
                    seen.add(w)
                    stack.append(w)
        assert tc[u] == seen
