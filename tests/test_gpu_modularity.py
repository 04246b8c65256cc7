"""The partition scorer against networkx.community.modularity (bit-exact:
same binary64 sequence), on the golden graphs' module decompositions and on
random partitions."""
from __future__ import annotations

import networkx as nx
import numpy as np
import pytest

from conftest import instance_doc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2308_00127_b200 as hs  # noqa: E402


def _nx(g, comms, res=1.0):
    sh = nx.Graph()
    sh.add_nodes_from(g.tasks)
    sh.add_edges_from(g.edges)
    return nx.community.modularity(sh, comms, resolution=res)


@pytest.mark.parametrize("name", ["ws_stack_10x20", "ws_stack_10x100",
                                  "er_stack_10x10", "er_stack_4x10_c2"])
def test_decompositions(name):
    doc = instance_doc(name)
    g, _, _ = hs.load_instance(doc)
    comms = [set(m) for m in doc["decomposition"]["modules"]]
    assert hs.modularity(g, comms) == _nx(g, comms)
    assert hs.modularity(g, comms, 0.5) == _nx(g, comms, 0.5)


@pytest.mark.parametrize("name", ["ws200", "rn50f", "tf96"])
def test_random_partitions(name):
    g, _, _ = hs.load_instance(instance_doc(name))
    ids = list(g.tasks)
    rng = np.random.default_rng(0)
    P, C = 64, 7
    labels = rng.integers(C, size=(P, len(ids))).astype(np.int32)
    got = hs.modularity_batch(g, labels, n_comm=C)
    for p in range(0, P, 9):
        comms = [{ids[k] for k in range(len(ids)) if labels[p, k] == c}
                 for c in range(C)]
        assert got[p] == _nx(g, comms)
    with pytest.raises(hs.GraphError):
        hs.modularity(g, [set(ids[:3])])
