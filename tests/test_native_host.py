"""Host-side checks of the native library without a GPU: the C ABI loads and
exports every symbol the header declares, and the plan compiler (pure host
C++) reproduces the reference's genome order, device numbering and the
instance flags that select kernel paths."""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import INSTANCES, ROOT, instance_doc, random_docs

import paper_2308_00127_b200 as hs
from paper_2308_00127_b200 import _native
from paper_2308_00127_b200.plan import Plan


def test_header_symbols_exported():
    lib = _native.load()
    with open(os.path.join(ROOT, "include", "hetsched_b200.h")) as f:
        text = f.read()
    declared = set(re.findall(r"\b(hs_[a-z_0-9]+)\s*\(", text))
    assert declared == set(_native.exported_symbols())
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.hs_abi_version() == 1


def test_best_merge_host():
    lib = _native.load()
    arr = (_native.Best * 4)((3.0, 9), (1.0, 7), (1.0, 4), (float("inf"), 0))
    out = _native.Best()
    assert lib.hs_best_merge(arr, 4, C.byref(out)) == 0
    assert (out.cost, out.index) == (1.0, 4)
    empty = (_native.Best * 1)((float("inf"), -1))
    assert lib.hs_best_merge(empty, 1, C.byref(out)) == 0
    assert out.index == -1


@pytest.mark.parametrize("name", INSTANCES)
def test_plan_order_matches_reference(name):
    doc = instance_doc(name)
    g, hw, t = hs.load_instance(doc)
    p = Plan(g, hw, t, 1)
    assert list(p.order) == doc["order"]
    assert list(p.devices) == doc["devices_sorted"]
    assert p.info.V == len(g.tasks) and p.info.E == len(g.edges)
    assert p.pref_ld >= p.V and (p.pref_ld // 4) % 2 == 1


def test_plan_random_instances_flags():
    seen = set()
    for doc in random_docs():
        g, hw, t = hs.load_instance(doc)
        p = Plan(g, hw, t, doc["L"])
        assert list(p.order) == doc["order"]
        i = p.info
        seen.add((i.uniform_comm, i.full_mesh, i.mem_check, i.all_batch_ok,
                  i.latency_complete))
    # every kernel feature path is exercised by the fixtures
    assert {s[0] for s in seen} == {0, 1}
    assert {s[1] for s in seen} == {0, 1}
    assert {s[2] for s in seen} == {0, 1}
    assert {s[3] for s in seen} == {0, 1}
    assert {s[4] for s in seen} == {0, 1}


def test_plan_errors():
    T = hs.TaskNode
    g = hs.DnnGraph([T("a"), T("b")], [("a", "b")])
    hw = hs.HardwareSystem([hs.Device("d", 1.0, (1,))], {})
    t = hs.LatencyTable({})
    with pytest.raises(hs.GraphError):
        Plan(g, hw, t, 1, order=("b", "a"))  # not topological
    with pytest.raises(hs.GraphError):
        Plan(g, hw, t, 1, order=("a",))
    Plan(g, hw, t, 1, order=("a", "b"))
    with pytest.raises(hs.GraphError, match="cycle"):
        hs.DnnGraph([T("a"), T("b")], [("a", "b"), ("b", "a")])


def test_live_slots_are_small_for_stacks():
    p = Plan(*hs.load_instance(instance_doc("tf96")), 1)
    assert p.info.live_slots == 2 and p.info.n_classes == 2
    p = Plan(*hs.load_instance(instance_doc("ws200")), 1)
    assert p.info.live_slots == 101 and p.info.uniform_comm == 1


def test_batched_options_match_reference_enumeration():
    from conftest import golden
    from oracle import hs_batched as B
    from oracle import hs_oracle as O
    for e in golden("batched"):
        g, hw, t = hs.load_instance(e)
        inst = O.Instance.from_doc(e)
        want = [(s, tuple(sorted(inst.dev_ids)[k] for k in dv))
                for s, dv in B.options(inst, e["L"])]
        assert hs.batched_options(g, hw, t, e["L"]) == want


def test_pack_genes_layouts():
    """2-bit and base-3 packings decode back to the genes (the kernels'
    expansion restated in numpy)."""
    rng = np.random.default_rng(7)
    for V in (1, 5, 32, 202, 1002):
        genes = rng.integers(3, size=(17, V), dtype=np.uint8)
        p3 = hs.pack_genes3(genes)
        assert p3.shape == (17, (V + 4) // 5)
        b = p3.astype(np.int64)
        digits = np.stack([(b // 3 ** d) % 3 for d in range(5)], axis=2)
        assert np.array_equal(digits.reshape(17, -1)[:, :V], genes)
        p2 = hs.pack_genes(genes)
        assert p2.shape[1] % 4 == 0 and p2.shape[1] * 4 >= V
        d2 = np.stack([(p2 >> (2 * j)) & 3 for j in range(4)], axis=2)
        assert np.array_equal(d2.reshape(17, -1)[:, :V], genes)
    with pytest.raises(hs.GraphError):
        hs.pack_genes3(np.full((1, 4), 3, np.uint8))


def test_host_pack_policy(monkeypatch):
    """hs_eval_host packs on the host by default when K <= 4 and the host
    has >= 8 threads; HS_HOST_PACK=0 / 1 override; small batches and K > 4
    never pack (hs_eval_host_packs reports the decision, host-only)."""
    g, hw, t = hs.load_instance(instance_doc("ws200"))
    plan = Plan(g, hw, t, 1)
    n = 1 << 20
    monkeypatch.delenv("HS_HOST_PACK", raising=False)
    assert plan.eval_host_packs(n) == ((os.cpu_count() or 1) >= 8)
    assert not plan.eval_host_packs(1000)
    monkeypatch.setenv("HS_HOST_PACK", "0")
    assert not plan.eval_host_packs(n)
    monkeypatch.setenv("HS_HOST_PACK", "1")
    assert plan.eval_host_packs(n)
    g, hw, t = hs.load_instance(instance_doc("tf96"))
    assert not Plan(g, hw, t, 1).eval_host_packs(n)  # K = 30
