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


def _pack2_ref(genes, pld):
    n, V = genes.shape
    g = np.zeros((n, pld * 4), np.uint8)
    g[:, :V] = genes
    g = g.reshape(n, pld, 4)
    return (g[:, :, 0] | (g[:, :, 1] << 2) | (g[:, :, 2] << 4)
            | (g[:, :, 3] << 6)).astype(np.uint8)


def test_host_packer_matches_numpy():
    """hs_pack_genes2 (the AVX2 thread-pool packer inside hs_eval_host)
    equals a numpy restatement of the 2-bit layout on ragged widths, row
    strides past V and row counts that split unevenly over the pool; an
    out-of-range gene anywhere (incl. the last row's tail) is reported."""
    import ctypes as C
    lib = _native.load()
    rng = np.random.default_rng(5)
    for V in (1, 3, 5, 17, 31, 32, 33, 63, 64, 202, 1002):
        for n in (1, 2, 7, 64, 1000, 4099):
            for extra in (0, 3, 29):
                ld = V + extra
                K = int(rng.integers(1, 5))
                buf = rng.integers(0, K, size=n * ld, dtype=np.uint8)
                # the buffer ends at the last gene byte (no slack after it)
                buf = buf[:(n - 1) * ld + V].copy()
                pld = ((V + 3) // 4 + 3) // 4 * 4
                out = np.full((n, pld), 0xAA, np.uint8)
                ok = C.c_int32(-1)
                assert lib.hs_pack_genes2(buf.ctypes.data, n, ld, V, K,
                                          out.ctypes.data, pld, C.byref(ok)) == 0
                rows = np.lib.stride_tricks.as_strided(buf, (n, V), (ld, 1))
                assert ok.value == 1
                assert np.array_equal(out, _pack2_ref(rows, pld)), (V, n, extra)
                if K < 4:
                    for r, c in ((n - 1, V - 1), (0, 0), (n // 2, V // 2)):
                        bad = buf.copy()
                        bad[r * ld + c] = K
                        assert lib.hs_pack_genes2(bad.ctypes.data, n, ld, V, K,
                                                  out.ctypes.data, pld,
                                                  C.byref(ok)) == 0
                        assert ok.value == 0, (V, n, extra, r, c)
    assert lib.hs_pack_genes2(None, 1, 4, 4, 5, None, 4, None) != 0


def test_host_packer_back_to_back_jobs():
    """Many small packing jobs issued back to back (the pool's workers wake
    late for finished jobs while the next one is published) and from two
    Python threads at once: every result equals the numpy packing."""
    import threading
    rng = np.random.default_rng(9)
    cases = [rng.integers(0, 4, size=(int(rng.integers(1, 300)),
                                      int(rng.integers(1, 90))), dtype=np.uint8)
             for _ in range(60)]
    want = [_pack2_ref(g, ((g.shape[1] + 3) // 4 + 3) // 4 * 4) for g in cases]
    errors = []

    def worker(rounds):
        for _ in range(rounds):
            for g, w in zip(cases, want):
                if not np.array_equal(hs.pack_genes(g), w):
                    errors.append(g.shape)
    ts = [threading.Thread(target=worker, args=(15,)) for _ in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors[:5]
    with pytest.raises(hs.GraphError):
        hs.pack_genes(np.full((2, 9), 4, np.uint8))
    with pytest.raises(hs.GraphError):
        hs.pack_genes(np.full((2, 9), 256, np.int64))


def test_native_greedy_equals_host_greedy():
    """hs_plan_greedy (SA's start, greedy()) equals the host restatement of
    greedy (heuristics.py:192-210) -- mapping, every start and the
    objective, bit for bit -- on every golden instance (L = 1, and 2 / 4 on
    the CNNs), the random fixtures (missing links, tight memory, L > 1) and
    the reference's recorded greedy runs; cases it leaves to the host
    (HS_EHOST) raise the same exception through greedy()."""
    import json as _json
    from paper_2308_00127_b200.heuristics import (_greedy_host,
                                                  _greedy_native)
    cases = [(instance_doc(n), 1) for n in INSTANCES]
    cases += [(instance_doc(n), L) for n in ("rn50f", "iv3f") for L in (2, 4)]
    cases += [(d, d.get("L", 1)) for d in random_docs()]
    native = host_only = 0
    for doc, L in cases:
        g, hw, t = hs.load_instance(doc)
        try:
            want = _greedy_host(g, hw, t, L)
        except Exception as exc:  # noqa: BLE001
            with pytest.raises(type(exc)):
                hs.greedy(g, hw, t, L)
            host_only += 1
            continue
        r = _greedy_native(g, hw, t, L)
        if r is None:
            host_only += 1
        else:
            native += 1
        got = hs.greedy(g, hw, t, L)
        assert got == want
        assert [b.start for b in got.batches] == [b.start for b in want.batches]
    assert native >= len(INSTANCES)
    path = os.path.join(ROOT, "tests", "golden", "heuristics.json")
    with open(path) as f:
        entries = _json.load(f)
    for e in entries:
        res = e["greedy"]
        g, hw, t = hs.load_instance(e)
        if "error" in res:
            with pytest.raises(hs.ScheduleError):
                hs.greedy(g, hw, t, e["L"])
            continue
        s = hs.greedy(g, hw, t, e["L"])
        assert s.objective.hex() == res["objective"] or \
            float.fromhex(res["objective"]) == s.objective
        assert {b.task: b.device for b in s.batches} == res["mapping"]
