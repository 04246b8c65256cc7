"""GPU parity: the CUDA evaluator through the C ABI against the reference's
golden makespans (bit-exact, hex-compared) and, at larger sizes, against the
pinned CPU oracle."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import (INSTANCES, case_genes, fhex, instance_doc,
                      random_docs)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2308_00127_b200 as hs  # noqa: E402
from paper_2308_00127_b200 import _native as N  # noqa: E402
from paper_2308_00127_b200.plan import get_plan  # noqa: E402
from oracle import hs_oracle as O  # noqa: E402
from oracle.hs_oracle_c import CTables  # noqa: E402


def _hexes(ms, st):
    return ["GraphError" if s >= N.ST_MISSING else fhex(v)
            for v, s in zip(ms, st)]


def _check_case(g, hw, t, case):
    genes = case_genes(case)
    order = case.get("order")
    L = case["L"]
    d = torch.from_numpy(genes).cuda()
    ms, st = hs.fitness_batch(d, g, hw, t, L, order=order, return_status=True)
    assert _hexes(ms.cpu().numpy(), st.cpu().numpy()) == case["expected"]
    hm, hst = hs.fitness_batch(genes, g, hw, t, L, order=order,
                               return_status=True)
    assert _hexes(hm, hst) == case["expected"]
    for tr in case.get("traces", []):
        row = genes[tr["row"]]
        genome = hs.MappingGenome(genes=tuple(int(x) for x in row),
                                  order=tuple(order or g._topo))
        if tr["objective"] == "GraphError":
            with pytest.raises(hs.GraphError):
                hs.decode(genome, g, hw, t, L)
            continue
        s = hs.decode(genome, g, hw, t, L)
        if tr["objective"] == "inf":
            assert s is None
            continue
        assert fhex(s.objective) == tr["objective"]
        got = [[b.task, b.device, b.size, list(b.inputs), fhex(b.start)]
               for b in s.batches]
        assert got == tr["batches"]


@pytest.mark.parametrize("name", INSTANCES)
def test_golden_instances(name):
    doc = instance_doc(name)
    g, hw, t = hs.load_instance(doc)
    for case in doc["cases"]:
        _check_case(g, hw, t, case)


def test_golden_random_instances():
    for doc in random_docs():
        g, hw, t = hs.load_instance(doc)
        for case in doc["cases"]:
            _check_case(g, hw, t, case)


def test_fitness_single_and_errors():
    doc = instance_doc("ws30")
    g, hw, t = hs.load_instance(doc)
    case = doc["cases"][0]
    genes = case_genes(case)
    for r in range(5):
        gm = hs.MappingGenome(tuple(int(x) for x in genes[r]), tuple(g._topo))
        assert fhex(hs.fitness(gm, g, hw, t, 1)) == case["expected"][r]
    bad = hs.MappingGenome(tuple([0] * (len(g.tasks) - 1) + [3]),
                           tuple(g._topo))
    with pytest.raises(hs.GraphError):
        hs.fitness(bad, g, hw, t, 1)
    with pytest.raises(hs.GraphError):
        hs.decode(bad, g, hw, t, 1)


def test_chain_known_answer():
    # test_heuristics.py:24-29: serial chain on d0 = 2 + 3 + 4
    T = hs.TaskNode
    g = hs.DnnGraph([T("a", 0, 0, 2.0), T("b", 0, 0, 2.0), T("c")],
                    [("a", "b"), ("b", "c")])
    hw = hs.HardwareSystem([hs.Device("d0", 1e9, (1,)),
                            hs.Device("d1", 1e9, (1,))],
                           {("d0", "d1"): 1.0, ("d1", "d0"): 1.0})
    t = hs.LatencyTable({(i, u, 1): {"d0": 2.0, "d1": 5.0}[u]
                         + {"a": 0, "b": 1, "c": 2}[i]
                         for i in "abc" for u in ("d0", "d1")})
    s = hs.decode(hs.genome_from_map(g, hw, {i: "d0" for i in "abc"}),
                  g, hw, t, 1)
    assert s.objective == 9.0


@pytest.mark.parametrize("name,n", [("ws200", 200_000), ("ws30", 100_000),
                                    ("tf96", 40_000), ("iv3f", 60_000),
                                    ("ws_stack_10x20", 50_000)])
def test_large_batches_vs_c_oracle(name, n, oracle_lib):
    doc = instance_doc(name)
    g, hw, t = hs.load_instance(doc)
    inst = O.Instance.from_doc(doc)
    tb = O.build_tables(inst, 1)
    K = len(hw.devices)
    genes = np.random.default_rng(11).integers(K, size=(n, len(g.tasks)),
                                               dtype=np.uint8)
    want, wst = CTables(tb).fitness(oracle_lib, genes, threads=8)
    plan = get_plan(g, hw, t, 1)
    # preferred stride (bulk TMA staging), natural stride, odd-offset view
    pad = np.zeros((n, plan.pref_ld), np.uint8)
    pad[:, :plan.V] = genes
    for arr in (torch.from_numpy(pad).cuda()[:, :plan.V],
                torch.from_numpy(genes).cuda()):
        ms, st = hs.fitness_batch(arr, g, hw, t, 1, return_status=True)
        assert np.array_equal(ms.cpu().numpy().view(np.uint64),
                              want.view(np.uint64))
        assert np.array_equal(st.cpu().numpy(), wst)
    buf = torch.zeros(n * plan.V + 1, dtype=torch.uint8, device="cuda")
    buf[1:].copy_(torch.from_numpy(genes.ravel()))
    odd = buf[1:].view(n, plan.V)  # misaligned base: manual staging path
    ms = hs.fitness_batch(odd, g, hw, t, 1)
    assert np.array_equal(ms.cpu().numpy().view(np.uint64),
                          want.view(np.uint64))
    cost, idx = hs.argmin_batch(odd, g, hw, t, 1)
    assert (cost, idx) == O.argmin_first(want)
    hc, hi = hs.argmin_batch(genes, g, hw, t, 1, index_base=5)
    assert (hc, hi) == (want[idx], idx + 5)


def test_batch_edges():
    doc = instance_doc("ws30")
    g, hw, t = hs.load_instance(doc)
    plan = get_plan(g, hw, t, 1)
    empty = torch.zeros((0, plan.V), dtype=torch.uint8, device="cuda")
    assert hs.fitness_batch(empty, g, hw, t, 1).numel() == 0
    assert hs.argmin_batch(empty, g, hw, t, 1) == (float("inf"), -1)
    tb = O.build_tables(O.Instance.from_doc(doc), 1)
    for n in (1, 31, 255, 257, 1000):
        genes = np.random.default_rng(n).integers(3, size=(n, plan.V),
                                                  dtype=np.uint8)
        want, _ = O.fitness_np(tb, genes)
        got = hs.fitness_batch(torch.from_numpy(genes).cuda(), g, hw, t, 1)
        assert np.array_equal(got.cpu().numpy(), want)
    # a stride wider than the staging buffer is compacted first
    wide = np.zeros((300, 4 * plan.V), np.uint8)
    wide[:, :plan.V] = np.random.default_rng(3).integers(3, size=(300, plan.V))
    want, _ = O.fitness_np(tb, wide[:, :plan.V])
    got = hs.fitness_batch(torch.from_numpy(wide).cuda()[:, :plan.V],
                           g, hw, t, 1)
    assert np.array_equal(got.cpu().numpy(), want)


@pytest.mark.parametrize("name", ["ws200", "tf96", "ws30"])
def test_generated_candidates(name):
    doc = instance_doc(name)
    g, hw, t = hs.load_instance(doc)
    plan = get_plan(g, hw, t, 1)
    tb = O.build_tables(O.Instance.from_doc(doc), 1)
    n, first, seed = 5000, 123_456, 99
    out = torch.empty((n, plan.V), dtype=torch.uint8, device="cuda")
    ms = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.empty(n, dtype=torch.uint8, device="cuda")
    best = torch.empty(2, dtype=torch.int64, device="cuda")
    plan.eval_gen(N.GEN_RANDOM, seed, first, n, makespan=ms, status=st,
                  genes_out=out, best=best)
    genes = O.gen_genes(seed, first, n, plan.V, plan.K)
    assert np.array_equal(out.cpu().numpy(), genes)
    want, _ = O.fitness_np(tb, genes)
    assert np.array_equal(ms.cpu().numpy(), want)
    b = best.cpu()
    c, i = float(b[:1].view(torch.float64).item()), int(b[1].item())
    wc, wi = O.argmin_first(want)
    assert (c, i) == (wc, wi + first)
    cost, idx, genome = hs.random_search(g, hw, t, 1, n, seed=seed,
                                         first=first, chunk=1777)
    assert (cost, idx) == (wc, wi + first)
    assert genome.genes == tuple(int(x) for x in genes[wi])


def test_enumeration_with_groups():
    doc = [d for d in random_docs() if d["name"] == "ri_5_L1"][0]
    g, hw, t = hs.load_instance(doc)
    plan = get_plan(g, hw, t, 1)
    V, K = plan.V, plan.K
    # tie positions 0 and 2, pin position 1 to device K-1
    group = np.array([0, -1, 0] + list(range(1, V - 2)), np.int16)
    template = np.zeros(V, np.uint8)
    template[1] = K - 1
    ng = V - 2
    n = K ** ng
    out = torch.empty((n, V), dtype=torch.uint8, device="cuda")
    ms = torch.empty(n, dtype=torch.float64, device="cuda")
    plan.eval_gen(N.GEN_ENUM, 0, 0, n, template=torch.from_numpy(template)
                  .cuda(), group=torch.from_numpy(group).cuda(), n_groups=ng,
                  makespan=ms, genes_out=out)
    genes = out.cpu().numpy()
    assert len({r.tobytes() for r in genes}) == n
    assert (genes[:, 1] == K - 1).all() and (genes[:, 0] == genes[:, 2]).all()
    tb = O.build_tables(O.Instance.from_doc(doc), 1)
    want, _ = O.fitness_np(tb, genes)
    assert np.array_equal(ms.cpu().numpy(), want)


def test_throughput_helper():
    assert list(hs.throughput(np.array([500.0, 0.0, np.inf]), 4)) == \
        [8.0, np.inf, 0.0]


@pytest.mark.parametrize("name", ["ws200", "ws30", "rn50f"])
def test_packed_genomes(name, oracle_lib):
    doc = instance_doc(name)
    g, hw, t = hs.load_instance(doc)
    tb = O.build_tables(O.Instance.from_doc(doc), 1)
    plan = get_plan(g, hw, t, 1)
    for n in (1, 33, 5000, 200_000, -1):
        if n < 0:  # once more through the graph-specialised kernel
            plan.specialize()
            n = 100_000
        genes = np.random.default_rng(n).integers(plan.K, size=(n, plan.V),
                                                  dtype=np.uint8)
        genes[0, -1] = 3  # out of range for K = 3 -> GraphError status
        want, wst = CTables(tb).fitness(oracle_lib, genes, threads=8)
        packed = hs.pack_genes(genes)
        # base-3: byte 255 decodes to digits 0,1,1,0,3 (out of range)
        genes3 = genes.copy()
        genes3[0, -1] = 2
        genes3[0, :5] = (0, 1, 1, 0, 3)
        want3, wst3 = CTables(tb).fitness(oracle_lib, genes3, threads=8)
        g3 = genes3.copy()
        g3[0, 4] = 0
        packed3 = hs.pack_genes3(g3)
        packed3[0, 0] = 255
        for radix, pk, w, ws in ((4, packed, want, wst),
                                 (3, packed3, want3, wst3)):
            for arg in (pk, torch.from_numpy(pk).cuda()):
                ms, st = hs.fitness_batch_packed(arg, g, hw, t, 1,
                                                 return_status=True,
                                                 radix=radix)
                ms = ms.cpu().numpy() if hasattr(ms, "cpu") else ms
                st = st.cpu().numpy() if hasattr(st, "cpu") else st
                assert np.array_equal(st, ws)
                ok = ws == 0
                assert np.array_equal(ms[ok].view(np.uint64),
                                      w[ok].view(np.uint64))
