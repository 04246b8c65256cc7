"""The graph-specialised evaluator (csrc/jit.cpp, NVRTC for sm_100a) must
give the same bits as the reference on every golden case it serves."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import INSTANCES, case_genes, fhex, instance_doc, random_docs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2308_00127_b200 as hs  # noqa: E402
from paper_2308_00127_b200 import _native as N  # noqa: E402
from paper_2308_00127_b200.plan import get_plan  # noqa: E402
from oracle import hs_oracle as O  # noqa: E402
from oracle.hs_oracle_c import CTables  # noqa: E402

ELIGIBLE = [n for n in INSTANCES if n not in ("ws1000", "ws_stack_10x100")]


def _hexes(ms, st):
    return ["GraphError" if s >= N.ST_MISSING else fhex(v)
            for v, s in zip(ms, st)]


@pytest.mark.parametrize("name", ELIGIBLE)
def test_specialised_golden(name):
    doc = instance_doc(name)
    g, hw, t = hs.load_instance(doc)
    for case in doc["cases"]:
        plan = get_plan(g, hw, t, case["L"], case.get("order"))
        if not plan.jit_eligible():
            continue
        plan.specialize()
        genes = case_genes(case)
        ms, st = hs.fitness_batch(torch.from_numpy(genes).cuda(), g, hw, t,
                                  case["L"], order=case.get("order"),
                                  return_status=True)
        assert _hexes(ms.cpu().numpy(), st.cpu().numpy()) == case["expected"]
        for tr in case.get("traces", []):
            if tr["objective"] in ("inf", "GraphError"):
                continue
            genome = hs.MappingGenome(tuple(int(x) for x in genes[tr["row"]]),
                                      tuple(g._topo))
            s = hs.decode(genome, g, hw, t, case["L"])
            assert [fhex(b.start) for b in s.batches] == \
                [b[4] for b in tr["batches"]]


def test_specialised_random_golden():
    """Every golden mini instance (per-pair bandwidths, missing links, tight
    memory, unsupported L, missing latency entries, out-of-range genes,
    non-BFS orders) through its specialised kernel."""
    served = 0
    for doc in random_docs():
        g, hw, t = hs.load_instance(doc)
        for case in doc["cases"]:
            plan = get_plan(g, hw, t, case["L"], case.get("order"))
            if not plan.jit_eligible():
                continue
            plan.specialize()
            genes = case_genes(case)
            ms, st = hs.fitness_batch(torch.from_numpy(genes).cuda(), g, hw,
                                      t, case["L"], order=case.get("order"),
                                      return_status=True)
            assert _hexes(ms.cpu().numpy(), st.cpu().numpy()) == \
                case["expected"], doc["name"]
            served += 1
        if served >= 150:
            break
    assert served >= 100


def _uniform_variant(doc):
    """The random mini instance with one bandwidth over a full mesh, ample
    memory and every batch size supported: inside the specialised scope."""
    g, hw, t = hs.load_instance(doc)
    devs = [hs.Device(d.id, 1e12, (1, 2, 4)) for d in hw.devices.values()]
    bw = {(a.id, b.id): 3.5 for a in devs for b in devs if a.id != b.id}
    hw2 = hs.HardwareSystem(devs, bw)
    ent = dict(t.entries)
    for i in g.tasks:
        for d in devs:
            for b in (1, 2, 4):
                ent.setdefault((i, d.id, b), 1.25 * b + len(i))
    return g, hw2, hs.LatencyTable(ent)


def test_specialised_random_structures():
    served = 0
    for doc in random_docs()[:120]:
        if doc["name"] in ("empty_graph",) or not doc["graph"]["tasks"]:
            continue
        g, hw, t = _uniform_variant(doc)
        L = doc["L"]
        plan = get_plan(g, hw, t, L)
        if not plan.jit_eligible():
            continue
        genes = np.random.default_rng(served).integers(
            plan.K, size=(3000, plan.V), dtype=np.uint8)
        tb = O.build_tables(O.Instance.from_doc({
            "graph": {"tasks": [{"id": x.id, "wm": x.wm, "im": x.im,
                                 "om": x.om} for x in g.tasks.values()],
                      "edges": [list(e) for e in g.edges]},
            "hardware": {"devices": [{"id": d.id, "memory": d.memory,
                                      "batch_sizes": list(d.batch_sizes)}
                                     for d in hw.devices.values()],
                         "bandwidth": {a: {b: v for (x, b), v in
                                           hw.bandwidth.items() if x == a}
                                       for a in hw.devices}},
            "latency": {i: {u: {str(b): t.entries[(i, u, b)]
                                for (i2, u2, b) in t.entries
                                if i2 == i and u2 == u}
                            for u in hw.devices} for i in g.tasks}}), L)
        want, _ = O.fitness_np(tb, genes)
        plan.specialize()
        got = hs.fitness_batch(torch.from_numpy(genes).cuda(), g, hw, t, L)
        assert np.array_equal(got.cpu().numpy().view(np.uint64),
                              want.view(np.uint64)), doc["name"]
        served += 1
    assert served >= 30


@pytest.mark.parametrize("name", ["ws200", "ws30", "rn50f", "ws_stack_10x20"])
def test_specialised_large_vs_c_oracle(name, oracle_lib):
    doc = instance_doc(name)
    g, hw, t = hs.load_instance(doc)
    plan = get_plan(g, hw, t, 1)
    plan.specialize()
    tb = O.build_tables(O.Instance.from_doc(doc), 1)
    n = 300_000
    genes = np.random.default_rng(21).integers(plan.K, size=(n, plan.V),
                                               dtype=np.uint8)
    genes[:7, 3] = 200  # out-of-range genes -> GraphError status
    want, wst = CTables(tb).fitness(oracle_lib, genes, threads=8)
    pad = np.zeros((n, plan.pref_ld), np.uint8)
    pad[:, :plan.V] = genes
    ms, st = hs.fitness_batch(torch.from_numpy(pad).cuda()[:, :plan.V], g, hw,
                              t, 1, return_status=True)
    st = st.cpu().numpy()
    ms = ms.cpu().numpy()
    assert np.array_equal(st, wst)
    ok = wst == 0
    assert np.array_equal(ms[ok].view(np.uint64), want[ok].view(np.uint64))
    cost, idx = hs.argmin_batch(torch.from_numpy(genes[7:]).cuda(), g, hw, t, 1)
    assert (cost, idx) == O.argmin_first(want[7:])
    # generated candidates through the specialised kernel
    out = torch.empty((4096, plan.V), dtype=torch.uint8, device="cuda")
    gms = torch.empty(4096, dtype=torch.float64, device="cuda")
    plan.eval_gen(N.GEN_RANDOM, 5, 77, 4096, makespan=gms, genes_out=out)
    gg = O.gen_genes(5, 77, 4096, plan.V, plan.K)
    assert np.array_equal(out.cpu().numpy(), gg)
    assert np.array_equal(gms.cpu().numpy(), O.fitness_np(tb, gg)[0])


@pytest.mark.parametrize("name", ["ws1000", "ws_stack_10x100"])
def test_specialised_large_graphs(name, oracle_lib):
    """~1000-task graphs: WS1000 keeps its 478 live end times in the
    global-memory slot tier, the 10x100 stack in shared memory."""
    doc = instance_doc(name)
    g, hw, t = hs.load_instance(doc)
    plan = get_plan(g, hw, t, 1)
    assert plan.jit_eligible()
    plan.specialize()
    for case in doc["cases"]:
        if case["L"] != 1 or case.get("order"):
            continue
        genes = case_genes(case)
        ms, st = hs.fitness_batch(torch.from_numpy(genes).cuda(), g, hw, t, 1,
                                  return_status=True)
        assert _hexes(ms.cpu().numpy(), st.cpu().numpy()) == case["expected"]
    tb = O.build_tables(O.Instance.from_doc(doc), 1)
    n = 40_000
    genes = np.random.default_rng(8).integers(plan.K, size=(n, plan.V),
                                              dtype=np.uint8)
    want, wst = CTables(tb).fitness(oracle_lib, genes, threads=8)
    ms, st = hs.fitness_batch(torch.from_numpy(genes).cuda(), g, hw, t, 1,
                              return_status=True)
    assert np.array_equal(st.cpu().numpy(), wst)
    assert np.array_equal(ms.cpu().numpy().view(np.uint64),
                          want.view(np.uint64))
    cost, idx = hs.argmin_batch(torch.from_numpy(genes).cuda(), g, hw, t, 1)
    assert (cost, idx) == O.argmin_first(want)
