"""The GPU ModuleSolver honours the reference's plug-in contract
(splitting.py:225-245): pins and same-device pairs respected, returned
objective equal to the oracle makespan of the returned mapping, exhaustive
sweeps optimal over decoder mappings, (None, None, False) when infeasible."""
from __future__ import annotations

import itertools

import numpy as np
import pytest

from conftest import instance_doc, random_docs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2308_00127_b200 as hs  # noqa: E402
from oracle import hs_oracle as O  # noqa: E402


def _oracle_fit(doc, s, L):
    inst = O.Instance.from_doc(doc)
    tb = O.build_tables(inst, L)
    genes = [tb.devs.index({b.task: b.device for b in s.batches}[t])
             for t in tb.order]
    return O.fitness_one(tb, genes)[0], tb


def test_exhaustive_is_decoder_optimal():
    solver = hs.gpu_module_solver()
    for doc in random_docs()[:40]:
        g, hw, t = hs.load_instance(doc)
        L = doc["L"]
        obj, s, opt = solver(g, hw, t, L, {}, [], None)
        inst = O.Instance.from_doc(doc)
        tb = O.build_tables(inst, L)
        allg = np.array(list(itertools.product(range(tb.K), repeat=tb.V)),
                        np.uint8).reshape(-1, tb.V)
        best = float(O.fitness_np(tb, allg)[0].min()) if tb.V else 0.0
        if not np.isfinite(best):
            assert obj is None and s is None and opt is False
            continue
        assert obj == best and opt is False
        assert _oracle_fit(doc, s, L)[0] == obj


def test_pins_and_same_device():
    solver = hs.gpu_module_solver()
    doc = instance_doc("er_stack_10x10")
    g, hw, t = hs.load_instance(doc)
    ids = list(g.tasks)
    sub = g.subgraph(ids[:12])
    pins = {ids[0]: "cpu", ids[5]: "gpuB"}
    same = [(ids[1], ids[2]), (ids[2], ids[7])]
    obj, s, _ = solver(sub, hw, t, 1, pins, same, None)
    dev = {b.task: b.device for b in s.batches}
    assert dev[ids[0]] == "cpu" and dev[ids[5]] == "gpuB"
    assert dev[ids[1]] == dev[ids[2]] == dev[ids[7]]
    assert s.objective == obj
    # clashing pins inside one tied group are infeasible
    assert solver(sub, hw, t, 1, {ids[1]: "cpu", ids[2]: "gpuA"}, same,
                  None) == (None, None, False)


def test_sampled_module_sweep_is_consistent():
    solver = hs.gpu_module_solver(exhaustive_limit=1000, samples=1 << 16)
    doc = instance_doc("ws_stack_10x20")
    g, hw, t = hs.load_instance(doc)
    mod = sorted(doc["decomposition"]["modules"][3])
    sub = g.subgraph(mod)
    obj, s, opt = solver(sub, hw, t, 1, {}, [], 5.0)
    assert opt is False and np.isfinite(obj)
    sdoc = {"graph": {"tasks": [{"id": x.id, "wm": x.wm, "im": x.im,
                                 "om": x.om} for x in sub.tasks.values()],
                      "edges": [list(e) for e in sub.edges]},
            "hardware": doc["hardware"], "latency": doc["latency"]}
    assert _oracle_fit(sdoc, s, 1)[0] == obj
    # never worse than MET on the same module
    assert obj <= hs.met(sub, hw, t, 1).objective


def test_neighbor_generation_matches_host():
    """HS_GEN_NEIGHBOR: every one- and two-group move of an incumbent,
    generated on the device, equals the host construction, and its
    makespan the evaluation of that row."""
    import numpy as np
    import torch
    from paper_2308_00127_b200 import _native as N
    from paper_2308_00127_b200.heuristics import _fit_rows
    from paper_2308_00127_b200.plan import get_plan
    g, hw, t = hs.load_instance(instance_doc("ws30"))
    plan = get_plan(g, hw, t, 1)
    V, K = plan.V, plan.K
    rng = np.random.default_rng(4)
    inc = rng.integers(K, size=V, dtype=np.uint8)
    group = np.full(V, -1, np.int16)
    free = [i for i in range(V) if i % 5]  # every fifth position pinned
    for k, i in enumerate(free):
        group[i] = min(k, 7 + k // 3)  # some ties
    # renumber groups by first position (the generator's contract)
    ren, nxt = {}, 0
    for i in range(V):
        if group[i] >= 0:
            if group[i] not in ren:
                ren[group[i]] = nxt
                nxt += 1
            group[i] = ren[group[i]]
    ng = nxt
    M = ng * K + ng * ng * K * K
    out = torch.empty((M, V), dtype=torch.uint8, device="cuda")
    ms = torch.empty(M, dtype=torch.float64, device="cuda")
    plan.eval_gen(N.GEN_NEIGHBOR, 0, 0, M,
                  template=torch.from_numpy(inc).cuda(),
                  group=torch.from_numpy(group).cuda(), n_groups=ng,
                  genes_out=out, makespan=ms)
    want = np.repeat(inc[None, :], M, axis=0)
    for c in range(M):
        if c < ng * K:
            want[c][group == c // K] = c % K
        else:
            p = c - ng * K
            vb, va = p % K, (p // K) % K
            p //= K * K
            l, j = p % ng, p // ng
            want[c][group == j] = va
            if l > j:
                want[c][group == l] = vb
    assert np.array_equal(out.cpu().numpy(), want)
    assert np.array_equal(ms.cpu().numpy().view(np.uint64),
                          _fit_rows(plan, want).view(np.uint64))
