"""Multi-start search on the GPU: `simulated_annealing_multi` runs one K10
chain per seed, one CTA (SM) each, in a single launch. Every chain must be
exactly the reference's simulated_annealing for its seed: the golden
north-star-scale runs (tests/golden/search_big.json, seeds 0-2, budget 2000)
and, for 148 seeds at once (one per SM), sampled chains against this
package's single-chain runs (themselves pinned to the reference)."""
from __future__ import annotations

import time

import pytest

from conftest import fhex, golden, instance_doc

import paper_2308_00127_b200 as hs

pytestmark = pytest.mark.gpu


def _mapping(s):
    return {b.task: b.device for b in s.batches}


@pytest.mark.parametrize("name", ["ws_stack_10x20", "ws200", "tf96"])
def test_sa_multi_equals_reference_seeds(name):
    g, hw, t = hs.load_instance(instance_doc(name))
    runs = [e for e in golden("search_big")
            if e["instance"] == name and e["algo"] == "sa"]
    got = hs.simulated_annealing_multi(g, hw, t, 1,
                                       [e["seed"] for e in runs], budget=2000)
    for e, s in zip(runs, got):
        assert fhex(s.objective) == e["objective"], e["seed"]
        assert _mapping(s) == e["mapping"]


def test_sa_multi_148_chains():
    g, hw, t = hs.load_instance(instance_doc("ws_stack_10x20"))
    hs.specialize(g, hw, t, 1)
    seeds = list(range(148))
    hs.simulated_annealing_multi(g, hw, t, 1, seeds[:2], budget=100)  # warm
    t0 = time.perf_counter()
    got = hs.simulated_annealing_multi(g, hw, t, 1, seeds, budget=2000)
    multi_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    one = hs.simulated_annealing(g, hw, t, 1, seed=0, budget=2000)
    one_s = time.perf_counter() - t0
    print(f"148 chains {multi_s * 1e3:.1f} ms, one chain {one_s * 1e3:.1f} ms")
    assert len(got) == 148
    assert fhex(got[0].objective) == fhex(one.objective)
    for c in (1, 37, 101, 147):
        s = hs.simulated_annealing(g, hw, t, 1, seed=c, budget=2000)
        assert fhex(got[c].objective) == fhex(s.objective), c
        assert _mapping(got[c]) == _mapping(s)
    best = min(got, key=lambda s: s.objective)
    assert best.objective <= one.objective


def test_sa_multi_aot_body(monkeypatch):
    """The same chains over the ahead-of-time plan walker (K10 AOT)."""
    monkeypatch.setenv("HS_SEARCH_AOT", "1")
    g, hw, t = hs.load_instance(instance_doc("ws30"))
    got = hs.simulated_annealing_multi(g, hw, t, 1, [3, 4, 5, 6], budget=500)
    for c, s in zip((3, 4, 5, 6), got):
        want = hs.simulated_annealing(g, hw, t, 1, seed=c, budget=500)
        assert fhex(s.objective) == fhex(want.objective)
        assert _mapping(s) == _mapping(want)


@pytest.mark.parametrize("name", ["ws_stack_10x20", "ws200", "tf96"])
def test_ea_multi_equals_reference_seeds(name):
    """Device-drawn mutation streams (K12) + one K9 chain per seed."""
    g, hw, t = hs.load_instance(instance_doc(name))
    runs = [e for e in golden("search_big")
            if e["instance"] == name and e["algo"] == "ea"]
    got = hs.one_plus_one_ea_multi(g, hw, t, 1, [e["seed"] for e in runs],
                                   budget=2000)
    for e, s in zip(runs, got):
        assert fhex(s.objective) == e["objective"], e["seed"]
        assert _mapping(s) == e["mapping"]


def test_ea_single_chain_device_draw():
    from paper_2308_00127_b200.heuristics import _last_chain_stats
    g, hw, t = hs.load_instance(instance_doc("ws200"))
    e = next(x for x in golden("search_big")
             if x["instance"] == "ws200" and x["algo"] == "ea")
    s = hs.one_plus_one_ea(g, hw, t, 1, seed=e["seed"], budget=2000)
    assert _last_chain_stats.get("ea_draw") == "device"
    assert fhex(s.objective) == e["objective"]


def test_ea_multi_148_chains_and_unbiased():
    g, hw, t = hs.load_instance(instance_doc("ws_stack_10x20"))
    hs.specialize(g, hw, t, 1)
    seeds = list(range(148))
    hs.one_plus_one_ea_multi(g, hw, t, 1, seeds[:2], budget=100)  # warm
    t0 = time.perf_counter()
    got = hs.one_plus_one_ea_multi(g, hw, t, 1, seeds, budget=2000)
    multi_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    one = hs.one_plus_one_ea(g, hw, t, 1, seed=0, budget=2000)
    one_s = time.perf_counter() - t0
    print(f"EA 148 chains {multi_s * 1e3:.1f} ms, one chain "
          f"{one_s * 1e3:.1f} ms")
    assert fhex(got[0].objective) == fhex(one.objective)
    for c in (1, 66, 147):
        s = hs.one_plus_one_ea(g, hw, t, 1, seed=c, budget=2000)
        assert fhex(got[c].objective) == fhex(s.objective), c
        assert _mapping(got[c]) == _mapping(s)
    ub = hs.one_plus_one_ea_multi(g, hw, t, 1, [7, 8], budget=500,
                                  biased=False)
    for c, s in zip((7, 8), ub):
        want = hs.one_plus_one_ea(g, hw, t, 1, seed=c, budget=500,
                                  biased=False)
        assert fhex(s.objective) == fhex(want.objective)


def test_ea_draw_matches_host_stream():
    """K12's CSR lists equal rng.py's host restatement (itself pinned to
    numpy) for several seeds, graph sizes and device counts."""
    import numpy as np
    from paper_2308_00127_b200 import rng as R
    from paper_2308_00127_b200.heuristics import _ea_draw_device, _gen_words
    for V, n_dev, budget in ((202, 3, 300), (7, 30, 200), (1, 2, 50),
                             (33, 1, 40), (2, 2, 500)):
        seeds = [0, 1, 99]
        states = []
        for s in seeds:
            gen = np.random.default_rng(s)
            if s == 99:
                gen.integers(n_dev, size=3)  # leaves a cached half word
            states.append((gen, _gen_words(gen)))
        moff, mpos, mval, status, _k = _ea_draw_device(
            [w for _, w in states], V, n_dev, 1.0 / V, budget)
        moff, mpos, mval = (x.cpu().numpy() for x in (moff, mpos, mval))
        assert not status.cpu().numpy().any()
        for c, (gen, _w) in enumerate(states):
            S, words, st = R.peek_words(gen, budget * (V + 2) + 64)
            muts = R.ea_mutations(S, words, st, budget, V, n_dev, 1.0 / V)
            for k, (m, _s) in enumerate(muts):
                a, b = moff[c, k], moff[c, k + 1]
                assert [(int(x), int(y)) for x, y in
                        zip(mpos[a:b], mval[a:b])] == m, (V, c, k)


def test_multi_edge_cases():
    """budget 0, one device, empty seed list, a single seed, and the
    reference's small golden instances (tight memory, missing links, L > 1)
    through the multi-chain paths: each element equals the single run."""
    from conftest import golden
    from paper_2308_00127_b200.core import load_graph, load_hardware, \
        load_latency
    import json
    assert hs.simulated_annealing_multi(*hs.load_instance(
        instance_doc("ws30")), 1, []) == []
    for e in golden("heuristics")[:8] + golden("heuristics")[-2:]:
        g = load_graph(json.dumps(e["graph"]))
        hw = load_hardware(json.dumps(e["hardware"]))
        t = load_latency(json.dumps(e["latency"]))
        L = e["L"]
        for budget in (0, 1, 150):
            for multi, single in (
                    (hs.simulated_annealing_multi, hs.simulated_annealing),
                    (hs.one_plus_one_ea_multi, hs.one_plus_one_ea)):
                try:
                    want = [single(g, hw, t, L, seed=s, budget=budget)
                            for s in (0, 1, 2)]
                except hs.ScheduleError:
                    with pytest.raises(hs.ScheduleError):
                        multi(g, hw, t, L, [0, 1, 2], budget=budget)
                    continue
                got = multi(g, hw, t, L, [0, 1, 2], budget=budget)
                assert [fhex(s.objective) for s in got] == \
                    [fhex(s.objective) for s in want], (e["name"], budget)
                assert [_mapping(s) for s in got] == \
                    [_mapping(s) for s in want]
