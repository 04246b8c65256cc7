"""Heuristic drivers on the GPU evaluator against the reference's recorded
results (tests/golden/heuristics.json): best-device, MET, greedy, and the
exact SA / (1+1) EA trajectories at fixed seeds."""
from __future__ import annotations

import pytest

from conftest import fhex, golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2308_00127_b200 as hs  # noqa: E402


def _entries():
    return golden("heuristics")


def _cmp(res, s):
    if "error" in res:
        return False
    return fhex(s.objective) == res["objective"] and \
        {b.task: b.device for b in s.batches} == res["mapping"]


@pytest.mark.parametrize("idx", range(14))
def test_baselines(idx):
    e = _entries()[idx]
    g, hw, t = hs.load_instance(e)
    L = e["L"]
    for fn, label in ((hs.best_device, "best_device"), (hs.met, "met"),
                      (hs.greedy, "greedy")):
        res = e[label]
        if "error" in res:
            with pytest.raises(hs.ScheduleError):
                fn(g, hw, t, L)
        else:
            assert _cmp(res, fn(g, hw, t, L)), (label, e["name"])


@pytest.mark.parametrize("idx", range(14))
def test_search_trajectories(idx):
    e = _entries()[idx]
    g, hw, t = hs.load_instance(e)
    L = e["L"]
    for run in e["search"]:
        kw = dict(seed=run["seed"], budget=run["budget"])
        if run["algo"] == "sa":
            call = lambda: hs.simulated_annealing(g, hw, t, L, **kw)  # noqa
        else:
            call = lambda: hs.one_plus_one_ea(  # noqa
                g, hw, t, L, biased=(run["algo"] == "ea"), **kw)
        if "error" in run:
            with pytest.raises(hs.ScheduleError):
                call()
        else:
            assert _cmp(run, call()), (e["name"], run["algo"], run["seed"],
                                       run["budget"])


def test_sa_window_sizes_agree():
    e = [x for x in _entries() if x["name"] == "ws30"][0]
    g, hw, t = hs.load_instance(e)
    a = hs.simulated_annealing(g, hw, t, 1, seed=4, budget=400, window=1,
                               device_chain=False)
    b = hs.simulated_annealing(g, hw, t, 1, seed=4, budget=400, window=128,
                               device_chain=False)
    b2 = hs.simulated_annealing(g, hw, t, 1, seed=4, budget=400)
    assert a == b == b2
    c = hs.one_plus_one_ea(g, hw, t, 1, seed=4, budget=300, window=1,
                           device_chain=False)
    d = hs.one_plus_one_ea(g, hw, t, 1, seed=4, budget=300, window=97,
                           device_chain=False)
    e2 = hs.one_plus_one_ea(g, hw, t, 1, seed=4, budget=300)
    assert c == d == e2


@pytest.mark.parametrize("name", ["ws_stack_10x20", "rn50f", "tf96", "ws1000"])
def test_ea_device_chain_matches_windows(name):
    """K9 (whole accept chain in one launch) == windowed GPU batches on
    larger graphs and budgets, biased and unbiased starts."""
    from conftest import instance_doc
    g, hw, t = hs.load_instance(instance_doc(name))
    for biased in (True, False):
        for seed in (0, 3):
            a = hs.one_plus_one_ea(g, hw, t, 1, seed=seed, budget=1500,
                                   biased=biased, device_chain=False)
            b = hs.one_plus_one_ea(g, hw, t, 1, seed=seed, budget=1500,
                                   biased=biased)
            assert a == b, (name, biased, seed)
    # again through the graph-specialised module's search kernel
    if len(g.tasks) <= 512 and hs.specialize(g, hw, t, 1) >= 0:
        c = hs.one_plus_one_ea(g, hw, t, 1, seed=3, budget=1500, biased=False)
        d = hs.one_plus_one_ea(g, hw, t, 1, seed=3, budget=1500, biased=False,
                               device_chain=False)
        assert c == d, name


@pytest.mark.parametrize("name", ["ws_stack_10x20", "rn50f", "tf96", "ws1000"])
def test_sa_device_chain_matches_windows(name):
    """K10 (speculative SA with PCG64 on the device, one launch) == the
    host-replayed windows."""
    from conftest import instance_doc
    g, hw, t = hs.load_instance(instance_doc(name))
    budget = 600 if name == "ws1000" else 1500
    for seed in (0, 3):
        a = hs.simulated_annealing(g, hw, t, 1, seed=seed, budget=budget,
                                   device_chain=False)
        b = hs.simulated_annealing(g, hw, t, 1, seed=seed, budget=budget)
        assert a == b, (name, seed)
    # again through the graph-specialised module's search kernel
    if len(g.tasks) <= 512 and hs.specialize(g, hw, t, 1) >= 0:
        c = hs.simulated_annealing(g, hw, t, 1, seed=3, budget=budget)
        assert c == a, name


def test_sa_host_exp_path(monkeypatch):
    """Every Metropolis test handed back to the host (the rare too-close-
    to-call path of K10) still gives the reference trajectory."""
    from conftest import instance_doc
    g, hw, t = hs.load_instance(instance_doc("ws30"))
    a = hs.simulated_annealing(g, hw, t, 1, seed=2, budget=300,
                               device_chain=False)
    monkeypatch.setenv("HS_SA_HOST_EXP", "1")
    b = hs.simulated_annealing(g, hw, t, 1, seed=2, budget=300)
    assert a == b


def test_search_kernels_genes_in_registers(monkeypatch):
    """The specialised body variant that reads whole words of the genome
    row (HS_JIT_OPTS=genes=reg) gives the same SA / EA trajectories."""
    from conftest import instance_doc
    monkeypatch.setenv("HS_JIT_OPTS", "genes=reg")
    g, hw, t = hs.load_instance(instance_doc("ws30"))  # fresh plan objects
    hs.specialize(g, hw, t, 1)
    for seed in (1, 5):
        assert hs.simulated_annealing(g, hw, t, 1, seed=seed, budget=500) == \
            hs.simulated_annealing(g, hw, t, 1, seed=seed, budget=500,
                                   device_chain=False)
        assert hs.one_plus_one_ea(g, hw, t, 1, seed=seed, budget=500,
                                  biased=False) == \
            hs.one_plus_one_ea(g, hw, t, 1, seed=seed, budget=500,
                               biased=False, device_chain=False)


def test_ea_single_launch_equals_chunks():
    """hs_ea_run (whole chain, one launch) and hs_ea_run_chunk (chained
    chunks, the default path) end on the same genome and fitness."""
    import numpy as np
    from conftest import instance_doc
    from paper_2308_00127_b200 import heuristics as H
    g, hw, t = hs.load_instance(instance_doc("ws_stack_10x20"))
    plan = H.get_plan(g, hw, t, 1)
    V, K = plan.V, plan.K
    genes0 = np.random.default_rng(9).integers(K, size=V, dtype=np.uint8)
    f0 = float(hs.fitness_batch(genes0[None, :], g, hw, t, 1)[0])
    budget = 900
    moff, mpos, mval = H._ea_draw_chunk(np.random.default_rng(3), budget, V,
                                        K, 1.0 / V)
    parent = torch.from_numpy(genes0.copy()).cuda()
    fit = torch.empty(1, dtype=torch.float64, device="cuda")
    info = torch.empty(4, dtype=torch.int32, device="cuda")
    plan.ea_run(parent, f0, moff.cuda(), mpos.cuda(), mval.cuda(), budget,
                fit, info)
    for chunks in (1, 3, 7):
        g2, f2 = H._ea_device_chain(plan, np.random.default_rng(3), genes0,
                                    f0, budget, V, K, 1.0 / V, chunks=chunks)
        assert np.array_equal(g2, parent.cpu().numpy()), chunks
        assert f2 == float(fit.cpu()[0]), chunks
    assert int(info.cpu()[2]) == -1
