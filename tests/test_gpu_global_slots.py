"""The global-memory end-time slot tier (csrc/capi.cu get_dev_state,
csrc/jit.cpp jit_build) on synthetic 600-task instances whose live end
times overflow shared memory, with every check the list scheduler has
(heuristics.py:92-106): per-pair bandwidths with a missing link, a device
without the batch size, tight memory, and genes out of range; K = 3 (device
state in registers) and K = 5 (generic K). Both evaluators -- the
plan-walking kernel and the specialised one -- must return the C oracle's
bits (oracle/hs_oracle.c, pinned to the reference)."""
from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2308_00127_b200 as hs  # noqa: E402
from paper_2308_00127_b200.plan import Plan  # noqa: E402
from oracle import hs_oracle as O  # noqa: E402
from oracle.hs_oracle_c import CTables  # noqa: E402


def _instance(V: int, K: int, seed: int) -> dict:
    rng = np.random.default_rng(seed)
    ids = [f"t{i:04d}" for i in range(V)]
    tasks = [{"id": t, "wm": float(rng.integers(0, 50)),
              "im": float(rng.integers(0, 20)),
              "om": float(rng.integers(0, 30))} for t in ids]
    edges = []
    for i in range(1, V):
        # one near and up to two far predecessors: hundreds of end times
        # stay live at once (the BFS order follows the ids here)
        srcs = {i - 1} | set(int(x) for x in
                             rng.integers(max(0, i - 700), i, size=2))
        edges += [[ids[j], ids[i]] for j in sorted(srcs)]
    devs = [f"d{k}" for k in range(K)]
    total = sum((t["im"] + t["om"]) + t["wm"] for t in tasks)
    hw_devs = []
    for k, u in enumerate(devs):
        mem = 0.55 * total if k == 0 else 1e12       # d0 can run out
        bs = [2] if k == K - 1 else [1, 2]           # last device lacks L=1
        hw_devs.append({"id": u, "memory": mem, "batch_sizes": bs})
    bw = {u: {v: float(rng.uniform(0.5, 4.0)) for v in devs if v != u}
          for u in devs}
    del bw["d1"]["d2"]                                # missing link d1 -> d2
    lat = {t: {u: {"1": float(rng.uniform(1, 10)),
                   "2": float(rng.uniform(2, 20))} for u in devs}
           for t in ids}
    return {"graph": {"tasks": tasks, "edges": edges},
            "hardware": {"devices": hw_devs, "bandwidth": bw},
            "latency": lat}


def _genes(plan, n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    K, V = plan.K, plan.V
    g = rng.integers(K, size=(n, V), dtype=np.uint8)
    # most rows avoid the failure modes so that makespans are compared too:
    # devices {0, 1} plus d3.. (no d1 -> d2 link, no L-less last device)
    safe = [k for k in range(K - 1) if k != 2]
    u = rng.random(n)
    rows = u < 0.65
    g[rows] = rng.choice(np.array(safe, np.uint8), size=(rows.sum(), V))
    heavy = (u >= 0.65) & (u < 0.7)  # ~75 % of the memory on d0
    g[heavy] = rng.choice(np.array([0, 0, 0, 1], np.uint8),
                          size=(heavy.sum(), V))
    g[:5, 7] = 250  # gene out of range -> GraphError status
    return g


@pytest.mark.parametrize("K,seed", [(3, 1), (5, 2)])
def test_global_slots_vs_c_oracle(K, seed, oracle_lib):
    doc = _instance(600, K, seed)
    g, hw, t = hs.load_instance(doc)
    tb = O.build_tables(O.Instance.from_doc(doc), 1)
    ct = CTables(tb)
    plan = Plan(g, hw, t, 1)
    genes = _genes(plan, 30_000, seed)
    want, wst = ct.fitness(oracle_lib, genes, threads=8)
    assert (wst == 0).sum() > 1000 and (wst == 2).sum() > 0  # both regimes
    d = torch.from_numpy(genes).cuda()
    for specialised in (False, True):
        if specialised:
            assert plan.jit_eligible()
            plan.specialize()
        ms = torch.empty(len(genes), dtype=torch.float64, device="cuda")
        st = torch.empty(len(genes), dtype=torch.uint8, device="cuda")
        best = torch.empty(2, dtype=torch.int64, device="cuda")
        plan.eval(d, ms, st, best)
        st = st.cpu().numpy()
        ms = ms.cpu().numpy()
        assert np.array_equal(st, wst), specialised
        ok = wst < 4
        assert np.array_equal(ms[ok].view(np.uint64), want[ok].view(np.uint64))
        b = best.cpu()
        key = np.where(wst >= 4, np.inf, want)
        assert (float(b[:1].view(torch.float64).item()), int(b[1].item())) == \
            O.argmin_first(key)
