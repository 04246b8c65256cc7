"""Small invocations of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck), e.g.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

Covers the graph-specialised evaluator on its TMEM slot tier (WS200, one
full persistent grid, mbarrier + TMA bulk tiles), its trace kernel, the SA
(K10) and EA (K9) search kernels over the specialised body, the
ahead-of-time plan walker (K1) with its fused argmin (K2), the batched
variant (K8), the bound kernels (K4 / K5) and the schedule validator (K11).
Results are checked against the CPU oracle so a silent corruption fails.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2308_00127_b200 as hs  # noqa: E402
from oracle import hs_oracle as O  # noqa: E402
from paper_2308_00127_b200.plan import get_plan  # noqa: E402


def doc(name):
    with open(f"tests/golden/instances/{name}.json") as f:
        return json.load(f)


def check(name, n, jit):
    d = doc(name)
    g, hw, t = hs.load_instance(d)
    plan = get_plan(g, hw, t, 1)
    if jit:
        plan.specialize()
    genes = np.random.default_rng(7).integers(plan.K, size=(n, plan.V),
                                              dtype=np.uint8)
    ms = hs.fitness_batch(torch.from_numpy(genes).cuda(), g, hw, t, 1)
    want, _ = O.fitness_np(O.build_tables(O.Instance.from_doc(d), 1), genes)
    ok = np.array_equal(ms.cpu().numpy().view(np.uint64), want.view(np.uint64))
    print(f"{name} jit={jit} n={n}: {'ok' if ok else 'MISMATCH'}")
    assert ok
    return g, hw, t


which = sys.argv[1:] or ["jit", "trace", "search", "aot", "batched", "batched_jit",
                         "gen", "bounds", "validate"]
if "jit" in which:
    check("ws200", 148 * 384 + 1000, True)
if "trace" in which:
    g, hw, t = hs.load_instance(doc("ws200"))
    hs.specialize(g, hw, t, 1)
    order = tuple(doc("ws200")["order"])
    s = hs.decode(hs.MappingGenome(genes=(0,) * len(order), order=order), g,
                  hw, t, 1)
    print("trace ok", s.objective)
if "search" in which:
    for name in ("ws30", "ws200"):
        g, hw, t = hs.load_instance(doc(name))
        hs.specialize(g, hw, t, 1)
        a = hs.simulated_annealing(g, hw, t, 1, seed=0, budget=300)
        b = hs.one_plus_one_ea(g, hw, t, 1, seed=0, budget=300)
        print("search", name, a.objective, b.objective)
if "sa_only" in which:
    # hs_jit_sa in a process where no kernel with an mbarrier ran before
    # (start fitness from the CPU oracle instead of a GPU evaluation)
    from paper_2308_00127_b200.heuristics import _sa_device_chain
    d = doc("ws30")
    g, hw, t = hs.load_instance(d)
    plan = get_plan(g, hw, t, 1)
    plan.specialize()
    genes = np.zeros(plan.V, np.uint8)
    f0, _ = O.fitness_np(O.build_tables(O.Instance.from_doc(d), 1),
                         genes[None, :])
    best, bf = _sa_device_chain(plan, np.random.default_rng(0), genes,
                                float(f0[0]), float(f0[0]), 0.1 * float(f0[0]),
                                0.995, 300, plan.K, 128)
    print("sa_only", bf)
if "aot" in which:
    check("ws30", 20000, False)
    check("tf96", 5000, False)
if "batched" in which:
    g, hw, t = hs.load_instance(doc("ws30"))
    opts = hs.batched_options(g, hw, t, 4)
    genes = np.random.default_rng(1).integers(len(opts), size=(3000, 32),
                                              dtype=np.uint8)
    ms = hs.fitness_batched(torch.from_numpy(genes).cuda(), g, hw, t, 4)
    print("batched ok", float(ms.min()))
if "batched_jit" in which:
    # specialised K8 on its global-memory slot tier (WS200, L = 4) against
    # the plan walker
    from paper_2308_00127_b200.plan import Plan
    g, hw, t = hs.load_instance(doc("ws200"))
    nopt = len(hs.batched_options(g, hw, t, 4))
    jit, aot = Plan(g, hw, t, 4, batched=()), Plan(g, hw, t, 4, batched=())
    jit.specialize()
    n = 2 * 148 * 192 + 77
    genes = torch.randint(0, nopt, (n, jit.pref_ld), dtype=torch.uint8, device="cuda")
    m1 = torch.empty(n, dtype=torch.float64, device="cuda")
    m2 = torch.empty_like(m1)
    jit.eval(genes, m1)
    aot.eval(genes, m2)
    assert torch.equal(m1.view(torch.int64), m2.view(torch.int64))
    print("batched_jit ok", float(m1.min()))
if "gen" in which:
    # hash-random generated rows (no gene check pass) through the
    # specialised evaluator, re-derived and re-scored by the oracle
    from paper_2308_00127_b200 import _native as N
    d = doc("ws200")
    g, hw, t = hs.load_instance(d)
    plan = get_plan(g, hw, t, 1)
    plan.specialize()
    n = 148 * 384 + 1000
    ms = torch.empty(n, dtype=torch.float64, device="cuda")
    out = torch.empty((n, plan.V), dtype=torch.uint8, device="cuda")
    plan.eval_gen(N.GEN_RANDOM, 11, 5, n, makespan=ms, genes_out=out)
    want_g = O.gen_genes(11, 5, n, plan.V, plan.K)
    assert np.array_equal(out.cpu().numpy(), want_g)
    want, _ = O.fitness_np(O.build_tables(O.Instance.from_doc(d), 1), want_g[:4000])
    assert np.array_equal(ms.cpu().numpy()[:4000].view(np.uint64), want.view(np.uint64))
    print("gen ok")
if "bounds" in which:
    g, hw, t = hs.load_instance(doc("ws_stack_10x20"))
    d = hs.k_edge_components(g, 1)
    lb = hs.lower_bound(g, hw, t, 1, d, subgraph_cap=0)
    print("bounds ok", lb.lower_bound_ms)
if "validate" in which:
    g, hw, t = hs.load_instance(doc("ws30"))
    s = hs.greedy(g, hw, t, 1)
    print("validate ok", hs.validate_schedule(g, hw, t, s))
torch.cuda.synchronize()
print("sanitize run done")
