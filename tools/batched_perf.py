"""Device throughput of the batched-variant (extended genome) evaluator
(K8, heuristics.py:337-433 semantics) on the paper's CNN graphs with the
throughput objective, L in {2, 4, 8}: explicit random extended genomes and
on-device generated ones.

    python tools/batched_perf.py rn50f iv3f      (QP_L=4 for one L)
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2308_00127_b200 as hs  # noqa: E402
from paper_2308_00127_b200 import _native as N  # noqa: E402
from paper_2308_00127_b200.batched import _plan  # noqa: E402

n = int(os.environ.get("QP_N", 1 << 22))
for name in sys.argv[1:] or ["rn50f"]:
    with open(f"tests/golden/instances/{name}.json") as f:
        doc = json.load(f)
    g, hw, t = hs.load_instance(doc)
    for L in [int(x) for x in os.environ.get("QP_L", "2,4,8").split(",")]:
        try:
            plan = _plan(g, hw, t, L, None)
        except Exception as exc:  # noqa: BLE001
            print(f"{name} L={L}: {exc}")
            continue
        nopt = len(plan.options)
        tag = "aot"
        if os.environ.get("QP_JIT", "1") == "1" and plan.jit_eligible():
            plan.specialize()
            tag = "jit"
        genes = torch.randint(0, nopt, (n, plan.pref_ld), dtype=torch.uint8,
                              device="cuda")
        ms = torch.empty(n, dtype=torch.float64, device="cuda")
        best = torch.empty(2, dtype=torch.int64, device="cuda")
        for _ in range(2):
            plan.eval(genes, ms, None, best)
        torch.cuda.synchronize()
        e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
        blocks = []
        for _ in range(3):
            e0.record()
            for _ in range(5):
                plan.eval(genes, ms, None, best)
            e1.record()
            torch.cuda.synchronize()
            blocks.append(e0.elapsed_time(e1) / 5 / 1e3)
        dt = statistics.median(blocks)
        e0.record()
        plan.eval_gen(N.GEN_RANDOM, 1, 0, n, best=best)
        e1.record()
        torch.cuda.synchronize()
        dg = e0.elapsed_time(e1) / 1e3
        print(f"{name} [{tag}] L={L} options={nopt} P={plan.max_parts}: explicit "
              f"{n / dt:.3e} cand/s  gen {n / dg:.3e} cand/s", flush=True)
        del genes
        torch.cuda.empty_cache()
