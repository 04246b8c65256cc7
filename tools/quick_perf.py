"""Device-side throughput probe of the evaluator (not the bench contract).

    python tools/quick_perf.py ws200 tf96 ...   (QP_N candidates, QP_JIT=0
    for the ahead-of-time kernel, HS_JIT_OPTS for code-generation options)

Median of QP_BLOCKS (5) blocks of 10 launches over QP_N explicit genomes (default
2**24, larger than L2), plus one block of on-device generated candidates.
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2308_00127_b200 as hs  # noqa: E402
from paper_2308_00127_b200 import _native as N  # noqa: E402
from paper_2308_00127_b200.plan import get_plan  # noqa: E402

n = int(os.environ.get("QP_N", 1 << 24))
for name in sys.argv[1:] or ["ws200"]:
    with open(f"tests/golden/instances/{name}.json") as f:
        doc = json.load(f)
    g, hw, t = hs.load_instance(doc)
    plan = get_plan(g, hw, t, 1)
    tag = "aot"
    if os.environ.get("QP_JIT", "1") == "1" and plan.jit_eligible():
        plan.specialize()
        tag = "jit"
    genes = torch.randint(0, plan.K, (n, plan.pref_ld), dtype=torch.uint8,
                          device="cuda")
    ms = torch.empty(n, dtype=torch.float64, device="cuda")
    best = torch.empty(2, dtype=torch.int64, device="cuda")
    for _ in range(3):
        plan.eval(genes, ms, None, best)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    blocks = []
    for _ in range(int(os.environ.get("QP_BLOCKS", 5))):
        e0.record()
        for _ in range(10):
            plan.eval(genes, ms, None, best)
        e1.record()
        torch.cuda.synchronize()
        blocks.append(e0.elapsed_time(e1) / 10 / 1e3)
    dt = statistics.median(blocks)
    dmin = min(blocks)
    e0.record()
    for _ in range(5):
        plan.eval_gen(N.GEN_RANDOM, 1, 0, n, best=best)
    e1.record()
    torch.cuda.synchronize()
    dg = e0.elapsed_time(e1) / 5 / 1e3
    print(f"{name} [{tag}]: V={plan.V} explicit {n / dt:.3e} cand/s "
          f"({dt * 1e3:.2f} ms, best {n / dmin:.3e}, blocks {[round(b * 1e3, 2) for b in blocks]})"
          f"  gen {n / dg:.3e} cand/s", flush=True)
    del genes
    torch.cuda.empty_cache()
