"""Quick device-side throughput probe (not the bench contract)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2308_00127_b200 as hs
from paper_2308_00127_b200.plan import get_plan
from paper_2308_00127_b200 import _native as N

for name in sys.argv[1:] or ["ws200"]:
    doc = json.load(open(f"tests/golden/instances/{name}.json"))
    g, hw, t = hs.load_instance(doc)
    plan = get_plan(g, hw, t, 1)
    if os.environ.get("QP_JIT", "1") == "1" and plan.jit_eligible():
        print("specialize ms", plan.specialize())
    n = int(os.environ.get("QP_N", 1 << 22))
    ld = plan.pref_ld
    genes = torch.randint(0, plan.K, (n, ld), dtype=torch.uint8, device="cuda")
    ms = torch.empty(n, dtype=torch.float64, device="cuda")
    best = torch.empty(2, dtype=torch.int64, device="cuda")
    for _ in range(3):
        plan.eval(genes, ms, None, best)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 10
    for _ in range(reps):
        plan.eval(genes, ms, None, best)
    e1.record(); torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) / reps / 1e3
    e0.record()
    for _ in range(reps):
        plan.eval_gen(N.GEN_RANDOM, 1, 0, n, best=best)
    e1.record(); torch.cuda.synchronize()
    dg = e0.elapsed_time(e1) / reps / 1e3
    print(f"{name}: V={plan.V} slots={plan.info.live_slots} explicit {n/dt:.3e} cand/s ({dt*1e3:.2f} ms)  gen {n/dg:.3e} cand/s")
