"""Workloads for ncu captures of the secondary kernels (one each):

    tf96       hs_jit_eval on the transformer case study (node-block classes)
    ws1000     hs_jit_eval on WS1000 (global slot tier)
    sa         one SA run, WS 10x20 (hs_jit_sa)
    sa_multi   148 SA chains, WS 10x20 (hs_jit_sa, grid 148)
    ea_multi   148 EA chains, WS 10x20 (ea_draw_kernel, hs_jit_ea)
    validate   K11 over 2,000 decoded WS200 schedules
    batched    K8 (batched variant) on fused ResNet-50, L = 4
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2308_00127_b200 as hs  # noqa: E402
from paper_2308_00127_b200.plan import get_plan  # noqa: E402


def load(name):
    with open(os.path.join(ROOT, "tests", "golden", "instances",
                           name + ".json")) as f:
        return hs.load_instance(json.load(f))


what = sys.argv[1]
if what in ("tf96", "ws1000"):
    g, hw, t = load(what)
    plan = get_plan(g, hw, t, 1)
    plan.specialize()
    n = 1 << (22 if what == "tf96" else 20)
    genes = torch.randint(0, plan.K, (n, plan.pref_ld), dtype=torch.uint8,
                          device="cuda")
    ms = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(4):
        plan.eval(genes, ms, None, None)
elif what in ("sa", "sa_multi", "ea_multi"):
    g, hw, t = load("ws_stack_10x20")
    hs.specialize(g, hw, t, 1)
    if what == "sa":
        for _ in range(3):
            hs.simulated_annealing(g, hw, t, 1, seed=0, budget=2000)
    elif what == "sa_multi":
        for _ in range(2):
            hs.simulated_annealing_multi(g, hw, t, 1, range(148), budget=2000)
    else:
        for _ in range(2):
            hs.one_plus_one_ea_multi(g, hw, t, 1, range(148), budget=2000)
elif what == "validate":
    g, hw, t = load("ws200")
    plan = get_plan(g, hw, t, 1)
    rng = np.random.default_rng(0)
    order = tuple(plan.order)
    rows = rng.integers(3, size=(2000, plan.V), dtype=np.uint8)
    from paper_2308_00127_b200.heuristics import _decode_rows
    scheds = [s for s in _decode_rows(plan, g, hw, t, 1, rows) if s]
    for _ in range(3):
        hs.validate_schedules(g, hw, t, scheds)
torch.cuda.synchronize()
print("done", what)
if what == "batched":
    # K8 on fused ResNet-50 at L = 4 (15 options, 3 parts)
    g, hw, t = load("rn50f")
    opts = hs.batched_options(g, hw, t, 4)
    genes = torch.randint(0, len(opts), (1 << 22, 112), dtype=torch.uint8,
                          device="cuda")
    for _ in range(3):
        hs.fitness_batched(genes, g, hw, t, 4)
    torch.cuda.synchronize()
    print("done batched")
