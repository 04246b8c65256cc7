"""Interleaved A/B of the EA search kernel with one and two speculation
levels (HS_EA_LEVELS), wall time per run, same process and box.

    python tools/ea_ab.py [instance] [reps]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2308_00127_b200 as hs  # noqa: E402
from paper_2308_00127_b200 import heuristics as H  # noqa: E402
from conftest import instance_doc  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "ws_stack_10x20"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 7
g, hw, t = hs.load_instance(instance_doc(name))
hs.specialize(g, hw, t, 1)
res = {"1": [], "2": []}
rounds = {}
for _ in range(reps):
    for lv in ("1", "2"):
        os.environ["HS_EA_LEVELS"] = lv
        w0 = time.perf_counter()
        hs.one_plus_one_ea(g, hw, t, 1, seed=0, budget=2000)
        res[lv].append(round(1e3 * (time.perf_counter() - w0), 1))
        rounds[lv] = H._last_chain_stats.get("ea_rounds")
for lv in ("1", "2"):
    v = sorted(res[lv])
    print(name, "levels", lv, "median ms", v[len(v) // 2], "rounds", rounds[lv], res[lv])
