"""Search time-to-solution under the current HS_JIT_OPTS: median wall time
of 5 warm SA and EA runs (budget 2000, seed 0) per instance.

    HS_JIT_OPTS=ahead=4 python tools/tts_sweep.py ws_stack_10x20 ws200 tf96
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2308_00127_b200 as hs  # noqa: E402

for name in sys.argv[1:] or ["ws_stack_10x20", "ws200", "tf96"]:
    with open(os.path.join(ROOT, "tests", "golden", "instances",
                           name + ".json")) as f:
        g, hw, t = hs.load_instance(json.load(f))
    hs.specialize(g, hw, t, 1)
    row = []
    for algo, fn in (("sa", hs.simulated_annealing),
                     ("ea", hs.one_plus_one_ea)):
        s = fn(g, hw, t, 1, seed=0, budget=2000)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            fn(g, hw, t, 1, seed=0, budget=2000)
            ts.append(time.perf_counter() - t0)
        row.append(f"{algo} {statistics.median(ts) * 1e3:.2f} ms "
                   f"(obj {s.objective:.3f})")
    print(os.environ.get("HS_JIT_OPTS", ""), name, " | ".join(row),
          flush=True)
