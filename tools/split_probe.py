"""Config 3 probe: the split heuristic with the GPU module solver on the WS
stacks -- objective, wall time, validation and lower-bound gap -- for a few
module-solver settings (local-search starts / pair moves)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2308_00127_b200 as hs  # noqa: E402

for name in sys.argv[1:] or ["ws_stack_10x20", "ws_stack_10x100"]:
    with open(os.path.join(ROOT, "tests", "golden", "instances",
                           name + ".json")) as f:
        g, hw, t = hs.load_instance(json.load(f))
    d = hs.k_edge_components(g, 1)
    lb = hs.lower_bound(g, hw, t, 1, d, subgraph_cap=0).lower_bound_ms
    for kw in ({"starts": 1, "pair_moves": False}, {"starts": 8},
               {"starts": 32}, {"starts": 8, "samples": 1 << 24}):
        t0 = time.perf_counter()
        s = hs.milp_split(g, hw, t, 1, d, workers=8,
                          module_solver=hs.gpu_module_solver(**kw))
        el = time.perf_counter() - t0
        mk = hs.validate_schedule(g, hw, t, s)
        print(f"{name} {kw}: objective {s.objective:.2f} ms (validated "
              f"{mk:.2f}), {el:.2f} s, gap to LB {s.objective / lb - 1:.3f}",
              flush=True)
