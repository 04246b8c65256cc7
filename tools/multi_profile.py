"""Host-side profile of the multi-chain searches (cProfile, cumulative):
where the wall time of simulated_annealing_multi / one_plus_one_ea_multi
goes besides the search kernel.

    python tools/multi_profile.py ws200
"""
import cProfile
import json
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2308_00127_b200 as hs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "ws200"
with open(f"tests/golden/instances/{name}.json") as f:
    g, hw, t = hs.load_instance(json.load(f))
hs.specialize(g, hw, t, 1)
for fn in (hs.simulated_annealing_multi, hs.one_plus_one_ea_multi):
    for _ in range(2):
        fn(g, hw, t, 1, range(148))
    torch.cuda.synchronize()
    w = []
    for _ in range(3):
        t0 = time.perf_counter()
        fn(g, hw, t, 1, range(148))
        w.append(time.perf_counter() - t0)
    print(fn.__name__, "wall ms", [round(x * 1e3, 2) for x in w])
    pr = cProfile.Profile()
    pr.enable()
    fn(g, hw, t, 1, range(148))
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
