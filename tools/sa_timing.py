"""Per-run device time (CUDA events around the search launch) and wall time
of SA / EA on one instance: separates GPU-side from host-side variance.

    python tools/sa_timing.py [instance] [reps]

SLEEP_CYCLES=N queues a busy-wait of N cycles before the start event, so the
host's launch preparation overlaps it and the events time the kernel alone.
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2308_00127_b200 as hs  # noqa: E402
from paper_2308_00127_b200 import heuristics as H  # noqa: E402
from conftest import instance_doc  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "ws_stack_10x20"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
g, hw, t = hs.load_instance(instance_doc(name))
hs.specialize(g, hw, t, 1)
orig = H.Plan.sa_run
dev_ms = []


SLEEP = int(os.environ.get("SLEEP_CYCLES", "0"))


def timed(self, *a, **k):
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if SLEEP:  # keep the GPU busy while the host prepares the launch, so
        torch.cuda._sleep(SLEEP)  # the events bracket device time only
    s0.record()
    orig(self, *a, **k)
    s1.record()
    s1.synchronize()
    dev_ms.append(s0.elapsed_time(s1))


H.Plan.sa_run = timed
parts = {"greedy": [], "chain": [], "decode": []}


def _timed_part(name, fn):
    def run(*a, **k):
        w0 = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            parts[name].append(round(1e3 * (time.perf_counter() - w0), 1))
    return run


H.greedy = _timed_part("greedy", H.greedy)
H._sa_device_chain = _timed_part("chain", H._sa_device_chain)
H.decode = _timed_part("decode", H.decode)
if os.environ.get("NOGC"):
    import gc
    gc.disable()
for algo in ("sa", "ea"):
    walls = []
    for _ in range(reps):
        w0 = time.perf_counter()
        if algo == "sa":
            hs.simulated_annealing(g, hw, t, 1, seed=0, budget=2000)
        else:
            hs.one_plus_one_ea(g, hw, t, 1, seed=0, budget=2000)
        walls.append(round(1e3 * (time.perf_counter() - w0), 1))
    print(name, algo, "wall ms", walls)
print(name, "sa kernel ms", [round(x, 1) for x in dev_ms])
for k, v in parts.items():
    print(name, "part", k, v[:reps])
