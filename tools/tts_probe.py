"""Where the heuristic time-to-solution goes (WS 10x20 stack, budget 2000):
start heuristic, device chain, final decode; cold and warm runs.

    python tools/tts_probe.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2308_00127_b200 as hs  # noqa: E402
from paper_2308_00127_b200 import heuristics as H  # noqa: E402
from conftest import instance_doc  # noqa: E402


def tick(label, fn):
    t0 = time.perf_counter()
    r = fn()
    print(f"  {label}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
    return r


def main():
    g, hw, t = hs.load_instance(instance_doc("ws_stack_10x20"))
    hs.fitness(hs.genome_from_map(g, hw, {i: sorted(hw.devices)[0] for i in g.tasks}),
               g, hw, t, 1)
    for rep in range(3):
        print(f"run {rep}")
        s = tick("greedy", lambda: hs.greedy(g, hw, t, 1))
        s = tick("met", lambda: hs.met(g, hw, t, 1))
        cur = hs.genome_from_map(g, hw, {b.task: b.device for b in s.batches})
        tick("fitness", lambda: hs.fitness(cur, g, hw, t, 1))
        tick("decode", lambda: hs.decode(cur, g, hw, t, 1))
        tick("SA total", lambda: hs.simulated_annealing(g, hw, t, 1, seed=0, budget=2000))
        tick("EA total", lambda: hs.one_plus_one_ea(g, hw, t, 1, seed=0, budget=2000))
        plan = H.get_plan(g, hw, t, 1)
        gen = np.random.default_rng(0)
        genes = np.array(cur.genes, np.uint8)
        f0 = hs.fitness(cur, g, hw, t, 1)
        tick("SA device chain only", lambda: H._sa_device_chain(
            plan, gen, genes, f0, f0, 0.1 * f0, 0.995, 2000, len(hw.devices), 128))
        gen = np.random.default_rng(0)
        tick("EA device chain only", lambda: H._ea_device_chain(
            plan, gen, genes, f0, 2000, len(genes), len(hw.devices), 1.0 / len(genes)))


if __name__ == "__main__":
    main()
