import os, sys, time
import numpy as np
ROOT = "/root/repo"
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_2308_00127_b200 as hs
from paper_2308_00127_b200 import heuristics as H
from conftest import instance_doc
g, hw, t = hs.load_instance(instance_doc("ws_stack_10x20"))
s = hs.greedy(g, hw, t, 1)
cur = hs.genome_from_map(g, hw, {b.task: b.device for b in s.batches})
f0 = hs.fitness(cur, g, hw, t, 1)
plan = H.get_plan(g, hw, t, 1)
genes = np.array(cur.genes, np.uint8)
for win in (128, 32, 8):
    ts = []
    for rep in range(5):
        gen = np.random.default_rng(0)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        H._sa_device_chain(plan, gen, genes, f0, f0, 0.1 * f0, 0.995, 2000, len(hw.devices), win)
        ts.append(round(1e3 * (time.perf_counter() - t0), 1))
    print("SA win", win, ts, flush=True)
p = 1.0 / len(genes)
ts = []
for rep in range(5):
    gen = np.random.default_rng(0)
    t0 = time.perf_counter()
    H._ea_device_chain(plan, gen, genes, f0, 2000, len(genes), len(hw.devices), p)
    ts.append(round(1e3 * (time.perf_counter() - t0), 1))
print("EA", ts)
