"""The reference's throughput-mode acceptance check (test_acceptance.py:
298-321) on the B200 path: on 20 random L = 2 instances, an exhaustive GPU
sweep (K8) of every extended genome -- every per-task choice of sub-batch
decomposition x devices the batched variants can make -- never beats the
brute-force optimum (oracle.py brute_force, throughput objective, frozen in
tests/golden/throughput.json) and never loses to the reference's bMET /
bGreedy schedules, whose own extended genomes K8 re-scores bit for bit;
bHEFT (insertion-based, not an extended genome) never beats the oracle
either."""
from __future__ import annotations

import itertools
import json

import numpy as np
import pytest

from conftest import fhex, golden

import paper_2308_00127_b200 as hs
from paper_2308_00127_b200.core import (Schedule, ScheduledBatch, load_graph,
                                        load_hardware, load_latency)

pytestmark = pytest.mark.gpu
TOL = 1e-6


def _sched(s, L):
    return Schedule(batches=tuple(
        ScheduledBatch(task=t, device=d, size=z, inputs=tuple(ins),
                       start=float.fromhex(st))
        for t, d, z, ins, st in s["batches"]),
        objective=float.fromhex(s["objective"]), input_count=L)


def test_throughput_mode_acceptance():
    import torch
    for e in golden("throughput"):
        g = load_graph(json.dumps(e["graph"]))
        hw = load_hardware(json.dumps(e["hardware"]))
        t = load_latency(json.dumps(e["latency"]))
        L = e["L"]
        opt = float.fromhex(e["oracle_objective"])
        nopt = len(hs.batched_options(g, hw, t, L))
        V = len(g.tasks)
        rows = np.array(list(itertools.product(range(nopt), repeat=V)),
                        np.uint8).reshape(-1, V)
        ms = hs.fitness_batched(torch.from_numpy(rows).cuda(), g, hw, t, L)
        best = float(ms.min().item())
        assert best >= opt - TOL, e["seed"]
        assert 1000.0 * L / best <= 1000.0 * L / opt * (1 + 1e-9)
        for algo, b in e["batched"].items():
            obj = float.fromhex(b["objective"])
            assert obj >= opt - TOL, (e["seed"], algo)
            if algo == "heft":
                continue
            s = _sched(b, L)
            genes = hs.batched_genes_from_schedule(s, g, hw, t, L)
            got = hs.fitness_batched(np.array([genes], np.uint8), g, hw, t, L)
            assert fhex(float(got[0])) == b["objective"], (e["seed"], algo)
            assert best <= obj, (e["seed"], algo)
