"""CPU ORACLE of the search heuristics -- test / baseline infrastructure only.

Restates the reference's consumers of the evaluator on top of the oracle
decoder (oracle/hs_oracle.py::fitness_one): MET (heuristics.py:170-189),
greedy (:192-210), simulated annealing (:259-299) and the (1+1) EA
(:302-334), one candidate per step exactly like the reference. Used (1) to
pin trajectories against tests/golden/heuristics.json and (2) as the CPU
arm of bench.py's heuristic time-to-solution. Never on the product path.
"""
from __future__ import annotations

import math

import numpy as np

from .hs_oracle import OK, Instance, Tables, build_tables, fitness_one


def _genes_from_map(tb: Tables, mapping: dict) -> list:
    return [tb.devs.index(mapping[t]) for t in tb.order]


def met_mapping(inst: Instance, L: int) -> dict:
    """heuristics.py:170-189 (ties within 1e-12 to the smaller id)."""
    devs = sorted(inst.dev_ids)
    di = {u: inst.dev_ids.index(u) for u in devs}
    out = {}
    for t in inst.task_ids:
        best = None
        for u in devs:
            if L not in inst.batch_sizes[di[u]]:
                continue
            ms = inst.latency[(t, u, L)]
            if best is None or ms < best[0] - 1e-12:
                best = (ms, u)
        out[t] = best[1]
    return out


def greedy_mapping(inst: Instance, tb: Tables, L: int) -> dict:
    """heuristics.py:192-210 on the oracle's flat list scheduler."""
    K = tb.K
    avail = [0.0] * K
    mem = [0.0] * K
    end = [0.0] * tb.V
    where = [0] * tb.V
    ms = 0.0
    out = {}
    for i in range(tb.V):
        choice = None
        for d in range(K):
            if not tb.okL[d] or mem[d] + tb.extra[i] > tb.cap[d]:
                continue
            r, ok = 0.0, True
            for p in tb.preds[i]:
                if not tb.link[where[p], d]:
                    ok = False
                    break
                c = 0.0 if where[p] == d else float(tb.comm[p, where[p], d])
                x = end[p] + c
                r = x if x > r else r
            if not ok:
                continue
            s = avail[d] if avail[d] > r else r
            e = s + float(tb.dur[i, d])
            cand = e if e > ms else ms
            if choice is None or cand < choice[0] - 1e-12:
                choice = (cand, d, e)
        _, d, e = choice
        end[i], where[i] = e, d
        avail[d] = e
        mem[d] += float(tb.extra[i])
        ms = e if e > ms else ms
        out[tb.order[i]] = tb.devs[d]
    return out


def simulated_annealing(inst: Instance, L: int, seed: int = 0,
                        budget: int = 2000, t0_fraction: float = 0.1,
                        alpha: float = 0.995):
    """heuristics.py:259-299 -> (best makespan, best genes)."""
    tb = build_tables(inst, L)
    rng = np.random.default_rng(seed)
    genes = _genes_from_map(tb, greedy_mapping(inst, tb, L))
    cur_fit = fitness_one(tb, genes)[0]
    best, best_fit = list(genes), cur_fit
    temp = max(t0_fraction * cur_fit, 1e-9)
    n_dev = tb.K
    for _ in range(budget):
        pos = int(rng.integers(len(genes)))
        old = genes[pos]
        if n_dev > 1:
            new = int(rng.integers(n_dev - 1))
            if new >= old:
                new += 1
        else:
            new = old
        genes[pos] = new
        cand_fit = fitness_one(tb, genes)[0]
        delta = cand_fit - cur_fit
        accept = delta <= 0 or (math.isfinite(cand_fit)
                                and rng.random() < math.exp(-delta / temp))
        if accept:
            cur_fit = cand_fit
            if cand_fit < best_fit:
                best, best_fit = list(genes), cand_fit
        else:
            genes[pos] = old
        temp *= alpha
    return best_fit, best


def one_plus_one_ea(inst: Instance, L: int, seed: int = 0, budget: int = 2000,
                    biased: bool = True):
    """heuristics.py:302-334 -> (final makespan, final genes)."""
    tb = build_tables(inst, L)
    rng = np.random.default_rng(seed)
    n_dev = tb.K
    if biased:
        genes = _genes_from_map(tb, met_mapping(inst, L))
    else:
        genes = [int(v) for v in rng.integers(n_dev, size=tb.V)]
    cur_fit = fitness_one(tb, genes)[0]
    p = 1.0 / max(tb.V, 1)
    for _ in range(budget):
        child = list(genes)
        for pos in range(len(child)):
            if rng.random() < p:
                child[pos] = int(rng.integers(n_dev))
        cand_fit = fitness_one(tb, child)[0]
        if cand_fit <= cur_fit:
            genes, cur_fit = child, cand_fit
    return cur_fit, genes
