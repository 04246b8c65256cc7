"""CPU ORACLE of the batched-variant schedule evaluator -- test infra only.

The reference's bMET / bGreedy (heuristics.py:363-433, non-insertion)
split each task's batch of L inputs into sub-batches (a decomposition of L
into allowed sizes, heuristics.py:337-360) placed on distinct devices (a
permutation, :389), choosing per task among those options. Fixing the
choice per task gives an *extended genome* (one option index per genome
position); evaluating it is what the reference does when it commits its
choices. Restated here:

* ``split_sizes`` / ``decompositions`` -- heuristics.py:337-360;
* ``options`` -- the (decomposition, device tuple) list in the order
  batched_variant enumerates it (:372-374, 388-392), devices as indices
  into ``sorted(hw.devices)``;
* ``eval_one`` -- per task in genome order, per part in order:
  ``ready_time`` over predecessors x the part's inputs (:67-78),
  non-insertion start ``max(ready, last end on device)`` (:414), end =
  start + table.get(task, dev, size) (:405), makespan = running max (:120);
  like batched_variant there is no memory check.
Parity is pinned by tests/test_oracle_golden.py against the reference's own
bMET / bGreedy schedules (tests/golden/batched.json).
"""
from __future__ import annotations

import itertools

from .hs_oracle import OK, ST_LINK, ST_MISSING, Instance, bfs_order, pymax

INF = float("inf")


def split_sizes(L: int) -> list:
    sizes = []
    for k in (1, 2, 3, 4):
        if (L * k) % 4 == 0:
            sizes.append(L * k // 4)
    return sorted(set(s for s in sizes if s >= 1))


def decompositions(L: int, sizes: list, max_parts: int) -> list:
    out = []

    def rec(remaining, start, acc):
        if remaining == 0:
            out.append(tuple(acc))
            return
        if len(acc) >= max_parts:
            return
        for k in range(start, len(sizes)):
            if sizes[k] <= remaining:
                rec(remaining - sizes[k], k, acc + [sizes[k]])

    rec(L, 0, [])
    return out


def options(inst: Instance, L: int, splits=None) -> list:
    """[(sizes, devs)] with devs = sorted-device indices."""
    sizes = sorted(set(splits)) if splits else split_sizes(L)
    decomps = decompositions(L, sizes, max_parts=len(inst.dev_ids))
    if (L,) not in decomps and L in sizes:
        decomps.append((L,))
    devs = sorted(inst.dev_ids)
    bsz = {u: inst.batch_sizes[inst.dev_ids.index(u)] for u in devs}
    out = []
    for dec in decomps:
        for perm in itertools.permutations(range(len(devs)), len(dec)):
            if any(dec[k] not in bsz[devs[perm[k]]] for k in range(len(dec))):
                continue
            out.append((tuple(dec), tuple(perm)))
    return out


def eval_one(inst: Instance, L: int, opts: list, genes, order=None,
             trace: bool = False):
    """Extended genome -> (makespan, status[, starts per (position, part)])."""
    order = list(order) if order is not None else bfs_order(inst)
    devs = sorted(inst.dev_ids)
    _, pred = inst.succ_pred()
    tix = {t: k for k, t in enumerate(inst.task_ids)}
    placed = {}  # (task, input) -> (device index, end)
    avail = {}
    ms = 0.0
    starts = []
    for i, t in enumerate(order):
        o = int(genes[i])
        if not 0 <= o < len(opts):
            return (INF, 5, None) if trace else (INF, 5)
        sizes, dv = opts[o]
        parts = []
        nxt = 1
        for k, size in enumerate(sizes):
            inputs = range(nxt, nxt + size)
            nxt += size
            d = dv[k]
            ready = 0.0
            for p in pred[t]:
                om = inst.om[tix[p]]
                for l in inputs:
                    src, end = placed[(p, l)]
                    if src == d:
                        comm = 0.0
                    else:
                        beta = inst.bandwidth.get((devs[src], devs[d]))
                        if beta is None:
                            return (INF, ST_LINK, None) if trace else \
                                (INF, ST_LINK)
                        comm = om / beta
                    ready = pymax(ready, end + comm)
            dur = inst.latency.get((t, devs[d], size))
            if dur is None:
                return (INF, ST_MISSING, None) if trace else (INF, ST_MISSING)
            start = pymax(ready, avail.get(d, 0.0))
            parts.append((d, inputs, start, start + dur))
        row = []
        for d, inputs, start, end in parts:
            avail[d] = end
            for l in inputs:
                placed[(t, l)] = (d, end)
            ms = pymax(ms, end)
            row.append(start)
        starts.append(row)
    return (ms, OK, starts) if trace else (ms, OK)


def genes_from_schedule(inst: Instance, L: int, opts: list, batches,
                        order=None):
    """Extended genome of a reference batched schedule (its commit order is
    task by task, parts in input order)."""
    order = list(order) if order is not None else bfs_order(inst)
    devs = sorted(inst.dev_ids)
    by_task = {}
    for b in batches:
        by_task.setdefault(b[0], []).append(b)
    index = {o: k for k, o in enumerate(opts)}
    return [index[(tuple(b[2] for b in by_task[t]),
                   tuple(devs.index(b[1]) for b in by_task[t]))]
            for t in order]
