"""GPU module solver for the split heuristic (MILP-SPLIT).

The reference's ``milp_split`` (/root/reference/pkg/src/hetsched/
splitting.py:259-402) solves every module once per pinning of its channel
endpoints through a pluggable ``ModuleSolver`` (splitting.py:225), called as
``solver(sub, hw, table, L, pins, same_device, timeout)`` and returning
``(objective, schedule, proven_optimal)`` or ``(None, None, False)``
(splitting.py:228-245, 338-340). ``gpu_module_solver`` is a drop-in for that
slot: it sweeps the module's mappings on the B200 -- exhaustively when the
free assignments number at most ``exhaustive_limit``, otherwise by on-device
random sampling followed by batched best-improvement 1-opt -- with pinned
tasks fixed and ``same_device`` pairs tied (milp.py:277-291), and returns the
decoded schedule of the best mapping. The objective is the list-scheduling
makespan, so ``proven_optimal`` is False (optimal over decoder mappings, not
a MILP certificate); the reference DP then flags the result quasi-optimal.
It is thread-safe (the DP may call it from a thread pool).
"""
from __future__ import annotations

import time
from typing import Callable, Optional

import numpy as np

from . import _native as N
from .core import Schedule
from .heuristics import MappingGenome, decode, _fit_rows
from .plan import get_plan

ModuleSolver = Callable[..., tuple[Optional[float], Optional[Schedule], bool]]


def _groups(order, devs, pins, same_device):
    """Union the same-device pairs; pinned groups become fixed genes.
    Returns (template u8[V], group i16[V], n_groups) or None if pins clash."""
    pos = {t: i for i, t in enumerate(order)}
    parent = list(range(len(order)))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    for a, b in same_device or ():
        if a in pos and b in pos:
            ra, rb = find(pos[a]), find(pos[b])
            if ra != rb:
                parent[max(ra, rb)] = min(ra, rb)
    dix = {u: k for k, u in enumerate(devs)}
    fixed: dict[int, int] = {}
    for t, u in (pins or {}).items():
        if t not in pos:
            continue
        r = find(pos[t])
        k = dix[u]
        if fixed.setdefault(r, k) != k:
            return None
    V = len(order)
    template = np.zeros(V, np.uint8)
    group = np.full(V, -1, np.int16)
    gid: dict[int, int] = {}
    for i in range(V):
        r = find(i)
        if r in fixed:
            template[i] = fixed[r]
        else:
            if r not in gid:
                gid[r] = len(gid)
            group[i] = gid[r]
    return template, group, len(gid)


def gpu_module_solver(objective: str = "latency", *,
                      exhaustive_limit: int = 1 << 24,
                      samples: int = 1 << 22, refine_rounds: int = 64,
                      seed: int = 0) -> ModuleSolver:
    """Build a ModuleSolver (see module docstring). `objective` is accepted
    for signature parity: latency and throughput share the makespan
    (milp.py:144-146)."""
    if objective not in ("latency", "throughput"):
        raise ValueError(f"unknown objective {objective!r}")

    def solver(sub, hw, table, L, pins, same_device, timeout):
        import torch
        plan = get_plan(sub, hw, table, L)
        V, K = plan.V, plan.K
        if V == 0:
            return 0.0, Schedule(batches=(), objective=0.0, input_count=L), False
        devs = sorted(hw.devices)
        gr = _groups(plan.order, devs, pins, same_device)
        if gr is None:
            return None, None, False
        template, group, ng = gr
        deadline = None if timeout is None else time.monotonic() + timeout
        d_t = torch.from_numpy(template).cuda()
        d_g = torch.from_numpy(group).cuda()
        best = torch.empty(2, dtype=torch.int64, device="cuda")
        space = K ** ng
        mode = N.GEN_ENUM if space <= exhaustive_limit else N.GEN_RANDOM
        total = space if mode == N.GEN_ENUM else samples
        chunk = 1 << 22
        found = (float("inf"), -1)
        for lo in range(0, total, chunk):
            m = min(chunk, total - lo)
            plan.eval_gen(mode, seed, lo, m, template=d_t, group=d_g,
                          n_groups=ng, best=best)
            b = best.cpu()
            c = (float(b[:1].view(torch.float64).item()), int(b[1].item()))
            if c < found:
                found = c
            if deadline is not None and time.monotonic() > deadline:
                break
        if found[1] < 0:
            return None, None, False
        out = torch.empty((1, V), dtype=torch.uint8, device="cuda")
        plan.eval_gen(mode, seed, found[1], 1, template=d_t, group=d_g,
                      n_groups=ng, genes_out=out)
        genes = out.cpu().numpy()[0].copy()
        cost = found[0]
        if mode == N.GEN_RANDOM and np.isfinite(cost):
            genes, cost = _refine(plan, genes, cost, group, K,
                                  refine_rounds, deadline)
        if not np.isfinite(cost):
            return None, None, False
        sched = decode(MappingGenome(genes=tuple(int(x) for x in genes),
                                     order=plan.order), sub, hw, table, L)
        if sched is None:
            return None, None, False
        return sched.objective, sched, False

    return solver


def _refine(plan, genes, cost, group, K, rounds, deadline):
    """Best-improvement 1-opt over free groups, one GPU batch per round."""
    ng = int(group.max()) + 1 if (group >= 0).any() else 0
    members = [np.flatnonzero(group == j) for j in range(ng)]
    for _ in range(rounds):
        rows, ok = [], []
        for j in range(ng):
            cur = genes[members[j][0]]
            for k in range(K):
                if k == cur:
                    continue
                r = genes.copy()
                r[members[j]] = k
                rows.append(r)
        if not rows:
            break
        fits = _fit_rows(plan, np.stack(rows))
        k = int(np.argmin(fits))
        if not fits[k] < cost:
            break
        genes, cost = rows[k], float(fits[k])
        if deadline is not None and time.monotonic() > deadline:
            break
    return genes, cost
