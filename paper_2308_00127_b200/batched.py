"""Batched-variant schedules (bMET / bGreedy placement) as extended genomes.

The reference's batched variants (heuristics.py:363-433) split each task's
batch of L inputs into sub-batches of allowed sizes placed on distinct
devices, choosing per task among options enumerated as decompositions
(:337-360) x device permutations (:389). Here the choice per task is a gene:
``batched_options`` lists the options in the reference's enumeration order,
and ``fitness_batched`` / ``decode_batched`` evaluate extended genomes on
the GPU with the reference's non-insertion placement (no memory check, like
batched_variant), so search loops can explore batched mappings for the
throughput objective 1000 * L / makespan.
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from . import _native as N
from .core import GraphError, Schedule, ScheduledBatch
from .heuristics import INF, _batch_genes, _raise_status
from .plan import get_plan


def _plan(g, hw, table, L, splits):
    return get_plan(g, hw, table, L, None, tuple(splits or ()))


def batched_options(g, hw, table, L: int, splits: Optional[Sequence[int]] = None
                    ) -> list:
    """[(sub-batch sizes, device ids)] in batched_variant's order; the index
    into this list is the extended gene."""
    return list(_plan(g, hw, table, L, splits).options)


def fitness_batched(genes, g, hw, table, L: int, *,
                    splits: Optional[Sequence[int]] = None,
                    return_status: bool = False):
    """Makespans of extended genomes uint8 [n, >=V] (numpy -> host path,
    CUDA tensor -> device path)."""
    plan = _plan(g, hw, table, L, splits)
    genes = _batch_genes(genes, plan.V)
    plan.maybe_specialize(len(genes))  # graph-specialised K8 for big batches
    if hasattr(genes, "data_ptr"):
        import torch
        n = genes.shape[0]
        ms = torch.empty(n, dtype=torch.float64, device=genes.device)
        st = torch.empty(n, dtype=torch.uint8, device=genes.device)
        plan.eval(genes, ms, st, None)
        if return_status:
            return ms, st
        if n and int(st.max().item()) >= N.ST_MISSING:
            _raise_status(int(st.max().item()))
        return ms
    ms = np.empty(len(genes), np.float64)
    st = np.empty(len(genes), np.uint8)
    if len(genes):
        plan.eval_host(genes, ms, st, None)
    if return_status:
        return ms, st
    if len(st) and st.max() >= N.ST_MISSING:
        _raise_status(int(st.max()))
    return ms


def decode_batched(genes: Sequence[int], g, hw, table, L: int, *,
                   splits: Optional[Sequence[int]] = None) -> Optional[Schedule]:
    """Schedule of one extended genome (batches in commit order: task by
    task in BFS order, sub-batches in input order), or None if a link is
    missing."""
    import torch
    plan = _plan(g, hw, table, L, splits)
    V, P = plan.V, plan.max_parts
    if len(genes) != V:
        raise GraphError("genome length must equal task count")
    if any(not 0 <= int(x) < len(plan.options) for x in genes):
        raise GraphError("gene value out of option range")
    if V == 0:
        return Schedule(batches=(), objective=0.0, input_count=L)
    row = np.zeros((1, plan.pref_ld), np.uint8)
    row[0, :V] = np.asarray(genes, np.uint8)
    d = torch.from_numpy(row).cuda()
    starts = torch.empty(V * P, dtype=torch.float64, device="cuda")
    ms = torch.empty(1, dtype=torch.float64, device="cuda")
    st = torch.empty(1, dtype=torch.uint8, device="cuda")
    plan.trace(d, starts, ms, st)
    s = int(st.item())
    _raise_status(s)
    if s != N.ST_OK:
        return None
    sv = starts.cpu().numpy().reshape(V, P)
    batches = []
    for i, t in enumerate(plan.order):
        sizes, devs = plan.options[int(genes[i])]
        lo = 1
        for k, (size, dev) in enumerate(zip(sizes, devs)):
            batches.append(ScheduledBatch(task=t, device=dev, size=size,
                                          inputs=tuple(range(lo, lo + size)),
                                          start=float(sv[i, k])))
            lo += size
    return Schedule(batches=tuple(batches), objective=float(ms.item()),
                    input_count=L)


def batched_genes_from_schedule(s, g, hw, table, L: int, *,
                                splits: Optional[Sequence[int]] = None) -> list:
    """Extended genome of a batched schedule (e.g. the reference's
    batched_variant("met" | "greedy") output)."""
    plan = _plan(g, hw, table, L, splits)
    index = {o: k for k, o in enumerate(plan.options)}
    parts: dict = {}
    for b in s.batches:
        parts.setdefault(b.task, []).append(b)
    out = []
    for t in plan.order:
        bs = sorted(parts[t], key=lambda b: b.inputs[0])
        key = (tuple(b.size for b in bs), tuple(b.device for b in bs))
        if key not in index:
            raise GraphError(f"task {t!r}: sub-batches {key} are not an option")
        out.append(index[key])
    return out


def random_search_batched(g, hw, table, L: int, n: int, *, seed: int = 0,
                          splits: Optional[Sequence[int]] = None):
    """Best of n on-device generated extended genomes:
    (makespan, index, genes)."""
    import torch
    plan = _plan(g, hw, table, L, splits)
    plan.maybe_specialize(n)
    best = torch.empty(2, dtype=torch.int64, device="cuda")
    plan.eval_gen(N.GEN_RANDOM, seed, 0, n, best=best)
    b = best.cpu()
    cost, idx = float(b[:1].view(torch.float64).item()), int(b[1].item())
    if idx < 0:
        return INF, -1, None
    out = torch.empty((1, plan.V), dtype=torch.uint8, device="cuda")
    plan.eval_gen(N.GEN_RANDOM, seed, idx, 1, genes_out=out)
    return cost, idx, [int(x) for x in out.cpu()[0]]
