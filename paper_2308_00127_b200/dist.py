"""Multi-GPU candidate sweeps: one process per GPU, contiguous candidate
shards, and one collective per batch to agree on the global best.

Candidates are independent, so rank r of W evaluates the
global index range ``shard_range(n, W, r)`` against its own replica of the
(KB-sized) plan, reduces it on device to a first-index (cost, index) best,
and the ranks exchange 16 bytes each with one ``all_gather`` (NCCL over
NVLink on GPUs; gloo in the CPU tests). The lexicographic merge is the
same on every rank, so every rank ends with the same answer. NCCL has no
argmin operator; gathering 16 B per rank and merging locally is one
latency-bound collective.
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

INF = float("inf")


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of rank `rank` when n candidates are split over `world`
    ranks as evenly as possible (the first n % world ranks get one more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    q, r = divmod(n, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def merge_best(bests: Sequence[tuple[float, int]]) -> tuple[float, int]:
    """Lexicographic (cost, index) minimum; entries with index < 0 (empty
    shards) are ignored; all empty -> (inf, -1)."""
    out = (INF, -1)
    for c, i in bests:
        if i < 0:
            continue
        if out[1] < 0 or c < out[0] or (c == out[0] and i < out[1]):
            out = (float(c), int(i))
    return out


def allgather_best(best: tuple[float, int], group=None,
                   device: Optional[str] = None) -> tuple[float, int]:
    """Exchange one (cost, index) per rank with a single all_gather and
    merge. The pair travels as two int64 words (cost bit pattern, index)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.empty(2, dtype=torch.int64, device=device)
    t[0] = torch.tensor([best[0]], dtype=torch.float64).view(torch.int64)[0]
    t[1] = int(best[1])
    out = torch.empty(2 * world, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out, t, group=group)
    o = out.cpu().view(world, 2)
    costs = o[:, 0].clone().view(torch.float64)
    return merge_best([(float(costs[r]), int(o[r, 1])) for r in range(world)])


def nccl_comm(group=None) -> int:
    """The ncclComm_t (as an int) of torch's NCCL process group on the
    current device. Initialise the group eagerly (``init_process_group(...,
    device_id=...)``) so the communicator exists."""
    import torch
    import torch.distributed as dist
    pg = group if group is not None else \
        dist.distributed_c10d._get_default_group()
    be = pg._get_backend(torch.device("cuda", torch.cuda.current_device()))
    ptr = int(be._comm_ptr())
    if not ptr:
        raise RuntimeError("NCCL communicator not initialised")
    return ptr


def best_allreduce_device(best, out, comm: int, stream=None) -> None:
    """hs_best_allreduce: `best` int64[2] device tensor (cost bits, global
    index; hs_eval's fused argmin) -> `out` int64[2], the lexicographic
    minimum over every rank of `comm` (one ncclAllGather of 16 B per rank
    and an on-device merge, all on `stream`)."""
    import ctypes as C

    import torch

    from . import _native as N
    s = stream if stream is not None else torch.cuda.current_stream()
    N.check(N.load().hs_best_allreduce(
        C.c_void_p(best.data_ptr()), C.c_void_p(out.data_ptr()),
        C.c_void_p(comm), C.c_void_p(int(s.cuda_stream))),
        "hs_best_allreduce")


def sharded_best(n: int, evaluate: Callable[[int, int], tuple[float, int]],
                 group=None, device: Optional[str] = None) -> tuple[float, int]:
    """Evaluate this rank's shard with `evaluate(lo, hi) -> (cost, global
    index)` and return the global best of all ranks."""
    import torch.distributed as dist
    lo, hi = shard_range(n, dist.get_world_size(group), dist.get_rank(group))
    local = evaluate(lo, hi) if hi > lo else (INF, -1)
    return allgather_best(local, group=group, device=device)


def random_search_sharded(g, hw, table, L: int, n: int, *, seed: int = 0,
                          group=None):
    """`heuristics.random_search` over all ranks: rank r sweeps its shard of
    the on-device generated candidates [0, n) on its own GPU."""
    from .heuristics import random_search

    def ev(lo, hi):
        cost, idx, _ = random_search(g, hw, table, L, hi - lo, seed=seed,
                                     first=lo)
        return cost, idx

    return sharded_best(n, ev, group=group, device="cuda")
