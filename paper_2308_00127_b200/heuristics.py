"""Genome encoding, the GPU-backed list-scheduling decoder, and the heuristics
that consume it -- the drop-in for ``hetsched.heuristics``
(/root/reference/pkg/src/hetsched/heuristics.py).

* ``decode`` / ``fitness`` (heuristics.py:127-148) evaluate on the B200
  through the C ABI (hs_trace / hs_eval); results are bit-identical to the
  reference's Python list scheduler.
* ``fitness_batch`` / ``argmin_batch`` / ``random_search`` are the batched
  entry points (no reference counterpart: the reference evaluates one genome
  per call).
* ``best_device`` / ``met`` (:151-189) compute their mapping on the host and
  decode on the GPU; ``greedy`` (:192-210) is a host list scheduler (K-way
  per-step choice, nothing to batch) used as SA's start.
* ``simulated_annealing`` / ``one_plus_one_ea`` (:259-334) keep the
  reference's exact trajectory for a given seed while evaluating their
  candidates in speculative GPU batches (rng.py replays numpy's stream).
"""
from __future__ import annotations

import functools
import gc
import math
import threading
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from . import rng as R
from .core import (GraphError, Schedule, ScheduledBatch, ScheduleError,
                   bfs_topological_order)
from .plan import Plan, get_plan

INF = float("inf")


@dataclass(frozen=True)
class MappingGenome:
    genes: tuple[int, ...]  # device index per task, BFS topological positions
    order: tuple[str, ...]  # the task ordering the positions refer to

    def __post_init__(self):
        if len(self.genes) != len(self.order):
            raise GraphError("genome length must equal task count")


def genome_from_map(g, hw, mapping: dict) -> MappingGenome:
    """Genes = index into sorted(hw.devices), positions = BFS order
    (heuristics.py:34-40)."""
    order = tuple(bfs_topological_order(g))
    idx = {u: k for k, u in enumerate(sorted(hw.devices))}
    return MappingGenome(genes=tuple(idx[mapping[t]] for t in order),
                         order=order)


# ---------------------------------------------------------------------------
# small-batch evaluation context (one per thread): reuses device buffers so
# single-genome calls cost one H2D, one launch and one D2H

class _Ctx(threading.local):
    def __init__(self):
        self.cap = 0
        self.genes = self.ms = self.st = self.starts = None
        self.stream = None


_ctx = _Ctx()


def _device_buffers(n: int, ld: int, V: int, trace: bool):
    import torch
    c = _ctx
    if c.stream is None:
        c.stream = torch.cuda.Stream()
    need = n * ld
    if c.genes is None or c.genes.numel() < need or c.cap < n:
        cap = max(n, 2 * c.cap, 64)
        c.cap = cap
        c.genes = torch.empty(cap * max(ld, 1) + 16, dtype=torch.uint8,
                              device="cuda")
        c.ms = torch.empty(cap, dtype=torch.float64, device="cuda")
        c.st = torch.empty(cap, dtype=torch.uint8, device="cuda")
        c.starts = None
    if trace and (c.starts is None or c.starts.numel() < n * max(V, 1)):
        c.starts = torch.empty(max(n * V, 1), dtype=torch.float64,
                               device="cuda")
    return c


def _eval_rows(plan: Plan, rows: np.ndarray, trace: bool = False):
    """Evaluate uint8 rows [n, V] on the GPU -> (makespan, status[, starts])
    as numpy arrays. Without a trace this is one hs_eval_host call (pinned
    per-thread staging, one H2D / launch / D2H)."""
    n, V = rows.shape
    if not trace:
        rows = np.ascontiguousarray(rows, np.uint8)
        ms = np.empty(n, np.float64)
        st = np.empty(n, np.uint8)
        if n:
            plan.eval_host(rows, ms, st, None)
        return ms, st
    import torch
    ld = plan.pref_ld if V else 1
    c = _device_buffers(n, ld, V, trace)
    host = np.zeros((n, ld), np.uint8)
    host[:, :V] = rows
    with torch.cuda.stream(c.stream):
        g = c.genes[: n * ld].view(n, ld)
        g.copy_(torch.from_numpy(host), non_blocking=False)
        ms, st = c.ms[:n], c.st[:n]
        sv = c.starts[: n * V].view(n, V) if V else c.starts[:0]
        plan.trace(g, c.starts, ms, st, stream=c.stream)
        out = (ms.cpu().numpy(), st.cpu().numpy(),
               sv.cpu().numpy().reshape(n, V))
    return out


def _batch_genes(genes, V: int):
    """The one input check of every batched entry point (fitness_batch,
    argmin_batch, fitness_batch_packed, fitness_batched). A CUDA tensor
    must be uint8 [n, >=V] with unit column stride and rows that do not
    overlap (stride(0) >= shape[1]); values >= K are reported by the kernel
    (status 5, GraphError). A host array is brought to uint8 with every
    value outside [0, 255] mapped to 255, so it stays out of range (status
    5) instead of wrapping into a valid gene."""
    if hasattr(genes, "data_ptr"):  # torch tensor on the GPU
        import torch
        if genes.dtype != torch.uint8 or genes.dim() != 2 \
                or genes.shape[1] < V:
            raise GraphError("genes must be a uint8 [n, >=V] tensor")
        if genes.numel() and (genes.stride(1) != 1 or (
                genes.shape[0] > 1 and genes.stride(0) < genes.shape[1])):
            raise GraphError("genes must be row-major with non-overlapping "
                             "rows (stride(1) == 1, stride(0) >= shape[1])")
        return genes
    genes = np.asarray(genes)
    if genes.ndim != 2 or genes.shape[1] < V:
        raise GraphError("genes must be a [n, >=V] array")
    if genes.dtype != np.uint8:
        if genes.dtype.kind not in "iub":
            raise GraphError("genes must be integers")
        genes = np.where((genes < 0) | (genes > 255), 255,
                         genes).astype(np.uint8)
    return genes


def _check_genes(genes: Sequence[int], K: int) -> None:
    # heuristics.py:133-134: validated before any placement
    if any(not 0 <= int(k) < K for k in genes):
        raise GraphError("gene value out of device range")


def _raise_status(st: int) -> None:
    if st == N.ST_GENE:
        raise GraphError("gene value out of device range")
    if st == N.ST_MISSING:
        raise GraphError("missing latency entry for a reached (task, device, "
                         "batch) placement")


def decode(genome: MappingGenome, g, hw, table, L: int) -> Optional[Schedule]:
    """List-schedule the genome's mapping in its order at the earliest
    feasible start (heuristics.py:127-143), on the GPU. Returns None for
    structurally infeasible genomes."""
    _check_genes(genome.genes, len(hw.devices))
    if len(genome.order) == 0:
        return Schedule(batches=(), objective=0.0, input_count=L)
    plan = get_plan(g, hw, table, L, genome.order)
    rows = np.asarray(genome.genes, np.uint8)[None, :]
    ms, st, starts = _eval_rows(plan, rows, trace=True)
    s = int(st[0])
    _raise_status(s)
    if s != N.ST_OK:
        return None
    # the batch tuple is built on first access (_LazySchedule: a search
    # that returns decode()'s Schedule pays for its V ScheduledBatch objects
    # only when a caller reads them)
    return _LazySchedule(
        objective=float(ms[0]), input_count=L,
        lazy=(tuple(genome.order), tuple(sorted(hw.devices)),
              [int(k) for k in genome.genes], starts[0].tolist(), L,
              tuple(range(1, L + 1))))


def fitness(genome: MappingGenome, g, hw, table, L: int) -> float:
    """Makespan of the decoded genome, +inf when infeasible
    (heuristics.py:146-148)."""
    _check_genes(genome.genes, len(hw.devices))
    if len(genome.order) == 0:
        return 0.0
    plan = get_plan(g, hw, table, L, genome.order)
    ms, st = _eval_rows(plan, np.asarray(genome.genes, np.uint8)[None, :])
    _raise_status(int(st[0]))
    return float(ms[0])


# ---------------------------------------------------------------------------
# batched API

def fitness_batch(genes, g, hw, table, L: int, *,
                  order: Optional[Sequence[str]] = None,
                  return_status: bool = False, index_base: int = 0):
    """Makespans of many genomes in one launch.

    ``genes`` is a uint8 [n, >=V] array of sorted-device indices in genome
    order (BFS unless ``order``): a numpy array (host path, hs_eval_host)
    or a CUDA torch tensor (device path, hs_eval; results stay on device).
    Raises GraphError where the reference's ``fitness`` would (gene out of
    range, missing latency entry) unless ``return_status`` is set, in which
    case (makespan, status) is returned.
    """
    plan = get_plan(g, hw, table, L, order)
    genes = _batch_genes(genes, plan.V)
    if hasattr(genes, "data_ptr"):  # torch tensor on the GPU
        import torch
        n = genes.shape[0]
        plan.maybe_specialize(n)
        ms = torch.empty(n, dtype=torch.float64, device=genes.device)
        st = torch.empty(n, dtype=torch.uint8, device=genes.device)
        plan.eval(genes, ms, st, None, index_base)
        if return_status:
            return ms, st
        worst = int(st.max().item()) if n else 0
        if worst >= N.ST_MISSING:
            bad = int(torch.nonzero(st >= N.ST_MISSING)[0].item())
            _raise_status(int(st[bad].item()))
        return ms
    n = genes.shape[0]
    plan.maybe_specialize(n)
    ms = np.empty(n, np.float64)
    st = np.empty(n, np.uint8)
    plan.eval_host(genes, ms, st, None, index_base)
    if return_status:
        return ms, st
    if n and st.max() >= N.ST_MISSING:
        _raise_status(int(st[np.argmax(st >= N.ST_MISSING)]))
    return ms


def pack_genes(genes: np.ndarray) -> np.ndarray:
    """2-bit packing of uint8 genes < 4 [n, V] -> [n, ceil(ceil(V/4)/4)*4]:
    gene i in bits 2*(i%4) of byte i//4 (hs_eval_packed's layout), by the
    native host packer hs_eval_host uses (hs_pack_genes2: AVX2, thread
    pool)."""
    import ctypes as C
    if isinstance(genes, np.ndarray) and genes.dtype != np.uint8:
        if genes.size and (genes.min() < 0 or genes.max() > 3):
            raise GraphError("2-bit packing needs genes < 4")
    genes = np.asarray(genes, np.uint8)
    if genes.ndim != 2:
        raise GraphError("pack_genes: genes must be [n, V]")
    if genes.strides[1] != 1 or genes.strides[0] < genes.shape[1]:
        genes = np.ascontiguousarray(genes)
    n, V = genes.shape
    pld = ((V + 3) // 4 + 3) // 4 * 4
    out = np.zeros((n, pld), np.uint8)
    if n == 0 or V == 0:
        return out
    ok = C.c_int32(0)
    N.check(N.load().hs_pack_genes2(genes.ctypes.data, n, genes.strides[0], V,
                                    4, out.ctypes.data, pld, C.byref(ok)),
            "pack_genes")
    if not ok.value:
        raise GraphError("2-bit packing needs genes < 4")
    return out


def pack_genes3(genes: np.ndarray) -> np.ndarray:
    """Base-3 packing of uint8 genes < 3 [n, V] -> [n, ceil(V/5)]: byte j =
    sum_d gene[5j+d] * 3**d (hs_eval_packed3's layout, 1.6 bits per gene)."""
    genes = np.asarray(genes, np.uint8)
    n, V = genes.shape
    if genes.size and genes.max() > 2:
        raise GraphError("base-3 packing needs genes < 3")
    pld = (V + 4) // 5
    g = np.zeros((n, pld * 5), np.uint8)
    g[:, :V] = genes
    g = g.reshape(n, pld, 5)
    return (g[:, :, 0] + 3 * g[:, :, 1] + 9 * g[:, :, 2] + 27 * g[:, :, 3]
            + 81 * g[:, :, 4]).astype(np.uint8)


def fitness_batch_packed(packed, g, hw, table, L: int, *,
                         return_status: bool = False, radix: int = 4):
    """fitness_batch for packed genomes: `radix` 4 = 2-bit (pack_genes),
    3 = base-3 (pack_genes3). numpy -> host path (a quarter / a fifth of
    the PCIe bytes), CUDA tensor -> device path."""
    if radix not in (3, 4):
        raise ValueError("radix must be 3 or 4")
    plan = get_plan(g, hw, table, L)
    # bytes a packed row needs (2-bit: ceil(V/4); base 3: ceil(V/5))
    packed = _batch_genes(packed, (plan.V + 3) // 4 if radix == 4
                          else plan.packed3_ld())
    n = int(packed.shape[0])
    plan.maybe_specialize(n)
    if hasattr(packed, "data_ptr"):
        import torch
        ms = torch.empty(n, dtype=torch.float64, device=packed.device)
        st = torch.empty(n, dtype=torch.uint8, device=packed.device)
        (plan.eval_packed if radix == 4 else plan.eval_packed3)(packed, ms, st)
        if return_status:
            return ms, st
        if n and int(st.max().item()) >= N.ST_MISSING:
            _raise_status(int(st.max().item()))
        return ms
    packed = np.ascontiguousarray(packed, np.uint8)
    ms = np.empty(n, np.float64)
    st = np.empty(n, np.uint8)
    if n:
        (plan.eval_host_packed if radix == 4
         else plan.eval_host_packed3)(packed, ms, st)
    if return_status:
        return ms, st
    if n and st.max() >= N.ST_MISSING:
        _raise_status(int(st.max()))
    return ms


def specialize(g, hw, table, L: int, order=None) -> float:
    """Compile the graph-specialised evaluator for this instance on the
    current device (csrc/jit.cpp); returns the compile time in ms."""
    return get_plan(g, hw, table, L, order).specialize()


def throughput(makespan, L: int):
    """Inputs per second, 1000 * L / makespan (cli.py:154, bounds.py:234);
    +inf where the makespan is 0 (the reference prints no throughput)."""
    m = np.asarray(makespan, np.float64)
    with np.errstate(divide="ignore"):
        out = (1000.0 * L) / m
    return np.where(m > 0, out, INF)


def argmin_batch(genes, g, hw, table, L: int, *,
                 order: Optional[Sequence[str]] = None,
                 index_base: int = 0) -> tuple[float, int]:
    """(makespan, index) of the first best genome (numpy.argmin semantics,
    +inf allowed) computed by the fused on-device reduction."""
    plan = get_plan(g, hw, table, L, order)
    genes = _batch_genes(genes, plan.V)
    n = int(genes.shape[0])
    plan.maybe_specialize(n)
    if hasattr(genes, "data_ptr"):
        import torch
        best = torch.empty(2, dtype=torch.int64, device=genes.device)
        st = torch.empty(n, dtype=torch.uint8, device=genes.device)
        plan.eval(genes, None, st, best, index_base)
        # the reference's fitness raises on these (GraphError), it does not
        # score them +inf
        if n and int(st.max().item()) >= N.ST_MISSING:
            bad = int(torch.nonzero(st >= N.ST_MISSING)[0].item())
            _raise_status(int(st[bad].item()))
        b = best.cpu()
        return float(b[:1].view(torch.float64).item()), int(b[1].item())
    b = N.Best()
    st = np.empty(n, np.uint8)
    plan.eval_host(genes, None, st, b, index_base)
    if n and st.max() >= N.ST_MISSING:
        _raise_status(int(st[np.argmax(st >= N.ST_MISSING)]))
    return float(b.cost), int(b.index)


def random_search(g, hw, table, L: int, n: int, *, seed: int = 0,
                  first: int = 0, chunk: int = 1 << 26):
    """Evaluate n on-device generated genomes (oracle gen_genes(seed, c) for
    c in [first, first + n)) and return (best makespan, index, genome)."""
    import torch
    plan = get_plan(g, hw, table, L)
    plan.maybe_specialize(n)
    bests = []
    dbest = torch.empty(2, dtype=torch.int64, device="cuda")
    for lo in range(first, first + n, chunk):
        m = min(chunk, first + n - lo)
        plan.eval_gen(N.GEN_RANDOM, seed, lo, m, best=dbest)
        b = dbest.cpu()
        bests.append((float(b[:1].view(torch.float64).item()),
                      int(b[1].item())))
    cost, idx = min(bests, key=lambda t: (t[0], t[1])) if bests \
        else (INF, -1)
    genome = None
    if idx >= 0:
        out = torch.empty((1, plan.V), dtype=torch.uint8, device="cuda")
        plan.eval_gen(N.GEN_RANDOM, seed, idx, 1, genes_out=out)
        genome = MappingGenome(genes=tuple(int(x) for x in out.cpu()[0]),
                               order=plan.order)
    return cost, idx, genome


# ---------------------------------------------------------------------------
# baseline heuristics

def best_device(g, hw, table, L: int) -> Schedule:
    """Whole graph serially on the single fastest device
    (heuristics.py:151-167)."""
    best = None
    for u in sorted(hw.devices):
        if L not in hw.devices[u].batch_sizes:
            continue
        total = sum(table.get(i, u, L) for i in g.tasks)
        if best is None or total < best[0] - 1e-12:
            best = (total, u)
    if best is None:
        raise ScheduleError(f"no device supports batch size {L}")
    s = decode(genome_from_map(g, hw, {i: best[1] for i in g.tasks}),
               g, hw, table, L)
    if s is None:
        raise ScheduleError(f"device {best[1]!r} cannot hold the whole graph")
    return s


def _met_mapping(g, hw, table, L: int) -> dict:
    mapping = {}
    devs = sorted(hw.devices)
    for i in g.tasks:
        best = None
        for u in devs:
            if L not in hw.devices[u].batch_sizes:
                continue
            ms = table.get(i, u, L)
            if best is None or ms < best[0] - 1e-12:
                best = (ms, u)
        if best is None:
            raise ScheduleError(f"no device supports batch size {L}")
        mapping[i] = best[1]
    return mapping


def met(g, hw, table, L: int) -> Schedule:
    """Each task on its minimum-execution-time device, ties to the smallest
    device id (heuristics.py:170-189)."""
    s = decode(genome_from_map(g, hw, _met_mapping(g, hw, table, L)),
               g, hw, table, L)
    if s is None:
        raise ScheduleError("MET mapping infeasible (missing links or memory)")
    return s


class _HostScheduler:
    """Host restatement of the non-insertion list scheduler for the K-way
    greedy choice (heuristics.py:43-124); per-step work is O(K * preds)."""

    def __init__(self, g, hw, table, L: int):
        self.g, self.hw, self.table, self.L = g, hw, table, L
        self.avail = {u: 0.0 for u in hw.devices}
        self.mem = {u: 0.0 for u in hw.devices}
        self.end: dict[str, tuple[str, float]] = {}
        self.batches: list[ScheduledBatch] = []
        self.makespan = 0.0

    def try_place(self, task: str, dev: str):
        node = self.g.tasks[task]
        d = self.hw.devices[dev]
        if self.L not in d.batch_sizes:
            return None
        extra = (node.im + node.om) * self.L
        extra += node.wm
        if self.mem[dev] + extra > d.memory + 1e-9:
            return None
        ready = 0.0
        for p in self.g.pred[task]:
            src, e = self.end[p]
            c = self.hw.comm_time(self.g.tasks[p].om, src, dev)
            if c is None:
                return None
            x = e + c
            if x > ready:
                ready = x
        dur = self.table.get(task, dev, self.L)
        a = self.avail[dev]
        start = a if a > ready else ready
        return start, start + dur, extra

    def commit(self, task, dev, start, end, extra):
        self.avail[dev] = end
        self.mem[dev] += extra
        self.end[task] = (dev, end)
        self.batches.append(ScheduledBatch(
            task=task, device=dev, size=self.L,
            inputs=tuple(range(1, self.L + 1)), start=start))
        if end > self.makespan:
            self.makespan = end


def _greedy_native(g, hw, table, L: int):
    """(plan, genes uint8 [V], starts [V], makespan) of greedy from the
    native scheduler over the plan's tables (hs_plan_greedy), or None when
    the case is left to the host scheduler (NaN-capable cost model, missing
    latency entry, infeasible task: it raises the reference's exception)."""
    import ctypes as C
    if not g.tasks:
        return None
    try:
        plan = get_plan(g, hw, table, L)
    except (GraphError, ValueError):
        return None  # the host path raises the reference's error
    genes = np.empty(plan.V, np.uint8)
    starts = np.empty(plan.V, np.float64)
    ms = C.c_double(0.0)
    rc = N.load().hs_plan_greedy(plan.handle, genes.ctypes.data,
                                 starts.ctypes.data, C.byref(ms))
    if rc == N.HS_EHOST:
        return None
    N.check(rc, "hs_plan_greedy")
    return plan, genes, starts, ms.value


def _greedy_genome(g, hw, table, L: int) -> MappingGenome:
    """SA's start genome: greedy's mapping in BFS positions."""
    r = _greedy_native(g, hw, table, L)
    if r is None:
        start = greedy(g, hw, table, L)
        return genome_from_map(g, hw, {b.task: b.device for b in start.batches})
    plan, genes, _, _ = r
    return MappingGenome(genes=tuple(genes.tolist()), order=tuple(plan.order))


def greedy(g, hw, table, L: int) -> Schedule:
    """BFS order, each task where the partial makespan grows least
    (heuristics.py:192-210): the native scheduler (hs_plan_greedy), the host
    restatement below for the cases it leaves to the host."""
    r = _greedy_native(g, hw, table, L)
    if r is not None:
        plan, genes, starts, ms = r
        devs = sorted(hw.devices)
        inputs = tuple(range(1, L + 1))
        return Schedule(batches=tuple(
            ScheduledBatch(task=t, device=devs[k], size=L, inputs=inputs,
                           start=x)
            for t, k, x in zip(plan.order, genes.tolist(), starts.tolist())),
            objective=ms, input_count=L)
    return _greedy_host(g, hw, table, L)


def _greedy_host(g, hw, table, L: int) -> Schedule:
    """Host restatement of greedy (heuristics.py:192-210)."""
    ls = _HostScheduler(g, hw, table, L)
    devs = sorted(hw.devices)
    for task in bfs_topological_order(g):
        choice = None
        for u in devs:
            spot = ls.try_place(task, u)
            if spot is None:
                continue
            cand = spot[1] if spot[1] > ls.makespan else ls.makespan
            if choice is None or cand < choice[0] - 1e-12:
                choice = (cand, u, spot)
        if choice is None:
            raise ScheduleError(f"no feasible placement for task {task!r}")
        ls.commit(task, choice[1], *choice[2])
    return Schedule(batches=tuple(ls.batches), objective=ls.makespan,
                    input_count=L)


# ---------------------------------------------------------------------------
# search loops with exact speculative GPU batches

def _fit_rows(plan: Plan, rows: np.ndarray) -> np.ndarray:
    ms, st = _eval_rows(plan, rows)
    if st.size and st.max() >= N.ST_MISSING:
        _raise_status(int(st[np.argmax(st >= N.ST_MISSING)]))
    return ms


def _gc_paused(fn):
    """Run a search loop with the cyclic garbage collector paused (and
    restored after): a full collection over torch's object graph costs
    50 ms - 1.8 s of wall time in the middle of a 10-50 ms run (measured,
    profiles/README.md r1o); cycles created meanwhile are collected later."""
    @functools.wraps(fn)
    def run(*a, **k):
        was = gc.isenabled()
        gc.disable()
        try:
            return fn(*a, **k)
        finally:
            if was:
                gc.enable()
    return run


_M64 = (1 << 64) - 1
_last_chain_stats: dict = {}  # rounds of the last K9 / K10 run (reporting)


def _sa_device_chain(plan: Plan, gen, genes: np.ndarray, cur_fit: float,
                     best_fit: float, temp: float, alpha: float, budget: int,
                     n_dev: int, window: int):
    """The whole annealing run in device launches (hs_sa_run, K10): the
    generator's PCG64 state goes to the device and comes back, so `gen` ends
    where the reference's would. Returns (best genes, best fitness)."""
    import torch
    dev = torch.device("cuda")
    bs = gen.bit_generator.state
    s, inc = int(bs["state"]["state"]), int(bs["state"]["inc"])
    words = [s & _M64, s >> 64, inc & _M64, inc >> 64]
    rng = torch.tensor(np.array(words, np.uint64).view(np.int64), device=dev)
    buf = torch.tensor(np.array([bs["has_uint32"], bs["uinteger"]],
                                np.uint32).view(np.int32), device=dev)
    f = torch.tensor([cur_fit, best_fit, temp, 0.0, 0.0],
                     dtype=torch.float64, device=dev)
    ist = torch.tensor([0, 8, 0, 0, 0, 0, 0], dtype=torch.int32, device=dev)
    d_genes = torch.from_numpy(genes.copy()).to(dev)
    d_best = torch.from_numpy(genes.copy()).to(dev)
    while True:
        plan.sa_run(d_genes, d_best, rng, buf, f, ist, alpha, n_dev, budget,
                    window)
        iv = ist.cpu().numpy()
        if iv[2] == 2:
            _raise_status(int(iv[3]))
        if iv[2] != 3:
            break
        # Metropolis too close to call on the device: CPython's exp decides
        fv = f.cpu().numpy()
        cur, bestf, tmp, cand, u = (float(x) for x in fv)
        pos, new = int(iv[4]), int(iv[5])
        acc = u < math.exp(-(cand - cur) / tmp)
        if acc:
            d_genes[pos] = new
            cur = cand
            if cand < bestf:
                bestf = cand
                d_best.copy_(d_genes)
        f.copy_(torch.tensor([cur, bestf, tmp * alpha, 0.0, 0.0],
                             dtype=torch.float64))
        ist.copy_(torch.tensor([int(iv[0]) + 1, 8, 0, 0, 0, 0, int(iv[6])],
                               dtype=torch.int32))
    _last_chain_stats["sa_rounds"] = int(ist[6].item())
    w = rng.cpu().numpy().view(np.uint64)
    b = buf.cpu().numpy().view(np.uint32)
    bs["state"]["state"] = int(w[0]) | (int(w[1]) << 64)
    bs["has_uint32"], bs["uinteger"] = int(b[0]), int(b[1])
    gen.bit_generator.state = bs
    return d_best.cpu().numpy(), float(f[1].item())


@_gc_paused
def simulated_annealing(g, hw, table, L: int, seed: int = 0,
                        budget: int = 2000, t0_fraction: float = 0.1,
                        alpha: float = 0.995, window: int = 64,
                        device_chain: bool = True) -> Schedule:
    """Single-gene reassignment, geometric cooling, Metropolis acceptance,
    greedy start, best-ever genome decoded (heuristics.py:259-299).

    Same trajectory as the reference for the same seed. Each GPU batch holds
    the candidates of the next `window` steps for every stream position the
    run can reach if those steps are rejected (a step draws ``random()`` only
    when the candidate is finite and worse, so positions branch); the host
    replays the steps against the batch until the first acceptance. With
    `device_chain` the same speculation and replay run inside one kernel
    launch (K10, hs_sa_run) with numpy's PCG64 restated on the device.
    """
    gen = np.random.default_rng(seed)
    cur = _greedy_genome(g, hw, table, L)
    cur_fit = fitness(cur, g, hw, table, L)
    best, best_fit = cur, cur_fit
    temp = max(t0_fraction * cur_fit, 1e-9)
    n_dev = len(hw.devices)
    V = len(cur.genes)
    plan = get_plan(g, hw, table, L)
    genes = np.array(cur.genes, np.uint8)
    step = 0
    if device_chain and V and budget > 0:
        best, best_fit = _sa_device_chain(plan, gen, genes, cur_fit, best_fit,
                                          temp, alpha, budget, n_dev,
                                          max(window, 128))
        step = budget
    k = max(1, min(window, 8))
    while step < budget:
        k = min(k, budget - step)
        S, st0 = R.peek(gen, 4 * k + 64)

        def draw(st):
            pos, st = S.integers(st, V)
            old = int(genes[pos])
            if n_dev > 1:
                new, st = S.integers(st, n_dev - 1)
                if new >= old:
                    new += 1
            else:
                new = old
            return pos, new, st

        # candidates for every state reachable through rejected steps
        cand: dict[tuple, tuple] = {}
        frontier = {st0}
        try:
            for _ in range(k):
                nxt = set()
                for s in frontier:
                    if s not in cand:
                        pos, new, s2 = draw(s)
                        cand[s] = (pos, new, s2)
                    s2 = cand[s][2]
                    nxt.add(s2)
                    nxt.add(S.next64(s2)[1])
                frontier = nxt
        except IndexError:  # ran out of peeked words: shorter window
            pass
        keys = list(cand)
        rows = np.repeat(genes[None, :], len(keys), axis=0)
        for r, s in enumerate(keys):
            pos, new, _ = cand[s]
            rows[r, pos] = new
        fits, sts = _eval_rows(plan, rows)
        fit_of = {s: float(fits[r]) for r, s in enumerate(keys)}
        st_of = {s: int(sts[r]) for r, s in enumerate(keys)}
        # replay the reference's steps
        s = st0
        accepted = False
        for _ in range(k):
            if s not in cand:
                break
            pos, new, s2 = cand[s]
            if st_of[s] >= N.ST_MISSING:  # the reference's fitness raises
                _raise_status(st_of[s])
            cand_fit = fit_of[s]
            delta = cand_fit - cur_fit
            accept = delta <= 0
            s = s2
            if not accept and math.isfinite(cand_fit):
                u, s = S.random(s)
                accept = u < math.exp(-delta / temp)
            step += 1
            if accept:
                genes = genes.copy()
                genes[pos] = new
                cur_fit = cand_fit
                if cand_fit < best_fit:
                    best, best_fit = genes.copy(), cand_fit
                accepted = True
            temp *= alpha
            if accepted:
                break
        R.commit(gen, s)
        k = 8 if accepted else min(window, 2 * k)
    best_genes = best.genes if isinstance(best, MappingGenome) \
        else tuple(int(x) for x in best)
    out = decode(MappingGenome(genes=tuple(best_genes), order=cur.order),
                 g, hw, table, L)
    assert out is not None
    return out


def _pcg_words(seed: int):
    """(PCG64 state words [4], buffered uint32 [2]) of default_rng(seed)."""
    bs = np.random.PCG64(seed).state  # == default_rng(seed)'s, 8x cheaper
    s, inc = int(bs["state"]["state"]), int(bs["state"]["inc"])
    return ([s & _M64, s >> 64, inc & _M64, inc >> 64],
            [bs["has_uint32"], bs["uinteger"]])


class _LazySchedule(Schedule):
    """A Schedule whose ScheduledBatch tuple is built on first access.

    The multi-chain searches decode 148 genomes in one trace launch; making
    148 x V ScheduledBatch objects up front (~30 K for WS200) cost more host
    time than the search kernel itself, and a caller usually reads only
    the objectives to pick the best restart. Equal to (and hashing like)
    the eager Schedule with the same fields."""

    def __init__(self, batches=None, objective: float = 0.0,
                 input_count: int = 1, flags: tuple = (), *, lazy=None):
        object.__setattr__(self, "objective", objective)
        object.__setattr__(self, "input_count", input_count)
        object.__setattr__(self, "flags", flags)
        object.__setattr__(self, "_batches", batches)
        object.__setattr__(self, "_lazy", lazy)

    @property
    def batches(self):
        b = self.__dict__["_batches"]
        if b is None:
            order, devs, genes, starts, size, inputs = self.__dict__["_lazy"]
            b = tuple(ScheduledBatch(task=t, device=devs[k], size=size,
                                     inputs=inputs, start=x)
                      for t, k, x in zip(order, genes, starts))
            object.__setattr__(self, "_batches", b)
            object.__setattr__(self, "_lazy", None)
        return b

    def _key(self):
        return (self.batches, self.objective, self.input_count, self.flags)

    def __eq__(self, other):
        if isinstance(other, Schedule):
            return self._key() == (other.batches, other.objective,
                                   other.input_count, other.flags)
        return NotImplemented

    def __hash__(self):
        return hash(self._key())

    def __repr__(self):
        return (f"Schedule(batches={self.batches!r}, objective="
                f"{self.objective!r}, input_count={self.input_count!r}, "
                f"flags={self.flags!r})")

    def __reduce__(self):  # pickles as a plain Schedule
        return (Schedule, self._key())


def _decode_rows(plan: Plan, g, hw, table, L: int, rows: np.ndarray) -> list:
    """Schedules of many genomes in one trace launch (as decode()); their
    batch tuples are built on first access (_LazySchedule)."""
    ms, st, starts = _eval_rows(plan, rows, trace=True)
    devs = tuple(sorted(hw.devices))
    inputs = tuple(range(1, L + 1))
    order = tuple(plan.order)
    out = []
    for r in range(len(rows)):
        _raise_status(int(st[r]))
        if int(st[r]) != N.ST_OK:
            out.append(None)
            continue
        out.append(_LazySchedule(
            objective=float(ms[r]), input_count=L,
            lazy=(order, devs, rows[r].tolist(), starts[r].tolist(), L,
                  inputs)))
    return out


@_gc_paused
def simulated_annealing_multi(g, hw, table, L: int, seeds: Sequence[int],
                              budget: int = 2000, t0_fraction: float = 0.1,
                              alpha: float = 0.995,
                              window: int = 128) -> list:
    """simulated_annealing at every seed of `seeds` at once: one K10 chain
    per seed, one CTA (one SM) each, all in one launch (hs_sa_run_multi), so
    148 independent restarts take about one run's time on a B200. Element c
    is exactly ``simulated_annealing(g, hw, table, L, seed=seeds[c],
    budget=budget, ...)`` (each chain replays its own seed's PCG64 stream);
    a chain that needs the host -- a Metropolis test within a few ulp of the
    device exp, or an evaluation that raises -- is finished by the
    single-chain path. Returns the Schedules in seed order; the best restart
    is ``min(result, key=lambda s: s.objective)``."""
    import torch
    seeds = [int(s) for s in seeds]
    if not seeds:
        return []
    cur = _greedy_genome(g, hw, table, L)
    cur_fit = fitness(cur, g, hw, table, L)
    V = len(cur.genes)
    if V == 0 or budget <= 0:
        return [simulated_annealing(g, hw, table, L, seed=s, budget=budget,
                                    t0_fraction=t0_fraction, alpha=alpha)
                for s in seeds]
    temp = max(t0_fraction * cur_fit, 1e-9)
    n_dev = len(hw.devices)
    plan = get_plan(g, hw, table, L)
    C = len(seeds)
    stride = -(-V // 16) * 16
    rows = np.zeros((C, stride), np.uint8)
    rows[:, :V] = np.asarray(cur.genes, np.uint8)
    rng = np.zeros((C, 4), np.uint64)
    buf = np.zeros((C, 2), np.uint32)
    for c, s in enumerate(seeds):
        w, b = _pcg_words(s)
        rng[c] = w
        buf[c] = b
    f = np.zeros((C, 8), np.float64)
    f[:, 0] = f[:, 1] = cur_fit
    f[:, 2] = temp
    ist = np.zeros((C, 8), np.int32)
    ist[:, 1] = 8
    dev = torch.device("cuda")
    d_genes = torch.from_numpy(rows).to(dev)
    d_best = d_genes.clone()
    d_rng = torch.from_numpy(rng.view(np.int64)).to(dev)
    d_buf = torch.from_numpy(buf.view(np.int32)).to(dev)
    d_f = torch.from_numpy(f).to(dev)
    d_ist = torch.from_numpy(ist).to(dev)
    plan.sa_run_multi(C, d_genes, d_best, d_rng, d_buf, d_f, d_ist, alpha,
                      n_dev, budget, max(window, 128))
    iv = d_ist.cpu().numpy()
    best = np.ascontiguousarray(d_best.cpu().numpy()[:, :V])
    _last_chain_stats["sa_multi_rounds"] = [int(x) for x in iv[:, 6]]
    out = _decode_rows(plan, g, hw, table, L, best)
    for c in range(C):
        if iv[c, 2] != 0 or out[c] is None:
            out[c] = simulated_annealing(g, hw, table, L, seed=seeds[c],
                                         budget=budget,
                                         t0_fraction=t0_fraction, alpha=alpha)
    return out


def _ea_draw_chunk(gen, steps: int, V: int, n_dev: int, p: float):
    """Mutation lists of the next `steps` EA children as CSR arrays in
    pinned host memory; moves `gen` past them."""
    import torch
    need = steps * (V + 2) + 64
    while True:
        S, words, st = R.peek_words(gen, need)
        try:
            muts = R.ea_mutations(S, words, st, steps, V, n_dev, p)
            break
        except IndexError:
            need *= 2
    R.commit(gen, muts[-1][1])
    counts = np.fromiter((len(m[0]) for m in muts), np.int32, steps)
    flat = [pv for m in muts for pv in m[0]]
    moff = torch.empty(steps + 1, dtype=torch.int32, pin_memory=True)
    mn = moff.numpy()
    mn[0] = 0
    np.cumsum(counts, out=mn[1:])
    mpos = torch.empty(max(len(flat), 1), dtype=torch.int32, pin_memory=True)
    mval = torch.empty(max(len(flat), 1), dtype=torch.uint8, pin_memory=True)
    if flat:
        mpos.numpy()[:len(flat)] = np.fromiter((pv[0] for pv in flat), np.int32,
                                               len(flat))
        mval.numpy()[:len(flat)] = np.fromiter((pv[1] for pv in flat), np.uint8,
                                               len(flat))
    return moff, mpos[:len(flat)], mval[:len(flat)]


def _ea_draw_device(states, V: int, n_dev: int, p: float, budget: int):
    """K12 (hs_ea_draw): the mutation lists of `budget` EA children for
    every generator state in `states` [(words[4], buf[2])], drawn on the
    device. Returns (moff [C, budget+1] absolute, mpos, mval, status [C])
    as device tensors; status != 0 marks a chain the host must redraw."""
    import torch
    from . import _native as NN
    C = len(states)
    dev = torch.device("cuda")
    rng = torch.from_numpy(np.array([w for w, _ in states], np.uint64)
                           .view(np.int64)).to(dev)
    buf = torch.from_numpy(np.array([b for _, b in states], np.uint32)
                           .view(np.int32)).to(dev)
    cap = 4 * budget + 256
    moff = torch.empty((C, budget + 1), dtype=torch.int32, device=dev)
    mpos = torch.empty(C * cap, dtype=torch.int32, device=dev)
    mval = torch.empty(C * cap, dtype=torch.uint8, device=dev)
    status = torch.empty(C, dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream()
    NN.check(NN.load().hs_ea_draw(
        C, rng.data_ptr(), buf.data_ptr(), V, n_dev, float(p), budget,
        moff.data_ptr(), mpos.data_ptr(), mval.data_ptr(), cap,
        status.data_ptr(), int(s.cuda_stream)), "hs_ea_draw")
    return moff, mpos, mval, status, (rng, buf)


def _gen_words(gen):
    bs = gen.bit_generator.state
    s, inc = int(bs["state"]["state"]), int(bs["state"]["inc"])
    return ([s & _M64, s >> 64, inc & _M64, inc >> 64],
            [bs["has_uint32"], bs["uinteger"]])


def _ea_device_chain(plan: Plan, gen, genes: np.ndarray, cur_fit: float,
                     budget: int, V: int, n_dev: int, p: float,
                     chunks: int = 4):
    """The accept chain on the device (K9). The mutation lists come from
    the device draw (K12) when it succeeds; otherwise the host draws them
    in `chunks` chained launches (hs_ea_run_chunk), chunk c+1's draw
    overlapping chunk c's run. Returns (genes, fitness)."""
    import torch
    dev = torch.device("cuda")
    stream = torch.cuda.current_stream()
    moff, mpos, mval, status, keep_d = _ea_draw_device(
        [_gen_words(gen)], V, n_dev, p, budget)
    d_parent = torch.from_numpy(genes.copy()).to(dev)
    d_cur = torch.tensor([cur_fit], dtype=torch.float64, device=dev)
    d_fit = torch.empty(1, dtype=torch.float64, device=dev)
    d_info = torch.empty(4, dtype=torch.int32, device=dev)
    plan.ea_run_multi(1, d_parent.view(1, -1), d_cur, moff, mpos, mval,
                      budget, d_fit, d_info, stream=stream)
    if int(status.item()) == 0:
        info = d_info.cpu().numpy()
        _last_chain_stats["ea_accepted"] = int(info[0])
        _last_chain_stats["ea_rounds"] = int(info[1])
        _last_chain_stats["ea_draw"] = "device"
        if info[2] >= 0:
            _raise_status(int(info[3]))
        return d_parent.cpu().numpy(), float(d_fit.cpu()[0])
    del keep_d
    _last_chain_stats["ea_draw"] = "host"
    d_parent = torch.from_numpy(genes.copy()).to(dev)
    d_fit = torch.tensor([cur_fit], dtype=torch.float64, device=dev)
    d_info = torch.tensor([0, 0, -1, 0], dtype=torch.int32, device=dev)
    size = -(-budget // max(1, chunks))
    keep = []  # device copies must outlive their (asynchronous) launches
    first = 0
    while first < budget:
        n = min(size, budget - first)
        moff, mpos, mval = _ea_draw_chunk(gen, n, V, n_dev, p)
        d = [x.to(dev, non_blocking=True) for x in (moff, mpos, mval)]
        keep.append((moff, mpos, mval, d))
        plan.ea_run_chunk(d_parent, d_fit, d[0], d[1], d[2], n, first, d_info,
                          stream=stream)
        first += n
    info = d_info.cpu().numpy()
    _last_chain_stats["ea_accepted"] = int(info[0])
    _last_chain_stats["ea_rounds"] = int(info[1])
    if info[2] >= 0:
        _raise_status(int(info[3]))
    return d_parent.cpu().numpy(), float(d_fit.cpu()[0])


@_gc_paused
def one_plus_one_ea_multi(g, hw, table, L: int, seeds: Sequence[int],
                          budget: int = 2000, biased: bool = True) -> list:
    """one_plus_one_ea at every seed of `seeds` at once: each seed's
    mutation stream drawn on the device (K12), then one K9 accept chain per
    seed, one CTA (one SM) each, in one launch (hs_ea_run_multi). Element c
    is exactly ``one_plus_one_ea(g, hw, table, L, seed=seeds[c], budget=
    budget, biased=biased)``; a chain whose draw needs the host, or whose
    evaluation raises, is finished by the single-chain path."""
    import torch
    seeds = [int(s) for s in seeds]
    if not seeds:
        return []
    order = tuple(bfs_topological_order(g))
    n_dev = len(hw.devices)
    V = len(order)
    if V == 0 or budget <= 0:
        return [one_plus_one_ea(g, hw, table, L, seed=s, budget=budget,
                                biased=biased) for s in seeds]
    plan = get_plan(g, hw, table, L)
    C = len(seeds)
    stride = -(-V // 16) * 16
    rows = np.zeros((C, stride), np.uint8)
    states = []
    if biased:
        start = genome_from_map(g, hw, _met_mapping(g, hw, table, L))
        ms0, st0 = _eval_rows(get_plan(g, hw, table, L, start.order),
                              np.asarray(start.genes, np.uint8)[None, :])
        _raise_status(int(st0[0]))
        if int(st0[0]) != N.ST_OK:  # as met() raises
            raise ScheduleError("MET mapping infeasible (missing links or memory)")
        rows[:, :V] = np.asarray(start.genes, np.uint8)
        fits = np.full(C, float(ms0[0]))
        # default_rng(s)'s state without a Generator per seed
        states = [_pcg_words(s) for s in seeds]
    else:
        for c, s in enumerate(seeds):
            gen = np.random.default_rng(s)
            rows[c, :V] = gen.integers(n_dev, size=V)
            states.append(_gen_words(gen))
        fits = _fit_rows(plan, np.ascontiguousarray(rows[:, :V]))
    p = 1.0 / max(V, 1)
    moff, mpos, mval, status, keep_d = _ea_draw_device(states, V, n_dev, p,
                                                       budget)
    dev = torch.device("cuda")
    d_parent = torch.from_numpy(rows).to(dev)
    d_cur = torch.from_numpy(fits.astype(np.float64)).to(dev)
    d_fit = torch.empty(C, dtype=torch.float64, device=dev)
    d_info = torch.empty((C, 4), dtype=torch.int32, device=dev)
    plan.ea_run_multi(C, d_parent, d_cur, moff, mpos, mval, budget, d_fit,
                      d_info)
    info = d_info.cpu().numpy()
    st = status.cpu().numpy()
    final = np.ascontiguousarray(d_parent.cpu().numpy()[:, :V])
    del keep_d
    _last_chain_stats["ea_multi_rounds"] = [int(x) for x in info[:, 1]]
    out = _decode_rows(plan, g, hw, table, L, final)
    for c in range(C):
        if st[c] != 0 or info[c, 2] >= 0 or out[c] is None:
            out[c] = one_plus_one_ea(g, hw, table, L, seed=seeds[c],
                                     budget=budget, biased=biased)
    return out


@_gc_paused
def one_plus_one_ea(g, hw, table, L: int, seed: int = 0, budget: int = 2000,
                    biased: bool = True, window: int = 256,
                    device_chain: bool = True) -> Schedule:
    """(1+1) EA: each gene mutated with probability 1/|V|, accept when not
    worse; biased start = MET, unbiased = uniform genes
    (heuristics.py:302-334). The mutation stream does not depend on fitness,
    so every child's mutation list is drawn ahead. With `device_chain` the
    whole accept chain runs in one kernel launch (K9, hs_ea_run); otherwise
    `window` children are evaluated per GPU batch and an acceptance re-bases
    the remaining children. Either way the trajectory is the reference's."""
    gen = np.random.default_rng(seed)
    order = tuple(bfs_topological_order(g))
    n_dev = len(hw.devices)
    V = len(order)
    if biased and V:
        # met()'s mapping and its feasibility from one evaluation (met()
        # itself traces and builds the Schedule, which the start discards)
        cur = genome_from_map(g, hw, _met_mapping(g, hw, table, L))
        ms0, st0 = _eval_rows(get_plan(g, hw, table, L, cur.order),
                              np.asarray(cur.genes, np.uint8)[None, :])
        _raise_status(int(st0[0]))
        if int(st0[0]) != N.ST_OK:
            raise ScheduleError("MET mapping infeasible (missing links or memory)")
        cur_fit = float(ms0[0])
    else:
        if biased:
            cur = genome_from_map(g, hw, {b.task: b.device for b in
                                          met(g, hw, table, L).batches})
        else:
            cur = MappingGenome(
                genes=tuple(int(v) for v in gen.integers(n_dev, size=V)),
                order=order)
        cur_fit = fitness(cur, g, hw, table, L)
    p = 1.0 / max(V, 1)
    genes = np.array(cur.genes, np.uint8)
    plan = get_plan(g, hw, table, L) if V else None
    step = 0
    if device_chain and V and budget > 0:
        genes, cur_fit = _ea_device_chain(plan, gen, genes, cur_fit, budget,
                                          V, n_dev, p)
        step = budget
    while step < budget:
        k = min(window, budget - step)
        S, words, st = R.peek_words(gen, k * (V + 2) + 64)
        try:
            muts = R.ea_mutations(S, words, st, k, V, n_dev, p)
        except IndexError:
            muts = []
            for kk in (k // 2, k // 4, 1):
                try:
                    muts = R.ea_mutations(S, words, st, max(kk, 1), V, n_dev,
                                          p)
                    break
                except IndexError:
                    continue
        if not muts:
            raise RuntimeError("RNG peek window too small")
        j = 0
        while j < len(muts):
            rows = np.repeat(genes[None, :], len(muts) - j, axis=0)
            for r in range(j, len(muts)):
                for pos, val in muts[r][0]:
                    rows[r - j, pos] = val
            if V:
                fits, sts = _eval_rows(plan, rows)
            else:
                fits, sts = np.zeros(len(rows)), np.zeros(len(rows), np.uint8)
            acc = None
            for r in range(len(rows)):
                if sts[r] >= N.ST_MISSING:  # the reference's fitness raises
                    _raise_status(int(sts[r]))
                if fits[r] <= cur_fit:
                    acc = r
                    break
            if acc is None:
                j = len(muts)
                break
            genes = rows[acc].copy()
            cur_fit = float(fits[acc])
            j += acc + 1
        step += len(muts)
        R.commit(gen, muts[-1][1])
    final = decode(MappingGenome(genes=tuple(int(x) for x in genes),
                                 order=order), g, hw, table, L)
    if final is None:
        raise ScheduleError("EA produced an infeasible genome")
    return final
