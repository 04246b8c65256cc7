"""The split heuristic (MILP-SPLIT) on the B200 path: module detection,
the GPU module solver, and the dynamic program that combines them.

* ``find_bridges_and_articulation_points`` / ``k_edge_components``
  (reference splitting.py:36-81, 178-219) run natively (csrc/decomp.cpp,
  C ABI ``hs_bridges_articulation`` / ``hs_k_edge_components``) and return
  the reference's ``ModuleDecomposition`` shape (modules in the same
  lexicographic topological order, cut edges in edge order).
* ``gpu_module_solver`` fills the reference's pluggable ``ModuleSolver``
  slot (splitting.py:225), called as ``solver(sub, hw, table, L, pins,
  same_device, timeout)`` and returning ``(objective, schedule,
  proven_optimal)`` or ``(None, None, False)`` (splitting.py:228-245,
  338-340). It sweeps the module's mappings on the B200 -- exhaustively when
  the free assignments number at most ``exhaustive_limit``, otherwise by
  on-device random sampling followed by batched best-improvement 1-opt --
  with pinned tasks fixed and ``same_device`` pairs tied (milp.py:277-291),
  and returns the decoded schedule of the best mapping. The objective is the
  list-scheduling makespan, so ``proven_optimal`` is False (optimal over
  decoder mappings, not a MILP certificate); the DP then flags the result
  quasi-optimal. It is thread-safe (the DP may call it from a thread pool).
* ``milp_split`` is the reference's DP over channel-endpoint device pinnings
  (splitting.py:259-402) with the same states, tie rules and flags; its
  default module solver here is ``gpu_module_solver`` (this package has no
  MILP: the reference's ``default_module_solver`` stays a CPU consumer that
  can be passed in).
"""
from __future__ import annotations

import ctypes as C
import itertools
import json
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np

from . import _native as N
from .core import GraphError, Schedule, ScheduledBatch, ScheduleError
from .heuristics import MappingGenome, decode, _fit_rows
from .plan import _strings, get_plan

MAX_PIN_TASKS = 4


# ---------------------------------------------------------------------------
# module detection (native)

def _edge_arrays(g):
    ids = list(g.tasks)
    tix = {t: k for k, t in enumerate(ids)}
    src = np.array([tix[a] for a, _ in g.edges], np.int32)
    dst = np.array([tix[b] for _, b in g.edges], np.int32)
    return ids, src, dst


def find_bridges_and_articulation_points(g):
    """(bridges in edge order and orientation, articulation set, connected)
    of the undirected shadow (reference splitting.py:36-81)."""
    lib = N.load()
    ids, src, dst = _edge_arrays(g)
    br = np.zeros(max(len(src), 1), np.uint8)
    art = np.zeros(max(len(ids), 1), np.uint8)
    conn = C.c_int32()
    N.check(lib.hs_bridges_articulation(
        len(ids), len(src), src.ctypes.data, dst.ctypes.data, br.ctypes.data,
        art.ctypes.data, C.byref(conn)), "hs_bridges_articulation")
    bridges = [e for e, b in zip(g.edges, br) if b]
    return bridges, {t for t, a in zip(ids, art) if a}, bool(conn.value)


@dataclass
class ModuleDecomposition:
    """Same shape and methods as the reference's (splitting.py:134-175)."""
    modules: list  # topologically ordered partition of V (frozensets)
    cut_edges: dict  # (from module, to module) -> [(src, dst)] edge order
    channels: int
    is_chain: bool

    def module_of(self) -> dict:
        return {t: k for k, mod in enumerate(self.modules) for t in mod}

    def in_edges(self, t: int) -> list:
        return [(a, e) for (a, b), es in self.cut_edges.items() if b == t
                for e in es]

    def max_cut_width(self) -> int:
        return max((len(e) for e in self.cut_edges.values()), default=0)

    def to_json(self) -> str:
        return json.dumps({
            "channels": self.channels, "is_chain": self.is_chain,
            "modules": [sorted(m) for m in self.modules],
            "cuts": [{"from": a, "to": b, "edges": [list(e) for e in es]}
                     for (a, b), es in sorted(self.cut_edges.items())],
        }, indent=2) + "\n"

    @classmethod
    def from_json(cls, text: str) -> "ModuleDecomposition":
        doc = json.loads(text)
        try:
            return cls(modules=[frozenset(m) for m in doc["modules"]],
                       cut_edges={(int(c["from"]), int(c["to"])):
                                  [(e[0], e[1]) for e in c["edges"]]
                                  for c in doc["cuts"]},
                       channels=int(doc["channels"]),
                       is_chain=bool(doc["is_chain"]))
        except (KeyError, TypeError, IndexError) as exc:
            raise GraphError(f"bad decomposition document: {exc}") from exc


def k_edge_components(g, c: int = 1) -> ModuleDecomposition:
    """Modules = (c+1)-edge-connected components of the undirected shadow,
    cycles merged, in the reference's lexicographic topological order
    (splitting.py:178-219); computed by hs_k_edge_components."""
    if c < 1:
        raise GraphError("channel budget c must be >= 1")
    lib = N.load()
    ids, src, dst = _edge_arrays(g)
    raw, off = _strings(ids)
    mod = np.zeros(max(len(ids), 1), np.int32)
    nm = C.c_int32()
    N.check(lib.hs_k_edge_components(
        len(ids), raw, off.ctypes.data, len(src), src.ctypes.data,
        dst.ctypes.data, int(c) + 1, mod.ctypes.data, C.byref(nm)),
        "hs_k_edge_components")
    groups: list = [[] for _ in range(nm.value)]
    for t, m in zip(ids, mod):
        groups[m].append(t)
    module_of = dict(zip(ids, (int(m) for m in mod)))
    cuts: dict = {}
    for a, b in g.edges:
        ma, mb = module_of[a], module_of[b]
        if ma != mb:
            cuts.setdefault((ma, mb), []).append((a, b))
    return ModuleDecomposition(
        modules=[frozenset(x) for x in groups], cut_edges=cuts, channels=c,
        is_chain=all(b == a + 1 for (a, b) in cuts))

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
                      starts: int = 8, pair_moves: bool = True,
                      seed: int = 0) -> ModuleSolver:
    """Build a ModuleSolver (see module docstring). `objective` is accepted
    for signature parity: latency and throughput share the makespan
    (milp.py:144-146). Sampled modules are refined by a batched multi-start
    local search: the `starts` best samples move together, each round
    evaluating every single-group and (with `pair_moves`) every two-group
    reassignment of every incumbent in one GPU batch, until none improves."""
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
        pool = []  # (cost, index) of the best samples (random mode)
        ms_buf = torch.empty(min(chunk, total), dtype=torch.float64,
                             device="cuda") if mode == N.GEN_RANDOM else None
        for lo in range(0, total, chunk):
            m = min(chunk, total - lo)
            plan.eval_gen(mode, seed, lo, m, template=d_t, group=d_g,
                          n_groups=ng, best=best,
                          makespan=ms_buf[:m] if ms_buf is not None else None)
            b = best.cpu()
            c = (float(b[:1].view(torch.float64).item()), int(b[1].item()))
            if c < found:
                found = c
            if ms_buf is not None and starts > 1:
                k = min(starts, m)
                v, ix = torch.topk(ms_buf[:m], k, largest=False, sorted=True)
                pool += [(float(a), lo + int(j)) for a, j in
                         zip(v.cpu().tolist(), ix.cpu().tolist())]
            if deadline is not None and time.monotonic() > deadline:
                break
        if found[1] < 0:
            return None, None, False
        idx = [found[1]]
        if pool:
            pool.sort()
            idx = [j for c, j in pool[:starts] if np.isfinite(c)] or idx
        rows = np.empty((len(idx), V), np.uint8)
        out = torch.empty((1, V), dtype=torch.uint8, device="cuda")
        for r, j in enumerate(idx):
            plan.eval_gen(mode, seed, j, 1, template=d_t, group=d_g,
                          n_groups=ng, genes_out=out)
            rows[r] = out.cpu().numpy()[0]
        genes = rows[0].copy()
        cost = found[0]
        if mode == N.GEN_RANDOM and np.isfinite(cost):
            genes, cost = _refine_multi(plan, rows, group, K, refine_rounds,
                                        pair_moves, deadline)
        if not np.isfinite(cost):
            return None, None, False
        sched = decode(MappingGenome(genes=tuple(int(x) for x in genes),
                                     order=plan.order), sub, hw, table, L)
        if sched is None:
            return None, None, False
        return sched.objective, sched, False

    return solver


def _refine_multi(plan, rows, group, K, rounds, pairs, deadline):
    """Best-improvement local search of several incumbents: each round, for
    every incumbent, one launch evaluates all of its one-group and (with
    `pairs`) two-group reassignments, generated on the device
    (HS_GEN_NEIGHBOR) and reduced by the fused first-index argmin; the
    incumbent moves to that neighbour if it improves, else it is done.
    Returns the best (genes, cost), ties to the earlier incumbent."""
    import torch
    ng = int(group.max()) + 1 if (group >= 0).any() else 0
    inc = np.ascontiguousarray(rows, np.uint8).copy()
    cost = _fit_rows(plan, inc).astype(np.float64)
    if ng == 0:
        return inc[0].copy(), float(cost[0])
    pairs = pairs and 1 < ng <= 512
    M = ng * K + (ng * ng * K * K if pairs else 0)
    d_group = torch.from_numpy(np.ascontiguousarray(group, np.int16)).cuda()
    d_tmpl = torch.empty(inc.shape[1], dtype=torch.uint8, device="cuda")
    best = torch.empty(2, dtype=torch.int64, device="cuda")
    live = np.isfinite(cost)
    for _ in range(rounds):
        moved = False
        for s in np.flatnonzero(live):
            d_tmpl.copy_(torch.from_numpy(inc[s]))
            plan.eval_gen(N.GEN_NEIGHBOR, 0, 0, M, template=d_tmpl,
                          group=d_group, n_groups=ng, best=best)
            b = best.cpu()
            c = float(b[:1].view(torch.float64).item())
            idx = int(b[1].item())
            if idx < 0 or not c < cost[s]:
                live[s] = False
                continue
            if idx < ng * K:
                j, va, l, vb = idx // K, idx % K, -1, 0
            else:
                p = idx - ng * K
                vb = p % K
                p //= K
                va = p % K
                p //= K
                l, j = p % ng, p // ng
                if l <= j:
                    l = -1
            inc[s][group == j] = va
            if l >= 0:
                inc[s][group == l] = vb
            cost[s] = c
            moved = True
        if not moved or (deadline is not None and time.monotonic() > deadline):
            break
    b = int(np.argmin(cost))
    return inc[b].copy(), float(cost[b])


# ---------------------------------------------------------------------------
# the split DP (reference splitting.py:248-402)

def _met_device(task, hw, table, L: int) -> str:
    """Fastest device for a task at L (or its smallest batch size), ties to
    the smaller id (splitting.py:248-256)."""
    pick = None
    for u in sorted(hw.devices):
        sizes = hw.devices[u].batch_sizes
        ms = table.get(task, u, L if L in sizes else sizes[0])
        if pick is None or ms < pick[0] - 1e-12:
            pick = (ms, u)
    return pick[1]


def milp_split(g, hw, table, L: int, decomposition: ModuleDecomposition,
               module_solver: Optional[ModuleSolver] = None,
               timeout: Optional[float] = None, objective: str = "latency",
               same_device: Optional[Sequence[tuple]] = None,
               max_pins: int = MAX_PIN_TASKS,
               workers: Optional[int] = None) -> Schedule:
    """Solve every module once per device pinning of its live channel
    endpoints and chain the solutions: cost(module t, pins) = cost of the
    predecessor state + the slowest incoming channel transfer + the module's
    objective, kept per live-endpoint state, first strict improvement by
    more than 1e-12 wins (splitting.py:259-402). Same flags, states and
    assembly as the reference; `module_solver` defaults to the GPU sweep."""
    solver = module_solver if module_solver is not None \
        else gpu_module_solver(objective)
    pairs = list(same_device or ())
    mods = decomposition.modules
    T = len(mods)
    width = decomposition.max_cut_width()
    flags: set = set()
    if width > 1:
        flags.add("multi-channel")
    if not decomposition.is_chain:
        flags.add("non-chain")
    if L > 1 and width > 1:
        flags.add("quasi-optimal")
    devs = sorted(hw.devices)
    # with every pair linked a zero-byte transfer is free wherever its ends
    # sit, so such a channel needs no pinning
    mesh = all((u, v) in hw.bandwidth for u in devs for v in devs if u != v)

    def pinned(src) -> bool:
        return g.tasks[src].om > 0 or not mesh

    outs: list = [[] for _ in range(T)]   # live sources leaving module t
    ins: list = [[] for _ in range(T)]    # channel targets inside module t
    last: dict = {}                       # last module reading a source
    for (a, b), es in decomposition.cut_edges.items():
        for src, dst in es:
            if not pinned(src):
                continue
            if src not in outs[a]:
                outs[a].append(src)
            if dst not in ins[b]:
                ins[b].append(dst)
            last[src] = max(last.get(src, -1), b)
    subs = [g.subgraph(m, name=f"module{t}") for t, m in enumerate(mods)]

    def combos(tasks: list):
        if len(tasks) > max_pins:
            flags.update(("quasi-optimal", "heuristic-pinning"))
            yield {t: _met_device(t, hw, table, L) for t in tasks}
            return
        for assign in itertools.product(devs, repeat=len(tasks)):
            pins = dict(zip(tasks, assign))
            if all(not (a in pins and b in pins and pins[a] != pins[b])
                   for a, b in pairs):
                yield pins

    def solve_all(t: int) -> dict:
        choices = list(combos(sorted(set(ins[t]) | set(outs[t]))))
        local = [(a, b) for a, b in pairs if a in mods[t] and b in mods[t]]

        def one(pins):
            return solver(subs[t], hw, table, L, pins, local, timeout)

        if workers and workers > 1 and len(choices) > 1:
            with ThreadPoolExecutor(max_workers=workers) as ex:
                res = list(ex.map(one, choices))
        else:
            res = [one(p) for p in choices]
        table_t = {}
        for pins, (obj, sched, exact) in zip(choices, res):
            if obj is None:
                continue
            if not exact:
                flags.add("quasi-optimal")
            table_t[tuple(sorted(pins.items()))] = (obj, sched, pins)
        return table_t

    states: dict = {(): (0.0, [])}
    for t in range(T):
        solved = solve_all(t)
        if not solved and mods[t]:
            raise ScheduleError(f"no feasible pinning for module {t}")
        incoming = [e for _a, e in decomposition.in_edges(t) if pinned(e[0])]
        nxt: dict = {}
        for state, (cost, trail) in sorted(states.items()):
            held = dict(state)
            for _key, (obj, sched, pins) in sorted(solved.items()):
                delay, ok = 0.0, True
                for src, dst in incoming:
                    c = hw.comm_time(g.tasks[src].om, held[src], pins[dst])
                    if c is None:
                        ok = False
                        break
                    delay = max(delay, c)
                if not ok:
                    continue
                total = cost + delay + obj
                keep = {s: d for s, d in held.items() if last[s] > t}
                keep.update({s: pins[s] for s in outs[t] if last[s] > t})
                key = tuple(sorted(keep.items()))
                cur = nxt.get(key)
                if cur is None or total < cur[0] - 1e-12:
                    nxt[key] = (total, trail + [(t, sched, cost + delay)])
        if not nxt:
            raise ScheduleError(f"no feasible pinning for module {t} "
                                "(missing links)")
        states = nxt
    total, trail = states[min(states, key=lambda k: states[k][0])]
    batches = [ScheduledBatch(task=b.task, device=b.device, size=b.size,
                              inputs=b.inputs, start=b.start + off)
               for _t, sched, off in trail for b in sched.batches]
    return Schedule(batches=tuple(batches), objective=total, input_count=L,
                    flags=tuple(sorted(flags)))
