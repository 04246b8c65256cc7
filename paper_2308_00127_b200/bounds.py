"""The paper's lower bound (Section IV.B.2) on GPU building blocks -- the
drop-in for ``hetsched.bounds`` (/root/reference/pkg/src/hetsched/bounds.py).

* ``dep_subgraph`` / ``pre_subgraph`` (bounds.py:29-54) intersect the
  descendant / ancestor bitsets that one hs_reach launch computes per graph.
* ``critical_path_bound`` (bounds.py:57-72) and the batched
  ``critical_path_bounds`` run hs_cp_bound: one thread per task mask.
* ``lower_bound`` (bounds.py:142-236) is the same recursion and the same
  ``terms`` report; every critical path a level needs is computed in one
  batched launch (the reference's ``prefetch`` points). Subgraphs of at most
  ``subgraph_cap`` tasks are solved exactly by an explicit MILP sub-solver
  (``milp=``; branch and bound stays on the CPU), run
  ``workers`` at a time in a thread pool at every prefetch point like the
  reference's ``_SubgraphOpt.prefetch`` (bounds.py:126-131). Left at its
  default, ``milp`` is the reference's own MILP (``hetsched.milp``) when that
  package is installed; with ``subgraph_cap > 0`` and no sub-solver the call
  raises instead of quietly using critical paths (which is what
  ``subgraph_cap=0`` asks for).
"""
from __future__ import annotations

import json
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from .core import Device, GraphError, HardwareSystem, LatencyTable
from .plan import get_plan

DEFAULT_SUBGRAPH_CAP = 40

# reachability needs only the graph: plan it against a one-device stub
_STUB_HW = HardwareSystem([Device("_", 1.0, (1,))], {})
_STUB_TABLE = LatencyTable({})


def _graph_plan(g):
    return get_plan(g, _STUB_HW, _STUB_TABLE, 1)


_REACH_LOCK = threading.Lock()
_REACH_SETS: dict = {}


def _bits_to_set(row: np.ndarray, ids: list) -> frozenset:
    out = []
    for w, word in enumerate(row):
        word = int(word)
        while word:
            b = word & -word
            out.append(ids[w * 64 + b.bit_length() - 1])
            word ^= b
    return frozenset(out)


def _reach_sets(g):
    """({task: descendants}, {task: ancestors}) from the GPU bitsets."""
    plan = _graph_plan(g)
    key = id(plan)
    with _REACH_LOCK:
        hit = _REACH_SETS.get(key)
        if hit is not None and hit[0] is plan:
            return hit[1]
    desc, anc = plan.reach()
    ids = plan.task_ids
    res = ({t: _bits_to_set(desc[k], ids) for k, t in enumerate(ids)},
           {t: _bits_to_set(anc[k], ids) for k, t in enumerate(ids)})
    with _REACH_LOCK:
        _REACH_SETS[key] = (plan, res)
        if len(_REACH_SETS) > 64:
            _REACH_SETS.pop(next(iter(_REACH_SETS)))
    return res


def dep_subgraph(g, u: str, T) -> frozenset:
    """Tasks of T reachable from u by a directed path, u excluded."""
    return _reach_sets(g)[0][u] & frozenset(T)


def pre_subgraph(g, u: str, T) -> frozenset:
    """Tasks of T with a directed path to u, u excluded."""
    return _reach_sets(g)[1][u] & frozenset(T)


def _masks(plan, sets: Sequence) -> np.ndarray:
    tix = {t: k for k, t in enumerate(plan.task_ids)}
    words = max(plan.words, 1)
    m = np.zeros((len(sets), words), np.uint64)
    for r, s in enumerate(sets):
        for t in s:
            k = tix[t]
            m[r, k >> 6] |= np.uint64(1 << (k & 63))
    return m


def critical_path_bounds(g, hw, table, task_sets: Sequence) -> list[float]:
    """critical_path_bound for many task sets in one launch."""
    import torch
    if not task_sets:
        return []
    plan = get_plan(g, hw, table, 1)
    m = torch.from_numpy(_masks(plan, task_sets).view(np.int64)).cuda()
    out = torch.empty(len(task_sets), dtype=torch.float64, device="cuda")
    st = torch.empty(len(task_sets), dtype=torch.uint8, device="cuda")
    plan.cp_bound(m, out, st)
    st = st.cpu().numpy()
    if st.any():
        k = int(np.argmax(st))
        raise GraphError("missing latency entry for a task of subgraph "
                         f"{k} (critical_path_bound)")
    return [float(x) for x in out.cpu().numpy()]


def critical_path_bound(g, hw, table, tasks) -> float:
    """Longest path through `tasks` with each task at its fastest possible
    execution over every (device, batch size); valid for any load >= 1."""
    tasks = set(tasks)
    if not tasks:
        return 0.0
    return critical_path_bounds(g, hw, table, [tasks])[0]


@dataclass
class BoundReport:
    lower_bound_ms: float
    throughput_upper_bound: float  # inputs per second
    input_count: int
    terms: list[dict] = field(default_factory=list)

    def to_json(self) -> str:
        return json.dumps({
            "lower_bound_ms": self.lower_bound_ms,
            "throughput_upper_bound_per_s": self.throughput_upper_bound,
            "input_count": self.input_count,
            "terms": self.terms,
        }, indent=2) + "\n"


def reference_milp_solver() -> Optional[Callable]:
    """Exact sub-solver backed by the reference's MILP (milp.py:137-494):
    ``solve(sub, hw, table, load, timeout) -> (status, objective,
    dual_bound)``; None when ``hetsched`` is not installed."""
    try:
        from hetsched import milp as milp_mod  # type: ignore
    except Exception:
        return None

    def solve(sub, hw, table, load, timeout):
        res = milp_mod.solve(milp_mod.build_milp(sub, hw, table, load),
                             timeout=timeout)
        return res.status, res.objective, res.dual_bound

    return solve


class _SubgraphValues:
    """OPT or a valid lower bound per (task set, load), memoised
    (bounds.py:91-131); the critical paths of a prefetch list are one GPU
    launch and its MILP sub-solves run `workers` at a time."""

    def __init__(self, g, hw, table, timeout, cap, milp, workers):
        self.g, self.hw, self.table = g, hw, table
        self.timeout, self.cap, self.milp = timeout, cap, milp
        self.workers = workers
        self.cache: dict = {}
        self.cp: dict = {}

    def prefetch(self, items) -> None:
        todo = []
        for tasks, _load in items:
            if tasks and tasks not in self.cp and tasks not in todo:
                todo.append(tasks)
        if todo:
            for t, v in zip(todo, critical_path_bounds(
                    self.g, self.hw, self.table, todo)):
                self.cp[t] = v
        if self.milp is None or not self.workers or self.workers < 2:
            return
        solve = []
        for it in items:
            if it[0] and len(it[0]) <= self.cap and it not in self.cache \
                    and it not in solve:
                solve.append(it)
        if len(solve) > 1:
            with ThreadPoolExecutor(max_workers=self.workers) as ex:
                list(ex.map(lambda it: self.value(*it), solve))

    def value(self, tasks: frozenset, load: int):
        if not tasks:
            return 0.0, "empty"
        key = (tasks, load)
        hit = self.cache.get(key)
        if hit is not None:
            return hit
        if tasks not in self.cp:
            self.prefetch([key])
        cp = self.cp[tasks]
        if len(tasks) > self.cap:
            out = (cp, "critical-path")
        else:
            sub = self.g.subgraph(tasks)
            status, obj, dual = self.milp(sub, self.hw, self.table, load,
                                          self.timeout)
            if status == "optimal":
                out = (obj, "optimal")
            elif status == "infeasible":
                raise GraphError(f"subgraph of {len(tasks)} tasks infeasible "
                                 f"at load {load}")
            else:
                # an incumbent is no lower bound: the solver's dual bound,
                # floored by the critical path
                out = (max(cp, dual if dual is not None else 0.0),
                       "dual-bound")
        self.cache[key] = out
        return out


def _common_batch(hw) -> Optional[int]:
    common = None
    for d in hw.devices.values():
        s = set(d.batch_sizes)
        common = s if common is None else common & s
    return min(common) if common else None


def lower_bound(g, hw, table, L: int, decomposition,
                timeout: Optional[float] = None,
                subgraph_cap: int = DEFAULT_SUBGRAPH_CAP,
                workers: Optional[int] = None,
                milp: Optional[Callable] = ...) -> BoundReport:
    """max of the two paper inequalities at every cut, recursively
    (bounds.py:142-236); see the module docstring for the sub-solver.
    `milp(sub, hw, table, load, timeout) -> (status, objective, dual)`."""
    if subgraph_cap <= 0:
        milp = None
    else:
        if milp is ...:
            milp = reference_milp_solver()
        if milp is None:
            raise ValueError(
                f"lower_bound: subgraph_cap={subgraph_cap} needs an exact "
                "sub-solver for subgraphs of at most that many tasks; pass "
                "milp=... (e.g. bounds.reference_milp_solver() with the "
                "reference installed) or subgraph_cap=0 for critical paths")
    vals = _SubgraphValues(g, hw, table, timeout, subgraph_cap, milp, workers)
    modules = decomposition.modules
    T = len(modules)
    terms: list[dict] = []
    desc, anc = _reach_sets(g)

    def pre(u, S):
        return anc[u] & S

    def dep(u, S):
        return desc[u] & S

    def bound(s: int, load: int) -> float:
        if s == T - 1:
            val, kind = vals.value(modules[s], load)
            terms.append({"module": s, "load": load, "opt": val, "kind": kind})
            return val
        rest = frozenset().union(*modules[s + 1:])
        suffix = frozenset(modules[s]) | rest
        b = 1 if load == 1 else _common_batch(hw)
        if b is None or b > load:
            val = critical_path_bound(g, hw, table, suffix)
            terms.append({"module": s, "load": load, "opt": val,
                          "kind": "critical-path-fallback"})
            return val
        residual = load - b + 1
        cuts = [e for (a, _c), es in decomposition.cut_edges.items() if a == s
                for e in es]
        cut_in = sorted({tgt for _src, tgt in cuts})
        cut_out = sorted({src for src, _tgt in cuts})
        entry = sorted(v for v in rest if not (set(g.pred[v]) & rest))
        rec = {"module": s, "load": load, "batch": b, "residual": residual}

        covered = set(cut_out)
        for o in cut_out:
            covered |= pre(o, modules[s])
        if cut_in and covered == set(modules[s]):
            ins = [dep(i, rest) | {i} for i in cut_in]
            vals.prefetch([(modules[s], b)] + [(d, residual) for d in ins])
            head, head_kind = vals.value(modules[s], b)
            term1 = head + min(vals.value(d, residual)[0] for d in ins)
            rec.update({"module_opt": head, "module_opt_kind": head_kind,
                        "dep_term": term1})
        else:
            pres = [pre(v, suffix) for v in entry]
            deps = [dep(v, rest) | {v} for v in entry]
            vals.prefetch([(p, b) for p in pres] +
                          [(d, residual) for d in deps])
            term1 = min(vals.value(p, b)[0] + vals.value(d, residual)[0]
                        for p, d in zip(pres, deps))
            rec["dep_term_fallback"] = term1

        tail = bound(s + 1, b)
        if entry and set(entry) <= set(cut_in):
            pres2 = [pre(o, modules[s]) | {o} for o in cut_out]
            vals.prefetch([(p, residual) for p in pres2])
            term2 = tail + min(vals.value(p, residual)[0] for p in pres2)
            rec["pre_term"] = term2
        else:
            pres3 = [pre(v, suffix) for v in entry]
            vals.prefetch([(p, residual) for p in pres3])
            term2 = tail + (min(vals.value(p, residual)[0] for p in pres3)
                            if entry else 0.0)
            rec["pre_term_fallback"] = term2
        terms.append(rec)
        return max(term1, term2)

    lb = 0.0 if T == 0 else bound(0, L)
    tput = 1000.0 * L / lb if lb > 0 else float("inf")
    return BoundReport(lower_bound_ms=lb, throughput_upper_bound=tput,
                       input_count=L, terms=terms)
