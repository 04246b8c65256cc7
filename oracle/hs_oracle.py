"""CPU ORACLE -- test infrastructure only, never the product path.

A from-scratch restatement of the reference evaluator that the CUDA path
must match bit-for-bit. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline leg may import this module; it is the checker,
never the thing measured or shipped.

Parity of this oracle is PINNED against the golden fixtures in
``tests/golden/`` that were produced by running the reference itself
(``tests/golden/make_golden.py``); ``tests/test_oracle_golden.py`` checks it.

What is restated (reference = /root/reference/pkg/src/hetsched):

* ``bfs_order`` -- heap-Kahn on string ids, ``core.py:82-96``.
* ``Tables`` -- the per-(task, device) inputs the list scheduler reads:
  ``comm_time`` (``core.py:148-155``: 0 on the same device, no link ->
  infeasible, else ``om / beta`` IEEE division), ``LatencyTable.get`` at batch
  L (``core.py:166-170``), ``_mem_extra`` (``heuristics.py:60-65``:
  ``(im + om) * L`` then ``+ wm``), capacity ``memory + 1e-9``
  (``heuristics.py:98-100``), batch-size support (``heuristics.py:96``), and
  the device numbering ``sorted(hw.devices)`` (``heuristics.py:132``).
* ``fitness_one`` -- ``decode``/``fitness`` (``heuristics.py:127-148``) as a
  flat loop: per task in genome order try_place (``:92-106``: batch size ->
  memory -> ready_time over preds (``:67-78``) -> latency lookup), non-
  insertion slot ``max(ready, last end)`` (``:80-84``), commit (``:108-120``).
  Python ``max(a, b)`` is restated as ``b if b > a else a``.
* ``fitness_np`` -- the same recurrence vectorised over candidates (numpy,
  one node at a time in genome order, identical IEEE operations per lane).
* ``critical_path`` -- ``bounds.py:57-72``; ``reach_dep``/``reach_pre`` --
  ``bounds.py:29-54``.
* ``gen_genes`` -- the on-device candidate generator's counter hash
  (splitmix64 per candidate + a multiply-xorshift per 8 genes)
  so any generated candidate can be re-derived.

Status codes (shared with the CUDA path): 0 feasible, 1 unsupported batch
size, 2 memory, 3 missing link, 4 missing latency entry (GraphError),
5 gene out of range (GraphError).
"""
from __future__ import annotations

import heapq
import math
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

OK, ST_BATCH, ST_MEM, ST_LINK, ST_MISSING, ST_GENE = 0, 1, 2, 3, 4, 5
INF = float("inf")


def pymax(a: float, b: float) -> float:
    """Python's max(a, b) for two floats: returns a unless b > a."""
    return b if b > a else a


# ---------------------------------------------------------------- instance
@dataclass
class Instance:
    """Wire-format instance (core.py:297-356) as plain Python lists."""
    task_ids: list
    wm: list
    im: list
    om: list
    edges: list            # (a, b) id pairs, insertion order
    dev_ids: list          # insertion order
    memory: list
    batch_sizes: list      # tuple per device
    bandwidth: dict        # (a, b) -> beta
    latency: dict          # (task, dev, b) -> ms

    @classmethod
    def from_doc(cls, doc: dict) -> "Instance":
        g, hw, lat = doc["graph"], doc["hardware"], doc["latency"]
        tids = [str(t["id"]) for t in g["tasks"]]
        bw = {}
        for a, row in hw.get("bandwidth", {}).items():
            for b, v in row.items():
                bw[(a, b)] = float(v)
        ent = {}
        for t, row in lat.items():
            for d, cells in row.items():
                for b, ms in cells.items():
                    ent[(t, d, int(b))] = float(ms)
        return cls(
            task_ids=tids,
            wm=[float(t.get("wm", 0)) for t in g["tasks"]],
            im=[float(t.get("im", 0)) for t in g["tasks"]],
            om=[float(t.get("om", 0)) for t in g["tasks"]],
            edges=[(str(a), str(b)) for a, b in g.get("edges", [])],
            dev_ids=[str(d["id"]) for d in hw["devices"]],
            memory=[float(d["memory"]) for d in hw["devices"]],
            batch_sizes=[tuple(int(b) for b in d["batch_sizes"])
                         for d in hw["devices"]],
            bandwidth=bw, latency=ent)

    def succ_pred(self):
        succ = {i: [] for i in self.task_ids}
        pred = {i: [] for i in self.task_ids}
        for a, b in self.edges:
            succ[a].append(b)
            pred[b].append(a)
        return succ, pred


def bfs_order(inst: Instance) -> list:
    """Kahn's algorithm popping the smallest id first (core.py:82-96)."""
    succ, pred = inst.succ_pred()
    indeg = {i: len(pred[i]) for i in inst.task_ids}
    ready = [i for i in inst.task_ids if indeg[i] == 0]
    heapq.heapify(ready)
    out = []
    while ready:
        i = heapq.heappop(ready)
        out.append(i)
        for j in succ[i]:
            indeg[j] -= 1
            if indeg[j] == 0:
                heapq.heappush(ready, j)
    if len(out) != len(inst.task_ids):
        raise ValueError("cycle detected")
    return out


# ------------------------------------------------------------------ tables
@dataclass
class Tables:
    order: list
    devs: list             # sorted device ids: gene k -> devs[k]
    V: int
    K: int
    L: int
    preds: list            # per position: list of predecessor positions
    dur: np.ndarray        # [V, K] float64 (NaN where missing)
    dur_ok: np.ndarray     # [V, K] bool
    extra: np.ndarray      # [V] float64
    cap: np.ndarray        # [K] float64
    okL: np.ndarray        # [K] bool
    comm: np.ndarray       # [V, K, K] float64, comm[p, u, v]
    link: np.ndarray       # [K, K] bool


def build_tables(inst: Instance, L: int,
                 order: Optional[Sequence[str]] = None) -> Tables:
    order = list(order) if order is not None else bfs_order(inst)
    pos = {t: k for k, t in enumerate(order)}
    _, pred = inst.succ_pred()
    devs = sorted(inst.dev_ids)
    di = {u: inst.dev_ids.index(u) for u in devs}
    V, K = len(order), len(devs)
    tix = {t: k for k, t in enumerate(inst.task_ids)}
    dur = np.full((V, K), np.nan)
    dur_ok = np.zeros((V, K), bool)
    for i, t in enumerate(order):
        for k, u in enumerate(devs):
            v = inst.latency.get((t, u, L))
            if v is not None:
                dur[i, k] = v
                dur_ok[i, k] = True
    extra = np.empty(V)
    for i, t in enumerate(order):
        j = tix[t]
        x = (inst.im[j] + inst.om[j]) * L
        x += inst.wm[j]
        extra[i] = x
    cap = np.array([inst.memory[di[u]] + 1e-9 for u in devs])
    okL = np.array([L in inst.batch_sizes[di[u]] for u in devs])
    link = np.zeros((K, K), bool)
    for a, u in enumerate(devs):
        for b, v in enumerate(devs):
            link[a, b] = (a == b) or (u, v) in inst.bandwidth
    comm = np.zeros((V, K, K))
    for i, t in enumerate(order):
        om = inst.om[tix[t]]
        for a, u in enumerate(devs):
            for b, v in enumerate(devs):
                if a != b:
                    beta = inst.bandwidth.get((u, v))
                    comm[i, a, b] = np.nan if beta is None else om / beta
    preds = [[pos[p] for p in pred[t]] for t in order]
    return Tables(order=order, devs=devs, V=V, K=K, L=L, preds=preds,
                  dur=dur, dur_ok=dur_ok, extra=extra, cap=cap, okL=okL,
                  comm=comm, link=link)


# --------------------------------------------------------------- evaluator
def fitness_one(tb: Tables, genes: Sequence[int], trace: bool = False):
    """One candidate, flat restatement of decode() (heuristics.py:127-143).
    Returns (makespan, status[, starts])."""
    if any(not 0 <= int(k) < tb.K for k in genes):
        return (INF, ST_GENE, None) if trace else (INF, ST_GENE)
    avail = [0.0] * tb.K
    mem = [0.0] * tb.K
    end = [0.0] * tb.V
    starts = [0.0] * tb.V
    ms = 0.0
    for i in range(tb.V):
        d = int(genes[i])
        status = OK
        if not tb.okL[d]:
            status = ST_BATCH
        elif mem[d] + tb.extra[i] > tb.cap[d]:
            status = ST_MEM
        else:
            r = 0.0
            for p in tb.preds[i]:
                gp = int(genes[p])
                if not tb.link[gp, d]:
                    status = ST_LINK
                    break
                c = 0.0 if gp == d else float(tb.comm[p, gp, d])
                r = pymax(r, end[p] + c)
            if status == OK and not tb.dur_ok[i, d]:
                status = ST_MISSING
        if status != OK:
            return (INF, status, None) if trace else (INF, status)
        s = pymax(r, avail[d])
        e = s + float(tb.dur[i, d])
        starts[i] = s
        end[i] = e
        avail[d] = e
        mem[d] += float(tb.extra[i])
        ms = pymax(ms, e)
    return (ms, OK, starts) if trace else (ms, OK)


def fitness_np(tb: Tables, genes: np.ndarray):
    """Vectorised over candidates: genes uint8 [n, V] -> (makespan f64 [n],
    status u8 [n]). The per-lane operation sequence is exactly the one of
    fitness_one (first failing event wins), so results are bit-identical."""
    genes = np.asarray(genes)
    n = genes.shape[0]
    status = np.zeros(n, np.uint8)
    if tb.V == 0:
        return np.zeros(n), status
    bad = (genes >= tb.K).any(axis=1)
    g = np.where(genes >= tb.K, 0, genes).astype(np.intp)
    avail = np.zeros((tb.K, n))
    mem = np.zeros((tb.K, n))
    end = np.zeros((tb.V, n))
    lane = np.arange(n)
    for i in range(tb.V):
        d = g[:, i]
        live = status == OK
        ev = live & ~tb.okL[d]
        status[ev] = ST_BATCH
        live &= ~ev
        ev = live & ((mem[d, lane] + tb.extra[i]) > tb.cap[d])
        status[ev] = ST_MEM
        live &= ~ev
        r = np.zeros(n)
        nolink = np.zeros(n, bool)
        for p in tb.preds[i]:
            gp = g[:, p]
            nolink |= ~tb.link[gp, d]
            c = np.where(gp == d, 0.0, tb.comm[p, gp, d])
            x = end[p] + c
            r = np.where(x > r, x, r)
        ev = live & nolink
        status[ev] = ST_LINK
        live &= ~ev
        ev = live & ~tb.dur_ok[i, d]
        status[ev] = ST_MISSING
        a = avail[d, lane]
        s = np.where(a > r, a, r)
        e = s + tb.dur[i, d]
        end[i] = e
        avail[d, lane] = e
        mem[d, lane] = mem[d, lane] + tb.extra[i]
    ms = np.zeros(n)
    for k in range(tb.K):
        ms = np.where(avail[k] > ms, avail[k], ms)
    status[bad] = ST_GENE
    ms[status != OK] = INF
    return ms, status


def argmin_first(values: np.ndarray) -> tuple:
    """numpy.argmin semantics over a float64 vector with +inf allowed:
    (value, first index of the minimum); empty -> (inf, -1)."""
    if len(values) == 0:
        return INF, -1
    k = int(np.argmin(values))
    return float(values[k]), k


def throughput(L: int, ms: float) -> float:
    """1000 * L / makespan (cli.py:154, bounds.py:234)."""
    return 1000.0 * L / ms if ms > 0 else INF


# ------------------------------------------------------------------ bounds
def critical_path(inst: Instance, tasks) -> float:
    """bounds.py:57-72: fastest execution over every (device, batch size)
    in hardware insertion order, longest path over g._topo restricted to
    `tasks`. Raises KeyError for a missing latency entry."""
    tasks = set(tasks)
    if not tasks:
        return 0.0
    _, pred = inst.succ_pred()
    fastest = {}
    for t in tasks:
        best = None
        for j, u in enumerate(inst.dev_ids):
            for b in inst.batch_sizes[j]:
                v = inst.latency[(t, u, b)]
                if best is None or v < best:
                    best = v
        fastest[t] = best
    best = {}
    out = None
    for t in bfs_order(inst):
        if t not in tasks:
            continue
        inc = None
        for p in pred[t]:
            if p in tasks:
                inc = best[p] if inc is None else pymax(inc, best[p])
        best[t] = fastest[t] + (inc if inc is not None else 0.0)
        out = best[t] if out is None else pymax(out, best[t])
    return out


def _reach(adj, u, T):
    seen, stack = set(), [u]
    while stack:
        for b in adj[stack.pop()]:
            if b not in seen:
                seen.add(b)
                stack.append(b)
    return frozenset(seen & set(T))


def reach_dep(inst: Instance, u, T):
    """bounds.py:29-40: tasks of T reachable from u (u excluded)."""
    return _reach(inst.succ_pred()[0], u, T)


def reach_pre(inst: Instance, u, T):
    """bounds.py:43-54: tasks of T with a path to u (u excluded)."""
    return _reach(inst.succ_pred()[1], u, T)


# --------------------------------------------------- on-device generator
M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
GEN_C1 = 0xD1B54A32D192ED03
GEN_C2 = 0xD6E8FEB86659FD93


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser over uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def gen_genes(seed: int, first: int, n: int, V: int, K: int) -> np.ndarray:
    """Candidate c (global index): h = splitmix64(seed + (c+1)*GOLDEN); for
    w = 0, 1, ..: z = h + (w+1)*C1 (mod 2^64), z ^= z >> 32, z *= C2,
    z ^= z >> 32; position 8w + q (q < 8) gets ((byte q of z) * K) >> 8
    (bytes little-endian). Mirrors gen_row (csrc/eval_common.cuh, gen 1)."""
    W8 = (V + 7) // 8
    c = np.arange(first, first + n, dtype=np.uint64)[:, None]
    w = np.arange(1, W8 + 1, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        h = splitmix64(np.uint64(seed & M64) + (c + np.uint64(1)) * np.uint64(GOLDEN))
        z = h + w * np.uint64(GEN_C1)
        z = z ^ (z >> np.uint64(32))
        z = z * np.uint64(GEN_C2)
        z = z ^ (z >> np.uint64(32))
    b = np.ascontiguousarray(z.astype("<u8")).view(np.uint8).reshape(n, 8 * W8)
    out = ((b.astype(np.uint32) * np.uint32(K)) >> np.uint32(8)).astype(np.uint8)
    return out[:, :V]
