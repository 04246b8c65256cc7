"""Evaluation plans: (graph, hardware, latency table, L[, genome order]) ->
native ``hs_plan`` handle, plus the device-side entry points that use it.

A plan is compiled once per instance by the native plan compiler
(csrc/plan.cpp) and cached on object identity plus a cheap shape
fingerprint (entry / link / device counts). The reference declares every
type immutable after construction (SPEC.md, "Concurrency Model"; core.py:38),
but ``LatencyTable.entries`` and
``HardwareSystem.bandwidth`` are plain dicts: adding or removing entries
after a first evaluation is detected (new plan), editing a value in place
is not -- build a new table / hardware object instead (a full content hash
would cost more than a small evaluation on every call).
"""
from __future__ import annotations

import ctypes as C
import threading
import weakref
from collections import OrderedDict
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from .core import GraphError


def _i64(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def _i32(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _f64(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u8(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def _strings(ids):
    raw = [s.encode("utf-8", "surrogatepass") for s in ids]
    off = np.zeros(len(raw) + 1, np.int64)
    off[1:] = np.cumsum([len(b) for b in raw])
    return b"".join(raw), off


def instance_desc(g, hw, table, L: int = 1,
                  order: Optional[Sequence[str]] = None):
    """The C ABI's hs_instance_desc of (g, hw, table, L[, genome order]) and
    the Python objects that must stay alive while it is used (the last
    three: task ids, device ids, latency column list)."""
    task_ids = list(g.tasks)
    tix = {t: k for k, t in enumerate(task_ids)}
    dev_ids = list(hw.devices)
    K = len(dev_ids)
    tnodes = [g.tasks[t] for t in task_ids]
    wm = np.array([float(t.wm) for t in tnodes], np.float64)
    im = np.array([float(t.im) for t in tnodes], np.float64)
    om = np.array([float(t.om) for t in tnodes], np.float64)
    src = np.array([tix[a] for a, _ in g.edges], np.int32)
    dst = np.array([tix[b] for _, b in g.edges], np.int32)
    devs = [hw.devices[u] for u in dev_ids]
    memory = np.array([float(d.memory) for d in devs], np.float64)
    sizes = [tuple(int(b) for b in d.batch_sizes) for d in devs]
    boff = np.zeros(K + 1, np.int32)
    boff[1:] = np.cumsum([len(s) for s in sizes])
    bs = np.array([b for s in sizes for b in s], np.int32)
    bw = np.zeros((K, K), np.float64)
    dix = {u: k for k, u in enumerate(dev_ids)}
    for (a, b), v in hw.bandwidth.items():
        bw[dix[a], dix[b]] = float(v)
    cols = [(u, b) for u, s in zip(dev_ids, sizes) for b in s]
    ent = table.entries
    lat = np.zeros((len(task_ids), max(len(cols), 1)), np.float64)
    ok = np.zeros(lat.shape, np.uint8)
    for r, t in enumerate(task_ids):
        for c, (u, b) in enumerate(cols):
            v = ent.get((t, u, b))
            if v is not None:
                lat[r, c] = v
                ok[r, c] = 1
    tid_bytes, toff = _strings(task_ids)
    did_bytes, doff = _strings(dev_ids)
    order_arr = None
    if order is not None:
        try:
            order_arr = np.array([tix[t] for t in order], np.int32)
        except KeyError as exc:
            raise GraphError(f"genome order names unknown task {exc}")
        if len(order_arr) != len(task_ids):
            raise GraphError("genome length must equal task count")
    keep = (wm, im, om, src, dst, memory, boff, bs, bw, lat, ok, tid_bytes,
            toff, did_bytes, doff, order_arr, task_ids, dev_ids, cols)
    d = N.InstanceDesc(
        n_tasks=len(task_ids), task_ids=tid_bytes, task_id_off=_i64(toff),
        wm=_f64(wm), im=_f64(im), om=_f64(om),
        n_edges=len(src), edge_src=_i32(src), edge_dst=_i32(dst),
        n_devices=K, dev_ids=did_bytes, dev_id_off=_i64(doff),
        memory=_f64(memory), batch_off=_i32(boff), batch_sizes=_i32(bs),
        bandwidth=_f64(bw), L=int(L), latency=_f64(lat), latency_ok=_u8(ok),
        order=_i32(order_arr) if order_arr is not None else None)
    return d, keep


class Plan:
    """Native evaluation plan of one instance at load L."""

    def __init__(self, g, hw, table, L: int,
                 order: Optional[Sequence[str]] = None,
                 batched: Optional[tuple] = None):
        """`batched` (a tuple of allowed sub-batch sizes, () = the
        reference's default L/4, L/2, 3L/4, L) makes a batched-variant plan
        whose genes are option indices (heuristics.py:337-433)."""
        lib = N.load()
        d, keep = instance_desc(g, hw, table, L, order)
        self._keep = keep
        task_ids, dev_ids, K = keep[-3], keep[-2], d.n_devices
        if K == 0:
            raise GraphError("gene value out of device range")
        h = C.c_void_p()
        if batched is None:
            N.check(lib.hs_plan_create(C.byref(d), C.byref(h)), "plan")
        else:
            sp = np.array(list(batched) or [0], np.int32)
            N.check(lib.hs_plan_create_batched(
                C.byref(d), sp.ctypes.data if batched else None, len(batched),
                C.byref(h)), "plan")
        self._keep = None
        self.handle = h
        self._lib = lib
        info = N.PlanInfo()
        N.check(lib.hs_plan_get_info(h, C.byref(info)))
        self.info = info
        self.V, self.K, self.L = info.V, info.K, int(L)
        o = np.zeros(max(self.V, 1), np.int32)
        dv = np.zeros(K, np.int32)
        N.check(lib.hs_plan_order(h, o.ctypes.data, dv.ctypes.data))
        self.task_ids = task_ids
        self.order = tuple(task_ids[k] for k in o[:self.V])
        self.devices = tuple(dev_ids[k] for k in dv)  # gene k -> device id
        self.pref_ld = info.pref_ld
        self.words = info.words
        self.batched = batched is not None
        self.options = None
        if self.batched:
            n_opt, P = info.batched_options, info.max_parts
            tab = np.zeros(max(n_opt * P * 4, 1), np.int32)
            N.check(lib.hs_plan_batched_options(h, None, None, tab.ctypes.data))
            tab = tab[:n_opt * P * 4].reshape(n_opt, P, 4)
            self.options = [
                (tuple(int(x[3]) for x in tab[o] if x[0] >= 0),
                 tuple(self.devices[int(x[0])] for x in tab[o] if x[0] >= 0))
                for o in range(n_opt)]
            self.max_parts = P
        self._reach = None
        self._lock = threading.Lock()
        self.specialized_ms = None

    # ------------------------------------------------------- specialisation
    def specialize(self) -> float:
        """Compile the graph-specialised evaluator for the current device
        (NVRTC, once per plan and device); returns the compile time in ms.
        Raises GraphError when the plan is outside its scope."""
        import torch
        torch.cuda.init()
        ms = C.c_double()
        N.check(self._lib.hs_plan_specialize(self.handle, C.byref(ms)),
                "specialize")
        self.specialized_ms = ms.value
        return ms.value

    def maybe_specialize(self, n: int) -> bool:
        """Specialise when a batch is large enough to amortise the compile
        (HS_JIT_MIN candidates, default 2**20; 2**27 above 512 tasks, where
        NVRTC takes tens of seconds); False if out of scope."""
        import os
        if self.specialized_ms is not None:
            return True
        if os.environ.get("HS_JIT", "1") == "0":
            return False
        floor = 1 << (20 if self.V <= 512 else 27)
        if n < int(os.environ.get("HS_JIT_MIN", floor)):
            return False
        if not self.jit_eligible():
            return False
        self.specialize()
        return True

    def jit_eligible(self) -> bool:
        """Inside the specialised evaluator's scope (csrc/jit.cpp)."""
        return bool(self.info.specializable)

    def specialized_source(self, lanes: int = 192) -> str:
        n = C.c_int64()
        N.check(self._lib.hs_plan_emit_specialized(self.handle, lanes, None, 0,
                                                   C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        N.check(self._lib.hs_plan_emit_specialized(self.handle, lanes, buf,
                                                   n.value + 1, C.byref(n)))
        return buf.value.decode()

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.hs_plan_destroy(h)
            except Exception:
                pass

    # ---------------------------------------------------------- device calls
    @staticmethod
    def _stream(stream=None) -> int:
        import torch
        if stream is None:
            stream = torch.cuda.current_stream()
        return int(stream.cuda_stream)

    def eval(self, genes, makespan=None, status=None, best=None,
             index_base: int = 0, stream=None) -> None:
        """hs_eval on device tensors: genes uint8 [n, ld] (ld >= V)."""
        n = int(genes.shape[0])
        ld = int(genes.stride(0)) if n > 1 else max(int(genes.shape[1]),
                                                     self.V)
        if n > 1 and ld < self.V:
            raise GraphError(f"genome rows overlap: stride(0) = {ld} < V = "
                             f"{self.V}")
        N.check(self._lib.hs_eval(
            self.handle, genes.data_ptr() if genes.numel() else None, n, ld,
            _ptr(makespan), _ptr(status), _ptr(best), int(index_base),
            self._stream(stream)), "hs_eval")

    def eval_host(self, genes: np.ndarray, makespan=None, status=None,
                  best: Optional[N.Best] = None, index_base: int = 0,
                  stream=None) -> None:
        """hs_eval_host: numpy uint8 [n, ld] host genes, results to host."""
        n = genes.shape[0]
        # rows must be unit-stride and non-overlapping (a view such as
        # genes[::-1] or a broadcast is copied); a length-1 leading axis may
        # carry stride 0 (x[None, :])
        if genes.dtype != np.uint8 or genes.strides[-1] != 1 or (
                n > 1 and genes.strides[0] < genes.shape[1]):
            genes = np.ascontiguousarray(genes, dtype=np.uint8)
        ld = genes.strides[0] if n > 1 else max(genes.shape[1], self.V)
        N.check(self._lib.hs_eval_host(
            self.handle, genes.ctypes.data if n else None, n, ld,
            makespan.ctypes.data if makespan is not None else None,
            status.ctypes.data if status is not None else None,
            C.byref(best) if best is not None else None, int(index_base),
            self._stream(stream)), "hs_eval_host")

    def eval_host_packs(self, n: int) -> bool:
        """hs_eval_host_packs: whether eval_host packs n rows on the host."""
        rc = int(self._lib.hs_eval_host_packs(self.handle, int(n)))
        if rc < 0:
            N.check(rc, "hs_eval_host_packs")
        return rc == 1

    def packed_ld(self) -> int:
        """Row bytes of 2-bit packed genomes (multiple of 4)."""
        return ((self.V + 3) // 4 + 3) // 4 * 4

    def eval_packed(self, packed, makespan=None, status=None, best=None,
                    index_base: int = 0, stream=None) -> None:
        """hs_eval_packed on device tensors: packed uint8 [n, packed_ld]."""
        n = int(packed.shape[0])
        N.check(self._lib.hs_eval_packed(
            self.handle, packed.data_ptr() if packed.numel() else None, n,
            int(packed.stride(0)) if n > 1 else self.packed_ld(),
            _ptr(makespan), _ptr(status), _ptr(best), int(index_base),
            self._stream(stream)), "hs_eval_packed")

    def eval_host_packed(self, packed: np.ndarray, makespan=None, status=None,
                         best: Optional[N.Best] = None, index_base: int = 0,
                         stream=None) -> None:
        packed = np.ascontiguousarray(packed, dtype=np.uint8)
        n = packed.shape[0]
        ld = packed.strides[0] if n > 1 else self.packed_ld()
        N.check(self._lib.hs_eval_host_packed(
            self.handle, packed.ctypes.data if n else None, n, ld,
            makespan.ctypes.data if makespan is not None else None,
            status.ctypes.data if status is not None else None,
            C.byref(best) if best is not None else None, int(index_base),
            self._stream(stream)), "hs_eval_host_packed")

    def ea_run(self, parent, cur_fit: float, moff, mpos, mval, budget: int,
               fit, info, stream=None) -> None:
        """hs_ea_run (K9) on device tensors: parent uint8 [V] (in/out),
        moff int32 [budget+1], mpos int32, mval uint8, fit f64 [1],
        info int32 [4]."""
        N.check(self._lib.hs_ea_run(
            self.handle, _ptr(parent), float(cur_fit), _ptr(moff),
            _ptr(mpos) if mpos.numel() else None,
            _ptr(mval) if mval.numel() else None, int(budget), _ptr(fit),
            _ptr(info), self._stream(stream)), "hs_ea_run")

    def ea_run_chunk(self, parent, fit, moff, mpos, mval, n_children: int,
                     first_child: int, info, stream=None) -> None:
        """hs_ea_run_chunk (K9 in chained chunks) on device tensors."""
        N.check(self._lib.hs_ea_run_chunk(
            self.handle, _ptr(parent), _ptr(fit), _ptr(moff),
            _ptr(mpos) if mpos.numel() else None,
            _ptr(mval) if mval.numel() else None, int(n_children),
            int(first_child), _ptr(info), self._stream(stream)),
            "hs_ea_run_chunk")

    def sa_run(self, genes, best, rng, buf, f, istate, alpha: float,
               n_dev: int, budget: int, window: int, stream=None) -> None:
        """hs_sa_run (K10) on device tensors (all state in/out): genes /
        best uint8 [V], rng int64 [4] (PCG64 words), buf int32 [2], f f64
        [5], istate int32 [7]."""
        N.check(self._lib.hs_sa_run(
            self.handle, _ptr(genes), _ptr(best), _ptr(rng), _ptr(buf),
            _ptr(f), _ptr(istate), float(alpha), int(n_dev), int(budget),
            int(window), self._stream(stream)), "hs_sa_run")

    def sa_run_multi(self, chains: int, genes, best, rng, buf, f, istate,
                     alpha: float, n_dev: int, budget: int, window: int,
                     stream=None) -> None:
        """hs_sa_run_multi: `chains` K10 chains, one CTA each; genes / best
        uint8 [chains, stride], rng int64 [chains, 4], buf int32 [chains, 2],
        f f64 [chains, 8], istate int32 [chains, 8] (contiguous)."""
        N.check(self._lib.hs_sa_run_multi(
            self.handle, int(chains), int(genes.stride(0)), _ptr(genes),
            _ptr(best), _ptr(rng), _ptr(buf), _ptr(f), _ptr(istate),
            float(alpha), int(n_dev), int(budget), int(window),
            self._stream(stream)), "hs_sa_run_multi")

    def ea_run_multi(self, chains: int, parent, cur_fit, moff, mpos, mval,
                     budget: int, fit, info, stream=None) -> None:
        """hs_ea_run_multi: `chains` K9 chains, one CTA each; parent uint8
        [chains, stride] (in/out), cur_fit / fit f64 [chains], moff int32
        [chains, budget + 1] (absolute), info int32 [chains, 4]."""
        N.check(self._lib.hs_ea_run_multi(
            self.handle, int(chains), int(parent.stride(0)), _ptr(parent),
            _ptr(cur_fit), _ptr(moff),
            _ptr(mpos) if mpos.numel() else None,
            _ptr(mval) if mval.numel() else None, int(budget), _ptr(fit),
            _ptr(info), self._stream(stream)), "hs_ea_run_multi")

    def packed3_ld(self) -> int:
        """Row bytes of base-3 packed genomes (5 genes per byte)."""
        return (self.V + 4) // 5

    def eval_packed3(self, packed, makespan=None, status=None, best=None,
                     index_base: int = 0, stream=None) -> None:
        """hs_eval_packed3 on device tensors: packed uint8 [n, packed3_ld]."""
        n = int(packed.shape[0])
        N.check(self._lib.hs_eval_packed3(
            self.handle, packed.data_ptr() if packed.numel() else None, n,
            int(packed.stride(0)) if n > 1 else self.packed3_ld(),
            _ptr(makespan), _ptr(status), _ptr(best), int(index_base),
            self._stream(stream)), "hs_eval_packed3")

    def eval_host_packed3(self, packed: np.ndarray, makespan=None,
                          status=None, best: Optional[N.Best] = None,
                          index_base: int = 0, stream=None) -> None:
        packed = np.ascontiguousarray(packed, dtype=np.uint8)
        n = packed.shape[0]
        ld = packed.strides[0] if n > 1 else self.packed3_ld()
        N.check(self._lib.hs_eval_host_packed3(
            self.handle, packed.ctypes.data if n else None, n, ld,
            makespan.ctypes.data if makespan is not None else None,
            status.ctypes.data if status is not None else None,
            C.byref(best) if best is not None else None, int(index_base),
            self._stream(stream)), "hs_eval_host_packed3")

    def eval_gen(self, mode: int, seed: int, first: int, n: int,
                 template=None, group=None, n_groups: int = 0,
                 makespan=None, status=None, genes_out=None, best=None,
                 stream=None) -> None:
        N.check(self._lib.hs_eval_gen_ex(
            self.handle, int(mode), int(seed) & 0xFFFFFFFFFFFFFFFF,
            int(first), int(n), _ptr(template), _ptr(group), int(n_groups),
            _ptr(makespan), _ptr(status), _ptr(genes_out), _ptr(best),
            self._stream(stream)), "hs_eval_gen")

    def trace(self, genes, starts, makespan, status, stream=None) -> None:
        n, ld = int(genes.shape[0]), int(genes.stride(0))
        N.check(self._lib.hs_trace(
            self.handle, genes.data_ptr(), n, ld, starts.data_ptr(),
            makespan.data_ptr(), status.data_ptr(), self._stream(stream)),
            "hs_trace")

    def cp_bound(self, masks, out, status, stream=None) -> None:
        N.check(self._lib.hs_cp_bound(
            self.handle, masks.data_ptr(), int(masks.shape[0]),
            out.data_ptr(), status.data_ptr(), self._stream(stream)),
            "hs_cp_bound")

    def reach(self):
        """(desc, anc) uint64 bitsets [n_tasks, words] as numpy (cached)."""
        with self._lock:
            if self._reach is None:
                import torch
                nt, w = len(self.task_ids), max(self.words, 1)
                desc = torch.zeros((nt, w), dtype=torch.int64, device="cuda")
                anc = torch.zeros((nt, w), dtype=torch.int64, device="cuda")
                N.check(self._lib.hs_reach(self.handle, desc.data_ptr(),
                                           anc.data_ptr(), self._stream()),
                        "hs_reach")
                self._reach = (desc.cpu().numpy().view(np.uint64),
                               anc.cpu().numpy().view(np.uint64))
            return self._reach


def _ptr(t):
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return C.addressof(t)


# ---------------------------------------------------------------------------
# identity cache

_CACHE: "OrderedDict[tuple, tuple]" = OrderedDict()
_CACHE_LOCK = threading.Lock()
_CACHE_MAX = 64


def _ref(o):
    try:
        return weakref.ref(o)
    except TypeError:
        return lambda o=o: o  # not weak-referenceable: hold it


def _fingerprint(g, hw, table) -> tuple:
    return (len(g.tasks), len(getattr(g, "edges", ())),
            len(hw.devices), len(getattr(hw, "bandwidth", ())),
            len(getattr(table, "entries", ())))


def get_plan(g, hw, table, L: int, order: Optional[Sequence[str]] = None,
             batched: Optional[tuple] = None) -> Plan:
    """Cached plan for (g, hw, table, L, order[, batched splits]); `order`
    None or equal to the graph's BFS order selects the default plan."""
    if order is not None:
        order = tuple(order)
        if order == tuple(g._topo):
            order = None
    if batched is not None:
        batched = tuple(sorted(set(int(x) for x in batched)))
    key = (id(g), id(hw), id(table), int(L), order, batched,
           _fingerprint(g, hw, table))
    with _CACHE_LOCK:
        hit = _CACHE.get(key)
        if hit is not None:
            refs, plan = hit
            if refs[0]() is g and refs[1]() is hw and refs[2]() is table:
                _CACHE.move_to_end(key)
                return plan
            del _CACHE[key]
    plan = Plan(g, hw, table, L, order, batched)
    with _CACHE_LOCK:
        _CACHE[key] = ((_ref(g), _ref(hw), _ref(table)), plan)
        while len(_CACHE) > _CACHE_MAX:
            _CACHE.popitem(last=False)
    return plan
