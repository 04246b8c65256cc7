"""Schedule validation on the GPU -- the drop-in for the reference's
``validate_schedule`` (/root/reference/pkg/src/hetsched/core.py:206-291).

``validate_schedules`` checks many schedules of one instance in one launch
of K11 (csrc/validate.cu, C ABI ``hs_validate_schedules``): the host only
encodes the ``ScheduledBatch`` records into flat arrays; every check runs
on the device in the reference's order and the first violation comes back
as a code with its indices and values, from which the reference's own
``ScheduleError`` (``GraphError`` for a missing latency entry) message is
rebuilt here word for word. ``validate_schedule`` is the one-schedule form
with the reference's signature: it returns the makespan or raises.
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import _native as N
from .core import TOL, GraphError, ScheduleError
from .plan import instance_desc

_BATCH = np.dtype([("task", np.int32), ("device", np.int32),
                   ("size", np.int32), ("n_inputs", np.int32),
                   ("in_off", np.int64), ("start", np.float64),
                   ("flags", np.int32), ("pad", np.int32)])
_VIOL = np.dtype([("code", np.int32), ("a", np.int32), ("b", np.int32),
                  ("c", np.int32), ("v0", np.float64), ("v1", np.float64),
                  ("v2", np.float64)])
_I32 = (-(1 << 31), (1 << 31) - 1)
_I64 = (-(1 << 63), (1 << 63) - 1)


def _clamp(x: int, lo_hi) -> int:
    # out-of-int64 input values stay out of range after clamping
    lo, hi = lo_hi
    return x if lo <= x <= hi else (lo if x < lo else hi)


def _encode(g, hw, schedules):
    tix = {t: k for k, t in enumerate(g.tasks)}
    dix = {u: k for k, u in enumerate(hw.devices)}
    nb = sum(len(s.batches) for s in schedules)
    recs = np.zeros(nb, _BATCH)
    off = np.zeros(len(schedules) + 1, np.int64)
    inputs: list = []
    r = 0
    for q, s in enumerate(schedules):
        for b in s.batches:
            ins = tuple(b.inputs)
            size = int(b.size)
            recs[r] = (tix.get(b.task, -1), dix.get(b.device, -1),
                       size if _I32[0] <= size <= _I32[1] else -1,
                       len(ins), len(inputs), float(b.start),
                       1 if len(set(ins)) != len(ins) else 0, 0)
            inputs.extend(_clamp(int(x), _I64) for x in ins)
            r += 1
        off[q + 1] = r
    return recs, off, np.array(inputs or [0], np.int64)


def validate_schedules(g, hw, table, schedules: Sequence, tol: float = TOL):
    """Check every schedule on the GPU. Returns one entry per schedule: the
    makespan (float) when valid, else the exception the reference's
    validate_schedule would raise (not raised)."""
    schedules = list(schedules)
    if not schedules:
        return []
    lib = N.load()
    desc, keep = instance_desc(g, hw, table)
    recs, off, inputs = _encode(g, hw, schedules)
    counts = np.array([int(s.input_count) for s in schedules], np.int32)
    objs = np.array([float(s.objective) for s in schedules], np.float64)
    out = np.zeros(len(schedules), _VIOL)
    import torch
    stream = torch.cuda.current_stream()
    N.check(lib.hs_validate_schedules(
        C.byref(desc), len(schedules), off.ctypes.data,
        recs.ctypes.data if len(recs) else None, inputs.ctypes.data,
        counts.ctypes.data, objs.ctypes.data, float(tol), out.ctypes.data,
        int(stream.cuda_stream)), "hs_validate_schedules")
    del keep
    return [_result(g, hw, table, s, o) for s, o in zip(schedules, out)]


def validate_schedule(g, hw, table, s, tol: float = TOL) -> float:
    """The reference's validate_schedule (core.py:206-291), checked on the
    GPU: returns the makespan or raises the same error with the same
    message."""
    res = validate_schedules(g, hw, table, [s], tol)[0]
    if isinstance(res, Exception):
        raise res
    return res


def _result(g, hw, table, s, o):
    code = int(o["code"])
    if code == 0:
        return float(o["v0"])
    bs = s.batches
    L = s.input_count
    if code <= 8:
        b = bs[int(o["a"])]
        if code == 1:
            return ScheduleError(f"unknown task {b.task!r}")
        if code == 2:
            return ScheduleError(f"unknown device {b.device!r}")
        if code == 3:
            return ScheduleError(f"batch {b.task}@{b.device}: size {b.size} "
                                 f"inconsistent with inputs {b.inputs}")
        if code == 4:
            return ScheduleError(f"batch {b.task}@{b.device}: unsupported "
                                 f"batch size {b.size}")
        if code == 5:
            return ScheduleError(f"batch {b.task}@{b.device}: negative start")
        if code == 6:
            l = tuple(b.inputs)[int(o["c"])]
            return ScheduleError(f"batch {b.task}@{b.device}: input index {l} "
                                 f"out of range 1..{L}")
        if code == 7:
            l = tuple(b.inputs)[int(o["c"])]
            return ScheduleError(f"({b.task}, input {l}) assigned more than "
                                 "once")
        return GraphError(f"missing latency entry for ({b.task!r}, "
                          f"{b.device!r}, {b.size})")
    if code == 9:
        return ScheduleError(f"({list(g.tasks)[int(o['a'])]}, input "
                             f"{int(o['c'])}) not assigned")
    if code in (10, 11):
        i, j = g.edges[int(o["a"])]
        l = int(o["c"])
        bi = bs[int(o["b"])]
        # the consumer's batch: the only one of task j holding input l
        bj = next(x for x in bs if x.task == j and l in x.inputs)
        if code == 10:
            return ScheduleError(
                f"precedence violation on edge ({i}->{j}), input {l}: "
                f"no link {bi.device}->{bj.device}")
        return ScheduleError(
            f"precedence violation on edge ({i}->{j}), input {l}: "
            f"start {bj.start} < {float(o['v1'])} + comm {float(o['v2'])}")
    if code == 12:
        b1, b2 = bs[int(o["a"])], bs[int(o["b"])]
        dev = list(hw.devices)[int(o["c"])]
        return ScheduleError(
            f"overlap on {dev}: batch {b1.task}{b1.inputs} "
            f"[{b1.start},{float(o['v0'])}] and batch {b2.task}{b2.inputs} "
            f"[{b2.start},{float(o['v1'])}]")
    if code == 13:
        dev = list(hw.devices)[int(o["a"])]
        return ScheduleError(f"memory capacity exceeded on {dev}: "
                             f"{float(o['v0'])} > {hw.devices[dev].memory}")
    if code == 14:
        return ScheduleError(f"objective mismatch: stated {s.objective}, "
                             f"actual {float(o['v0'])}")
    return RuntimeError(f"hs_validate_schedules: unknown code {code}")
