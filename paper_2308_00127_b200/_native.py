"""ctypes binding of the C ABI in include/hetsched_b200.h.

The shared library is the product: there is no Python or CPU fallback. If
``libhetsched_b200.so`` is missing or a GPU call fails, the error surfaces
(ImportError / RuntimeError). ctypes releases the GIL around every foreign
call, so evaluations issued from a thread pool (the reference's
ModuleSolver contract, splitting.py:342-344) run concurrently.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhetsched_b200.so")

HS_OK, HS_EINVAL, HS_ECYCLE, HS_ECUDA, HS_ENOMEM, HS_EHOST = 0, 1, 2, 3, 4, 5
ST_OK, ST_BATCH, ST_MEMORY, ST_LINK, ST_MISSING, ST_GENE = 0, 1, 2, 3, 4, 5

GEN_RANDOM, GEN_ENUM, GEN_NEIGHBOR = 1, 2, 3

_p = C.POINTER


class InstanceDesc(C.Structure):
    _fields_ = [
        ("n_tasks", C.c_int32),
        ("task_ids", C.c_char_p),
        ("task_id_off", _p(C.c_int64)),
        ("wm", _p(C.c_double)), ("im", _p(C.c_double)), ("om", _p(C.c_double)),
        ("n_edges", C.c_int32),
        ("edge_src", _p(C.c_int32)), ("edge_dst", _p(C.c_int32)),
        ("n_devices", C.c_int32),
        ("dev_ids", C.c_char_p),
        ("dev_id_off", _p(C.c_int64)),
        ("memory", _p(C.c_double)),
        ("batch_off", _p(C.c_int32)),
        ("batch_sizes", _p(C.c_int32)),
        ("bandwidth", _p(C.c_double)),
        ("L", C.c_int32),
        ("latency", _p(C.c_double)),
        ("latency_ok", _p(C.c_uint8)),
        ("order", _p(C.c_int32)),
    ]


class PlanInfo(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "V", "E", "K", "L", "live_slots", "n_classes", "uniform_comm",
        "full_mesh", "mem_check", "all_batch_ok", "latency_complete", "words",
        "pref_ld", "specializable", "batched_options", "max_parts")]


class Best(C.Structure):
    _fields_ = [("cost", C.c_double), ("index", C.c_int64)]


_lib = None
_lock = threading.Lock()


def load() -> C.CDLL:
    """Load the native library (built by paper_2308_00127_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with "
                "`python -c 'import __graft_entry__; __graft_entry__.build()'`"
                " (there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
        sig = {
            "hs_last_error": (C.c_char_p, []),
            "hs_abi_version": (C.c_int, []),
            "hs_scratch_trim": (C.c_int, []),
            "hs_plan_create": (C.c_int, [_p(InstanceDesc), _p(vp)]),
            "hs_plan_destroy": (None, [vp]),
            "hs_plan_create_batched": (C.c_int, [_p(InstanceDesc), vp, i32,
                                                 _p(vp)]),
            "hs_plan_batched_options": (C.c_int, [vp, vp, vp, vp]),
            "hs_plan_get_info": (C.c_int, [vp, _p(PlanInfo)]),
            "hs_plan_order": (C.c_int, [vp, vp, vp]),
            "hs_plan_greedy": (C.c_int, [vp, vp, vp, _p(C.c_double)]),
            "hs_plan_specialize": (C.c_int, [vp, _p(C.c_double)]),
            "hs_plan_emit_specialized": (C.c_int, [vp, i32, vp, i64,
                                                   _p(C.c_int64)]),
            "hs_eval": (C.c_int, [vp, vp, i64, i64, vp, vp, vp, i64, vp]),
            "hs_eval_host": (C.c_int, [vp, vp, i64, i64, vp, vp, vp, i64, vp]),
            "hs_eval_host_packs": (C.c_int, [vp, i64]),
            "hs_pack_genes2": (C.c_int, [vp, i64, i64, i32, i32, vp, i64,
                                         _p(C.c_int32)]),
            "hs_eval_packed": (C.c_int, [vp, vp, i64, i64, vp, vp, vp, i64,
                                         vp]),
            "hs_eval_host_packed": (C.c_int, [vp, vp, i64, i64, vp, vp, vp,
                                              i64, vp]),
            "hs_eval_packed3": (C.c_int, [vp, vp, i64, i64, vp, vp, vp, i64,
                                          vp]),
            "hs_eval_host_packed3": (C.c_int, [vp, vp, i64, i64, vp, vp, vp,
                                               i64, vp]),
            "hs_ea_run": (C.c_int, [vp, vp, C.c_double, vp, vp, vp, i32, vp,
                                    vp, vp]),
            "hs_ea_run_chunk": (C.c_int, [vp, vp, vp, vp, vp, vp, i32, i32,
                                          vp, vp]),
            "hs_sa_run": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, C.c_double,
                                    i32, i32, i32, vp]),
            "hs_sa_run_multi": (C.c_int, [vp, i32, i64, vp, vp, vp, vp, vp,
                                          vp, C.c_double, i32, i32, i32, vp]),
            "hs_ea_run_multi": (C.c_int, [vp, i32, i64, vp, vp, vp, vp, vp,
                                          i32, vp, vp, vp]),
            "hs_ea_draw": (C.c_int, [i32, vp, vp, i32, i32, C.c_double, i32,
                                     vp, vp, vp, i64, vp, vp]),
            "hs_eval_gen": (C.c_int, [vp, C.c_uint64, i64, i64, vp, vp, vp,
                                      vp, vp]),
            "hs_eval_gen_ex": (C.c_int, [vp, C.c_int, C.c_uint64, i64, i64,
                                         vp, vp, i32, vp, vp, vp, vp, vp]),
            "hs_trace": (C.c_int, [vp, vp, i64, i64, vp, vp, vp, vp]),
            "hs_cp_bound": (C.c_int, [vp, vp, i64, vp, vp, vp]),
            "hs_reach": (C.c_int, [vp, vp, vp, vp]),
            "hs_modularity": (C.c_int, [vp, vp, i64, i32, C.c_double, vp, vp,
                                        vp]),
            "hs_best_merge": (C.c_int, [_p(Best), i64, _p(Best)]),
            "hs_best_allreduce": (C.c_int, [vp, vp, vp, vp]),
            "hs_bridges_articulation": (C.c_int, [i32, i32, vp, vp, vp, vp,
                                                  vp]),
            "hs_k_edge_components": (C.c_int, [i32, C.c_char_p, vp, i32, vp,
                                               vp, i32, vp, vp]),
            "hs_validate_schedules": (C.c_int, [_p(InstanceDesc), i64, vp, vp,
                                                vp, vp, vp, C.c_double, vp,
                                                vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.hs_abi_version() != 1:
            raise ImportError("libhetsched_b200.so ABI mismatch")
        _lib = lib
        return lib


def exported_symbols() -> list[str]:
    """Names declared by include/hetsched_b200.h (checked by the tests)."""
    return ["hs_last_error", "hs_abi_version", "hs_scratch_trim",
            "hs_plan_create",
            "hs_plan_destroy", "hs_plan_create_batched",
            "hs_plan_batched_options", "hs_plan_get_info", "hs_plan_order",
            "hs_plan_greedy",
            "hs_plan_specialize", "hs_plan_emit_specialized", "hs_eval",
            "hs_eval_host", "hs_eval_host_packs", "hs_pack_genes2", "hs_eval_packed", "hs_eval_host_packed",
            "hs_eval_packed3", "hs_eval_host_packed3", "hs_ea_run",
            "hs_ea_run_chunk", "hs_sa_run", "hs_sa_run_multi",
            "hs_ea_run_multi", "hs_ea_draw", "hs_eval_gen", "hs_eval_gen_ex", "hs_trace",
            "hs_cp_bound", "hs_reach", "hs_modularity", "hs_best_merge",
            "hs_best_allreduce", "hs_bridges_articulation",
            "hs_k_edge_components", "hs_validate_schedules"]


def check(rc: int, what: str = "") -> None:
    """Map an HS_E* return code onto the reference's exception types."""
    if rc == HS_OK:
        return
    msg = load().hs_last_error().decode("utf-8", "replace")
    if what:
        msg = f"{what}: {msg}"
    from .core import GraphError
    if rc in (HS_EINVAL, HS_ECYCLE):
        raise GraphError(msg)
    if rc == HS_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)
