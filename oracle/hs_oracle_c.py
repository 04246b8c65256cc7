"""ctypes loader for the C oracle (oracle/hs_oracle.c) -- test
infrastructure only (tests/, smoke(), bench.py's cpu_baseline leg)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from .hs_oracle import Tables

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libhs_oracle.so")


class _T(C.Structure):
    _fields_ = [("V", C.c_int), ("K", C.c_int),
                ("pred_off", C.c_void_p), ("pred_pos", C.c_void_p),
                ("dur", C.c_void_p), ("dur_ok", C.c_void_p),
                ("extra", C.c_void_p), ("cap", C.c_void_p),
                ("okL", C.c_void_p), ("comm", C.c_void_p),
                ("link", C.c_void_p)]


def load():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    lib = C.CDLL(LIB)
    lib.hso_fitness.argtypes = [C.POINTER(_T), C.c_void_p, C.c_int64,
                                C.c_int64, C.c_void_p, C.c_void_p, C.c_int]
    lib.hso_trace.argtypes = [C.POINTER(_T), C.c_void_p, C.c_void_p,
                              C.c_void_p]
    return lib


class CTables:
    """Flat copies of oracle Tables kept alive for the C calls."""

    def __init__(self, tb: Tables):
        self.tb = tb
        off = np.zeros(tb.V + 1, np.int32)
        off[1:] = np.cumsum([len(p) for p in tb.preds])
        self.off = off
        self.pos = np.array([p for ps in tb.preds for p in ps] or [0],
                            np.int32)
        self.dur = np.ascontiguousarray(np.where(np.isnan(tb.dur), 0.0, tb.dur))
        self.dur_ok = np.ascontiguousarray(tb.dur_ok, np.uint8)
        self.extra = np.ascontiguousarray(tb.extra)
        self.cap = np.ascontiguousarray(tb.cap)
        self.okL = np.ascontiguousarray(tb.okL, np.uint8)
        self.comm = np.ascontiguousarray(np.where(np.isnan(tb.comm), 0.0, tb.comm))
        self.link = np.ascontiguousarray(tb.link, np.uint8)
        self.s = _T(tb.V, tb.K, off.ctypes.data, self.pos.ctypes.data,
                    self.dur.ctypes.data, self.dur_ok.ctypes.data,
                    self.extra.ctypes.data, self.cap.ctypes.data,
                    self.okL.ctypes.data, self.comm.ctypes.data,
                    self.link.ctypes.data)

    def fitness(self, lib, genes: np.ndarray, threads: int = 1):
        genes = np.ascontiguousarray(genes, np.uint8)
        n = genes.shape[0]
        out = np.empty(n, np.float64)
        st = np.empty(n, np.uint8)
        lib.hso_fitness(C.byref(self.s), genes.ctypes.data, n,
                        genes.shape[1] if n else 0, out.ctypes.data,
                        st.ctypes.data, threads)
        return out, st
