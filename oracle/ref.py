"""The REFERENCE itself, as a checker -- test infrastructure only.

``import_reference()`` returns the reference package ``hetsched`` unmodified:
from ``/root/reference/pkg/src`` when that tree exists (the build container)
or from ``oracle/_ref`` (the copy ``make -C oracle ref`` makes during
``__graft_entry__.build()``, git-ignored, shipped with the snapshot to the GPU
box). Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
reference / CPU-baseline legs use it; the product package never imports it.
"""
from __future__ import annotations

import importlib
import os
import sys
from typing import Optional

HERE = os.path.dirname(os.path.abspath(__file__))
CANDIDATES = ("/root/reference/pkg/src", os.path.join(HERE, "_ref"))


def reference_path() -> Optional[str]:
    for p in CANDIDATES:
        if os.path.exists(os.path.join(p, "hetsched", "heuristics.py")):
            return p
    return None


def import_reference():
    """The reference package (hetsched) or None when it is not available.
    Its modules import networkx / scipy / numpy, all in this image."""
    if "hetsched" in sys.modules:
        return sys.modules["hetsched"]
    p = reference_path()
    if p is None:
        return None
    if p not in sys.path:
        sys.path.append(p)
    sys.dont_write_bytecode = True  # never write into the reference tree
    try:
        mod = importlib.import_module("hetsched")
        for sub in ("core", "heuristics", "bounds", "splitting", "milp",
                    "benchgen"):
            importlib.import_module("hetsched." + sub)
    except Exception:
        return None
    return mod


def load_instance(doc: dict):
    """(g, hw, table) as the reference's own objects, from a golden
    instance document (the reference wire format, core.py:297-356)."""
    import json
    ref = import_reference()
    if ref is None:
        raise ImportError("reference hetsched not available")
    RC = sys.modules["hetsched.core"]
    return (RC.load_graph(json.dumps(doc["graph"])),
            RC.load_hardware(json.dumps(doc["hardware"])),
            RC.load_latency(json.dumps(doc["latency"])))
