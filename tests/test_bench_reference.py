"""bench.py's reference arm on CPU: it runs the reference's own
hetsched.heuristics.fitness (imported unmodified through oracle/ref.py) and
prints one JSON line with impl "reference", kind "reference", the same
config as the GPU arm and an e2e of zero copied bytes."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT


def test_reference_arm_line():
    from oracle import ref
    if ref.import_reference() is None:
        pytest.skip("reference not importable")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"),
                          "--impl", "reference", "--steps", "1",
                          "--warmup", "1"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.splitlines()
                    if l.startswith("{")][-1])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference"
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"],
                        "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench._config(1 << 24, 1)
    assert d["metric"] == bench.METRIC and d["higher_is_better"] is True
