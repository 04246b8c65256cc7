"""patch_reference() rebinds the reference's call-time globals and restores
them (structure only; running the patched reference needs a GPU)."""
from __future__ import annotations

import os
import sys

import pytest

REF = "/root/reference/pkg/src"


def test_patch_and_restore():
    if not os.path.isdir(REF):
        pytest.skip("reference not present")
    sys.path.insert(0, REF)
    try:
        import hetsched.bounds as RB
        import hetsched.heuristics as RH
    except Exception as exc:  # pragma: no cover
        pytest.skip(f"reference not importable: {exc}")
    finally:
        sys.path.remove(REF)
    from paper_2308_00127_b200.integrate import patch_reference
    orig = (RH.fitness, RH.decode, RB.critical_path_bound, RB.dep_subgraph,
            RB.pre_subgraph)
    restore = patch_reference()
    try:
        assert RH.fitness is not orig[0] and RH.decode is not orig[1]
        assert RB.critical_path_bound is not orig[2]
        assert RB.dep_subgraph.__module__ == "paper_2308_00127_b200.bounds"
    finally:
        restore()
    assert (RH.fitness, RH.decode, RB.critical_path_bound, RB.dep_subgraph,
            RB.pre_subgraph) == orig
