"""Shared fixtures: golden documents (produced by the reference, see
tests/golden/make_golden.py), decoding helpers, and the `gpu` marker."""
from __future__ import annotations

import base64
import functools
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

INSTANCES = ["ws30", "ws200", "ws1000", "ws_stack_10x20", "ws_stack_10x100",
             "er_stack_10x10", "er_stack_4x10_c2", "tf96", "rn50f", "iv3f"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@functools.lru_cache(maxsize=None)
def instance_doc(name: str) -> dict:
    with open(os.path.join(GOLDEN, "instances", name + ".json")) as f:
        return json.load(f)


@functools.lru_cache(maxsize=None)
def random_docs() -> list:
    with open(os.path.join(GOLDEN, "random_instances.json")) as f:
        return json.load(f)


@functools.lru_cache(maxsize=None)
def golden(name: str):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        return json.load(f)


def case_genes(case: dict) -> np.ndarray:
    raw = np.frombuffer(base64.b64decode(case["genes_b64"]), np.uint8)
    return raw.reshape(case["n"], case["V"]).copy()


def parse_expected(exp):
    """-> (float values with nan for errors, error mask)."""
    vals = np.array([float.fromhex(x) if x not in ("inf", "GraphError")
                     else (np.inf if x == "inf" else np.nan) for x in exp])
    return vals, np.array([x == "GraphError" for x in exp])


def fhex(x: float) -> str:
    if x != x:
        return "nan"
    if x == float("inf"):
        return "inf"
    return float(x).hex()


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import hs_oracle_c
    return hs_oracle_c.load()
