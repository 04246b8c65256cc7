"""CPU check of the specialiser's code generator: the emitted CUDA for a
golden graph compiles for sm_100a with nvcc (no GPU needed), and plans
outside its scope are refused."""
from __future__ import annotations

import os
import shutil
import subprocess

import pytest

from conftest import ROOT, instance_doc, random_docs

import paper_2308_00127_b200 as hs
from paper_2308_00127_b200.plan import Plan


def test_emit_and_compile(tmp_path):
    nvcc = "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    p = Plan(*hs.load_instance(instance_doc("ws30")), 1)
    src = p.specialized_source(64)
    assert "hs_jit_eval" in src and src.count("pymax(") > 10
    shutil.copy(os.path.join(ROOT, "paper_2308_00127_b200", "csrc",
                             "eval_common.cuh"), tmp_path)
    (tmp_path / "k.cu").write_text(src)
    r = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a",
                        "-std=c++17", "--fmad=false", "-cubin", "-o",
                        str(tmp_path / "k.cubin"), str(tmp_path / "k.cu")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]


def test_scope():
    p = Plan(*hs.load_instance(instance_doc("tf96")), 1)  # K = 30
    assert not p.jit_eligible()
    with pytest.raises(hs.GraphError):
        p.specialized_source()
    assert Plan(*hs.load_instance(instance_doc("ws200")), 1).jit_eligible()
    # straight-line code for ~1000 tasks would take ptxas minutes
    assert not Plan(*hs.load_instance(instance_doc("ws1000")), 1).jit_eligible()
    for doc in random_docs()[:50]:  # per-pair bandwidths: out of scope
        assert not Plan(*hs.load_instance(doc), doc["L"]).jit_eligible()
