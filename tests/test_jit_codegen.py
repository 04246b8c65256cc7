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


def _nvrtc_compile(src: str) -> tuple[int, str]:
    """Compile like csrc/jit.cpp does (NVRTC, sm_100a); no GPU needed."""
    import ctypes as C
    lib = C.CDLL("/usr/local/cuda/lib64/libnvrtc.so.12")
    with open(os.path.join(ROOT, "paper_2308_00127_b200", "csrc",
                           "eval_common.cuh"), "rb") as f:
        hdr = f.read()
    prog = C.c_void_p()
    assert lib.nvrtcCreateProgram(
        C.byref(prog), src.encode(), b"k.cu", 1, (C.c_char_p * 1)(hdr),
        (C.c_char_p * 1)(b"eval_common.cuh")) == 0
    opts = [b"--gpu-architecture=sm_100a", b"--std=c++17", b"--fmad=false"]
    rc = lib.nvrtcCompileProgram(prog, len(opts), (C.c_char_p * 3)(*opts))
    n = C.c_size_t()
    lib.nvrtcGetProgramLogSize(prog, C.byref(n))
    log = C.create_string_buffer(n.value)
    lib.nvrtcGetProgramLog(prog, log)
    lib.nvrtcDestroyProgram(C.byref(prog))
    return rc, log.value.decode(errors="replace")


@pytest.mark.parametrize("which", ["ws30", "ri_missing_4", "ri_1000_L2"])
def test_emit_and_compile(which):
    if not os.path.exists("/usr/local/cuda/lib64/libnvrtc.so.12"):
        pytest.skip("NVRTC not available")
    if which.startswith("ri_"):
        doc = [d for d in random_docs() if d["name"] == which][0]
        p = Plan(*hs.load_instance(doc), doc["L"])
    else:
        p = Plan(*hs.load_instance(instance_doc(which)), 1)
    src = p.specialized_source(64)
    assert "hs_jit_eval" in src and "hs_jit_trace" in src
    # single-CTA search kernels (SA K10 / EA K9) for graphs up to 512 tasks
    assert ("hs_jit_sa" in src and "hs_jit_ea" in src) == (p.V <= 512)
    rc, log = _nvrtc_compile(src)
    assert rc == 0, log[-2000:]


def test_scope():
    # batched-variant plans: specialised on uniform full-mesh platforms
    # (the CNN / WS instances); per-pair bandwidths stay on the AOT K8
    p = Plan(*hs.load_instance(instance_doc("ws30")), 4, batched=())
    assert p.jit_eligible()
    rc, log = _nvrtc_compile(p.specialized_source(128))
    assert rc == 0, log[-2000:]
    g, hw, t = hs.load_instance(instance_doc("ws30"))
    devs = sorted(hw.devices)
    hw2 = hs.HardwareSystem(list(hw.devices.values()), {
        (u, v): 1e6 if {u, v} != {devs[0], devs[1]} else 1e5
        for u in devs for v in devs if u != v})
    q = Plan(g, hw2, t, 2, batched=())
    assert not q.jit_eligible()  # two bandwidths
    with pytest.raises(hs.GraphError):
        q.specialized_source()
    assert Plan(*hs.load_instance(instance_doc("ws200")), 1).jit_eligible()
    assert Plan(*hs.load_instance(instance_doc("tf96")), 1).jit_eligible()
    # ~1000 tasks: eligible, with the end-time slots in global memory
    assert Plan(*hs.load_instance(instance_doc("ws1000")), 1).jit_eligible()
    assert all(Plan(*hs.load_instance(d), d["L"]).jit_eligible()
               for d in random_docs()[:50] if d["graph"]["tasks"])


@pytest.mark.parametrize("opts", ["fma=1", "genes=reg", "near=0,ahead=0",
                                  "sync=16", "avail=reg,dur=sel",
                                  "max=int,ahead=4", "dom=0",
                                  "tmem=1,tcols=170,regs=8"])
def test_emit_options_compile(opts, monkeypatch):
    """Every code-generation option of the specialiser (HS_JIT_OPTS) emits
    CUDA that NVRTC accepts for sm_100a."""
    if not os.path.exists("/usr/local/cuda/lib64/libnvrtc.so.12"):
        pytest.skip("NVRTC not available")
    monkeypatch.setenv("HS_JIT_OPTS", opts)
    p = Plan(*hs.load_instance(instance_doc("ws30")), 1)
    src = p.specialized_source(64)
    rc, log = _nvrtc_compile(src)
    assert rc == 0, (opts, log[-2000:])
