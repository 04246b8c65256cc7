"""The host-side 2-bit packer of hs_eval_host (csrc/host_pack.cpp, AVX2 with
masked row tails and a scalar path) against the layout definition, on the
CPU: compiled with g++ from the product source and run."""
from __future__ import annotations

import os
import shutil
import subprocess

import pytest

from conftest import ROOT

CSRC = os.path.join(ROOT, "paper_2308_00127_b200", "csrc")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_host_pack_matches_layout(tmp_path):
    exe = str(tmp_path / "host_pack_check")
    subprocess.run(
        ["g++", "-O2", "-std=c++17", f"-I{CSRC}", f"-I{CUDA}/include",
         os.path.join(ROOT, "tests", "native", "host_pack_check.cpp"),
         os.path.join(CSRC, "host_pack.cpp"), f"-L{CUDA}/lib64", "-lcudart",
         "-lpthread", f"-Wl,-rpath,{CUDA}/lib64", "-o", exe],
        check=True, capture_output=True)
    for threads in ("1", "4"):
        env = dict(os.environ, HS_HOST_THREADS=threads)
        out = subprocess.run([exe], env=env, capture_output=True, text=True,
                             timeout=300)
        assert out.returncode == 0 and "fails 0" in out.stdout, out.stdout
