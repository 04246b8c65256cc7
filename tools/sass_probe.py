"""Offline SASS probe of the graph-specialised evaluator (no GPU): emit the
kernel source for an instance with HS_JIT_OPTS, compile it for sm_100a with
nvcc (the flags NVRTC uses) and print the opcode histogram of hs_jit_eval.

    HS_JIT_OPTS=tcols=170,regs=40 python tools/sass_probe.py ws200 384
"""
import collections
import json
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2308_00127_b200 as hs  # noqa: E402
from paper_2308_00127_b200.plan import Plan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "ws200"
lanes = int(sys.argv[2]) if len(sys.argv) > 2 else 384
fun = sys.argv[3] if len(sys.argv) > 3 else "hs_jit_eval"
with open(os.path.join(ROOT, "tests", "golden", "instances", name + ".json")) as f:
    doc = json.load(f)
p = Plan(*hs.load_instance(doc), 1)
src = p.specialized_source(lanes)
d = tempfile.mkdtemp()
cu = os.path.join(d, "k.cu")
with open(cu, "w") as f:
    f.write(src)
cub = os.path.join(d, "k.cubin")
subprocess.run(["nvcc", "-cubin", "-arch", "sm_100a", "--fmad=false",
                "-std=c++17", "-I", os.path.join(ROOT, "paper_2308_00127_b200",
                                                 "csrc"), cu, "-o", cub],
               check=True)
sass = subprocess.run(["cuobjdump", "-sass", "-fun", fun, cub],
                      capture_output=True, text=True).stdout
ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", sass)
c = collections.Counter(ops)
print(name, fun, "instructions", sum(c.values()))
print(" ".join(f"{k}:{v}" for k, v in c.most_common(30)))
if os.environ.get("SASS_OUT"):
    with open(os.environ["SASS_OUT"], "w") as f:
        f.write(sass)
