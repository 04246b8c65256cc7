"""One SA and one (1+1) EA run (budget 2000, WS 10x20 stack) through the
graph-specialised search kernels -- the target of an ncu capture:

    ncu --set full -k regex:hs_jit_sa -c 1 python tools/search_once.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2308_00127_b200 as hs  # noqa: E402
from conftest import instance_doc  # noqa: E402

g, hw, t = hs.load_instance(instance_doc(sys.argv[1] if len(sys.argv) > 1
                                         else "ws_stack_10x20"))
hs.specialize(g, hw, t, 1)
s = hs.simulated_annealing(g, hw, t, 1, seed=0, budget=2000)
e = hs.one_plus_one_ea(g, hw, t, 1, seed=0, budget=2000)
print("sa", s.objective, "ea", e.objective)
