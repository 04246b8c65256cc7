"""Wall time of hs_eval_host on WS200 with uint8 rows in pinned host memory
(the bench's e2e call), per packing policy; HS_PACK_TRACE=1 adds the
library's per-phase split of the host-packing pipeline.

    python tools/e2e_probe.py [n] [reps]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2308_00127_b200 as hs  # noqa: E402
from paper_2308_00127_b200 import _native as N  # noqa: E402
from paper_2308_00127_b200.plan import get_plan  # noqa: E402
from conftest import instance_doc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 23
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
g, hw, t = hs.load_instance(instance_doc("ws200"))
hs.specialize(g, hw, t, 1)
plan = get_plan(g, hw, t, 1)
hp = torch.empty((n, plan.V), dtype=torch.uint8, pin_memory=True)
hp.numpy()[:] = np.random.default_rng(0).integers(3, size=(n, plan.V), dtype=np.uint8)
hm = torch.empty(n, dtype=torch.float64, pin_memory=True)
b = N.Best()
for pol in ("1", "0"):
    os.environ["HS_HOST_PACK"] = pol
    plan.eval_host(hp.numpy(), hm.numpy(), None, b)
    walls = []
    for _ in range(reps):
        w0 = time.perf_counter()
        plan.eval_host(hp.numpy(), hm.numpy(), None, b)
        walls.append(time.perf_counter() - w0)
    w = sorted(walls)[len(walls) // 2]
    print(f"HS_HOST_PACK={pol}: median {w * 1e3:.2f} ms, {n / w:.3g} cand/s "
          f"(runs {[round(x * 1e3, 1) for x in walls]})", flush=True)
