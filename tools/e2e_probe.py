"""Breakdown of the host-buffer (e2e) path on WS200: pinned H2D / D2H
bandwidth at the chunk size hs_eval_host uses, device time of each input
format's kernel on one chunk, and the whole host call per format.

    python tools/e2e_probe.py [n]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_00127_b200 as hs  # noqa: E402
from paper_2308_00127_b200 import _native as N  # noqa: E402
from paper_2308_00127_b200.heuristics import get_plan  # noqa: E402
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import instance_doc  # noqa: E402


def ev_time(fn, reps=10):
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 23
    g, hw, t = hs.load_instance(instance_doc("ws200"))
    plan = get_plan(g, hw, t, 1)
    plan.specialize()
    V = plan.V
    chunk = 1 << 19
    rows = np.random.default_rng(0).integers(3, size=(n, V), dtype=np.uint8)
    fmts = {"packed3": (hs.pack_genes3(rows), plan.eval_packed3, plan.eval_host_packed3),
            "packed2": (hs.pack_genes(rows), plan.eval_packed, plan.eval_host_packed)}
    u8 = np.zeros((n, plan.pref_ld), np.uint8)
    u8[:, :V] = rows
    fmts["u8"] = (u8, plan.eval, plan.eval_host)
    dm = torch.empty(chunk, dtype=torch.float64, device="cuda")
    hm = torch.empty(n, dtype=torch.float64, pin_memory=True)
    for name, (src, dev_call, host_call) in fmts.items():
        hp = torch.empty(src.shape, dtype=torch.uint8, pin_memory=True)
        hp.numpy()[:] = src
        dp = torch.empty((chunk, src.shape[1]), dtype=torch.uint8, device="cuda")
        h2d = ev_time(lambda: dp.copy_(hp[:chunk], non_blocking=True))
        d2h = ev_time(lambda: hm[:chunk].copy_(dm, non_blocking=True))
        dp.copy_(hp[:chunk])
        kt = ev_time(lambda: dev_call(dp, dm, None, None))
        hb = N.Best()
        host_call(hp.numpy(), hm.numpy(), None, hb)
        w0 = time.perf_counter()
        for _ in range(3):
            host_call(hp.numpy(), hm.numpy(), None, hb)
        el = (time.perf_counter() - w0) / 3
        print(f"{name}: row {src.shape[1]} B; chunk {chunk}: H2D {h2d*1e6:.0f} us "
              f"({chunk*src.shape[1]/h2d/1e9:.1f} GB/s), D2H {d2h*1e6:.0f} us "
              f"({chunk*8/d2h/1e9:.1f} GB/s), kernel {kt*1e6:.0f} us "
              f"({chunk/kt:.3g} cand/s); host call n={n}: {el*1e3:.1f} ms "
              f"= {n/el:.3g} cand/s", flush=True)


if __name__ == "__main__":
    main()
