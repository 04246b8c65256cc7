"""hs_best_allreduce (C ABI, capi.cu) over a real NCCL communicator: the
communicator torch's NCCL process group owns, world size 1 (one GPU per
gpurun box). The merge kernel must return the lexicographic (cost, index)
minimum over ranks -- here the rank's own best -- with the same bits, and
the NCCL path of bench.py's step must run end to end."""
from __future__ import annotations

import os
import socket

import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def comm():
    import torch
    import torch.distributed as dist
    from paper_2308_00127_b200.dist import nccl_comm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield nccl_comm()
    dist.destroy_process_group()


def test_best_allreduce_world1(comm):
    import numpy as np
    import torch
    from paper_2308_00127_b200.dist import best_allreduce_device
    for cost, idx in ((3.25, 17), (float("inf"), -1), (0.0, 0),
                      (1e300, (1 << 40) + 3)):
        bits = int(np.array([cost], np.float64).view(np.int64)[0])
        b = torch.tensor([bits, idx], dtype=torch.int64, device="cuda")
        out = torch.full((2,), 7, dtype=torch.int64, device="cuda")
        best_allreduce_device(b, out, comm, torch.cuda.current_stream())
        torch.cuda.synchronize()
        assert out.tolist() == [bits, idx]


def test_best_allreduce_after_eval(comm):
    """The bench step: fused argmin of a batch, then the NCCL merge."""
    import numpy as np
    import torch
    import paper_2308_00127_b200 as hs
    from conftest import instance_doc
    from paper_2308_00127_b200.dist import best_allreduce_device
    from paper_2308_00127_b200.plan import get_plan
    g, hw, t = hs.load_instance(instance_doc("ws200"))
    plan = get_plan(g, hw, t, 1)
    genes = torch.randint(0, 3, (100_000, plan.pref_ld), dtype=torch.uint8,
                          device="cuda")
    ms = torch.empty(100_000, dtype=torch.float64, device="cuda")
    best = torch.empty(2, dtype=torch.int64, device="cuda")
    gbest = torch.empty(2, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    plan.eval(genes, ms, None, best, index_base=5_000_000, stream=s)
    best_allreduce_device(best, gbest, comm, s)
    m = ms.cpu().numpy()
    k = int(np.argmin(m))
    got = gbest.cpu()
    assert float(got[:1].view(torch.float64).item()) == m[k]
    assert int(got[1]) == 5_000_000 + k


def test_best_allreduce_rejects_null():
    import ctypes as C
    from paper_2308_00127_b200 import _native as N
    assert N.load().hs_best_allreduce(None, None, None, None) != 0
