"""Parity at the benchmark's full size (BASELINE.json config: WS200, 16.8 M
candidates per step) through size-independent properties: the C oracle
(oracle/hs_oracle.c, pinned to the reference) checks a random sample of the
rows bit-for-bit, and the rest is covered by identities that must hold for
any batch -- the fused first-index argmin equals the argmin of the returned
makespans, rows evaluate independently of their position (permutation and
shard invariance), and the host-buffer and packed-genome entry points return
the device path's bits."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import instance_doc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2308_00127_b200 as hs  # noqa: E402
from paper_2308_00127_b200 import _native as N  # noqa: E402
from paper_2308_00127_b200.plan import get_plan  # noqa: E402
from oracle import hs_oracle as O  # noqa: E402
from oracle.hs_oracle_c import CTables  # noqa: E402

N_FULL = 1 << 24  # bench.py's candidates per GPU per step


@pytest.fixture(scope="module")
def full():
    doc = instance_doc("ws200")
    g, hw, t = hs.load_instance(doc)
    plan = get_plan(g, hw, t, 1)
    plan.specialize()
    gen = torch.Generator(device="cuda")
    gen.manual_seed(99)
    genes = torch.randint(0, plan.K, (N_FULL, plan.pref_ld), dtype=torch.uint8,
                          device="cuda", generator=gen)
    ms = torch.empty(N_FULL, dtype=torch.float64, device="cuda")
    st = torch.empty(N_FULL, dtype=torch.uint8, device="cuda")
    best = torch.empty(2, dtype=torch.int64, device="cuda")
    plan.eval(genes, ms, st, best)
    torch.cuda.synchronize()
    tb = O.build_tables(O.Instance.from_doc(doc), 1)
    yield plan, genes, ms, st, best, tb
    del genes, ms, st
    torch.cuda.empty_cache()


def test_sample_vs_c_oracle(full, oracle_lib):
    plan, genes, ms, st, _, tb = full
    rows = np.sort(np.random.default_rng(5).choice(N_FULL, 50_000,
                                                   replace=False))
    # include the first and last tiles and the ragged tail
    rows = np.unique(np.concatenate([rows, np.arange(300),
                                     np.arange(N_FULL - 300, N_FULL)]))
    idx = torch.from_numpy(rows).cuda()
    sample = genes[idx, :plan.V].cpu().numpy()
    want, wst = CTables(tb).fitness(oracle_lib, sample, threads=8)
    assert np.array_equal(st[idx].cpu().numpy(), wst)
    assert np.array_equal(ms[idx].cpu().numpy().view(np.uint64),
                          want.view(np.uint64))


def test_fused_argmin_is_first_argmin(full):
    _, _, ms, _, best, _ = full
    m = ms.cpu().numpy()
    cost = float(best[:1].cpu().view(torch.float64).item())
    index = int(best[1].item())
    assert (cost, index) == O.argmin_first(m)


def test_shards_and_permutation(full):
    plan, genes, ms, _, best, _ = full
    # 8 contiguous shards with global index bases merge to the full best
    # (the multi-GPU decomposition, dist.py / bench.py)
    shard = N_FULL // 8
    parts = []
    b = torch.empty(2, dtype=torch.int64, device="cuda")
    for r in range(8):
        plan.eval(genes[r * shard:(r + 1) * shard], None, None, b,
                  index_base=r * shard)
        bb = b.cpu()
        parts.append((float(bb[:1].view(torch.float64).item()),
                      int(bb[1].item())))
    full_best = (float(best[:1].cpu().view(torch.float64).item()),
                 int(best[1].item()))
    assert min(parts) == full_best
    # a permuted batch evaluates to the permuted makespans
    n = 1 << 20
    perm = torch.randperm(n, device="cuda")
    pm = torch.empty(n, dtype=torch.float64, device="cuda")
    plan.eval(genes[:n][perm].contiguous(), pm, None, None)
    assert torch.equal(pm.view(torch.int64), ms[:n][perm].view(torch.int64))


def test_host_and_packed_paths(full):
    plan, genes, ms, _, _, _ = full
    n = 1 << 20
    rows = genes[:n, :plan.V].cpu().numpy()
    hm = np.empty(n, np.float64)
    hb = N.Best()
    plan.eval_host(np.ascontiguousarray(genes[:n].cpu().numpy()), hm, None,
                   hb)
    want = ms[:n].cpu().numpy()
    assert np.array_equal(hm.view(np.uint64), want.view(np.uint64))
    assert (hb.cost, hb.index) == O.argmin_first(want)
    packed = hs.pack_genes(rows)
    hm2 = np.empty(n, np.float64)
    plan.eval_host_packed(packed, hm2, None, hb)
    assert np.array_equal(hm2.view(np.uint64), want.view(np.uint64))
    hm3 = np.empty(n, np.float64)
    hb3 = N.Best()
    plan.eval_host_packed3(hs.pack_genes3(rows), hm3, None, hb3)
    assert np.array_equal(hm3.view(np.uint64), want.view(np.uint64))
    assert (hb3.cost, hb3.index) == O.argmin_first(want)
