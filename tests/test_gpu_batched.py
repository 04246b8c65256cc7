"""Extended-genome (batched-variant) evaluator against the reference's own
bMET / bGreedy schedules and the pinned oracle restatement."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import fhex, golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2308_00127_b200 as hs  # noqa: E402
from paper_2308_00127_b200 import _native as N  # noqa: E402
from paper_2308_00127_b200.core import Schedule, ScheduledBatch  # noqa: E402
from paper_2308_00127_b200.plan import get_plan  # noqa: E402
from oracle import hs_batched as B  # noqa: E402
from oracle import hs_oracle as O  # noqa: E402


def test_reference_batched_schedules():
    checked = 0
    for e in golden("batched"):
        g, hw, t = hs.load_instance(e)
        L = e["L"]
        for algo in ("met", "greedy"):
            res = e[algo]
            if "error" in res:
                continue
            ref = Schedule(batches=tuple(
                ScheduledBatch(task=b[0], device=b[1], size=b[2],
                               inputs=tuple(b[3]), start=float.fromhex(b[4]))
                for b in res["batches"]), objective=0.0, input_count=L)
            genes = hs.batched_genes_from_schedule(ref, g, hw, t, L)
            s = hs.decode_batched(genes, g, hw, t, L)
            assert fhex(s.objective) == res["objective"]
            got = [[b.task, b.device, b.size, list(b.inputs), fhex(b.start)]
                   for b in s.batches]
            assert got == res["batches"]
            ms = hs.fitness_batched(np.array([genes], np.uint8), g, hw, t, L)
            assert fhex(ms[0]) == res["objective"]
            checked += 1
    assert checked > 150


def test_random_extended_genomes_vs_oracle():
    served = 0
    for e in golden("batched"):
        g, hw, t = hs.load_instance(e)
        L = e["L"]
        inst = O.Instance.from_doc(e)
        opts = B.options(inst, L)
        if not opts:
            continue
        rng = np.random.default_rng(served)
        genes = rng.integers(len(opts), size=(200, len(g.tasks)),
                             dtype=np.uint8)
        genes[0, 0] = len(opts)  # out of range -> GraphError status
        want = [B.eval_one(inst, L, opts, row) for row in genes]
        ms, st = hs.fitness_batched(torch.from_numpy(genes).cuda(), g, hw, t,
                                    L, return_status=True)
        ms, st = ms.cpu().numpy(), st.cpu().numpy()
        for r, (wm, ws) in enumerate(want):
            assert st[r] == ws, (e["name"], r)
            if ws == 0:
                assert ms[r] == wm, (e["name"], r)
        hm, hst = hs.fitness_batched(genes, g, hw, t, L, return_status=True)
        assert np.array_equal(hst, st)
        ok = st == 0
        assert np.array_equal(hm[ok], ms[ok])
        served += 1
    assert served > 60


def test_generated_extended_genomes():
    e = [x for x in golden("batched") if x["name"] == "ws30_L4"][0]
    g, hw, t = hs.load_instance(e)
    inst = O.Instance.from_doc(e)
    opts = B.options(inst, 4)
    plan = get_plan(g, hw, t, 4, None, ())
    n = 3000
    out = torch.empty((n, plan.V), dtype=torch.uint8, device="cuda")
    ms = torch.empty(n, dtype=torch.float64, device="cuda")
    plan.eval_gen(N.GEN_RANDOM, 3, 10, n, makespan=ms, genes_out=out)
    genes = O.gen_genes(3, 10, n, plan.V, len(opts))
    assert np.array_equal(out.cpu().numpy(), genes)
    want = np.array([B.eval_one(inst, 4, opts, r)[0] for r in genes])
    assert np.array_equal(ms.cpu().numpy(), want)
    cost, idx, best = hs.random_search_batched(g, hw, t, 4, n + 10, seed=3)
    allg = O.gen_genes(3, 0, n + 10, plan.V, len(opts))
    allw = np.array([B.eval_one(inst, 4, opts, r)[0] for r in allg])
    assert (cost, idx) == O.argmin_first(allw)
    assert best == [int(x) for x in allg[idx]]


def test_global_slot_tier_ws200():
    """WS200 at L=4 (3 parts per task): the per-part end times overflow
    shared memory and live in the global-memory slot tier."""
    from conftest import instance_doc
    doc = instance_doc("ws200")
    g, hw, t = hs.load_instance(doc)
    inst = O.Instance.from_doc(doc)
    opts = B.options(inst, 4)
    rng = np.random.default_rng(4)
    genes = rng.integers(len(opts), size=(300, len(g.tasks)), dtype=np.uint8)
    genes[1, 5] = len(opts)  # out of range -> GraphError status
    want = [B.eval_one(inst, 4, opts, row) for row in genes]
    ms, st = hs.fitness_batched(torch.from_numpy(genes).cuda(), g, hw, t, 4,
                                return_status=True)
    ms, st = ms.cpu().numpy(), st.cpu().numpy()
    for r, (wm, ws) in enumerate(want):
        assert st[r] == ws, r
        if ws == 0:
            assert fhex(ms[r]) == fhex(wm), r
    # generated extended genomes through the same tier
    plan = get_plan(g, hw, t, 4, None, ())
    n = 500
    gm = torch.empty(n, dtype=torch.float64, device="cuda")
    plan.eval_gen(N.GEN_RANDOM, 9, 0, n, makespan=gm)
    gg = O.gen_genes(9, 0, n, plan.V, len(opts))
    assert [fhex(x) for x in gm.cpu().numpy()] == \
        [fhex(B.eval_one(inst, 4, opts, r)[0]) for r in gg]


def _jit_env(monkeypatch):
    # specialise every batched plan the test builds, whatever the batch size
    monkeypatch.setenv("HS_JIT_MIN", "0")


def test_specialised_reference_batched_schedules(monkeypatch):
    """The graph-specialised K8 (jit.cpp, jit_emit_batched) reproduces the
    reference's bMET / bGreedy schedules: objective and every sub-batch
    start (trace kernel), on every golden instance it serves."""
    from paper_2308_00127_b200.batched import _plan
    _jit_env(monkeypatch)
    served = 0
    for e in golden("batched"):
        g, hw, t = hs.load_instance(e)
        L = e["L"]
        plan = _plan(g, hw, t, L, None)
        if not plan.jit_eligible():
            continue
        plan.specialize()
        served += 1
        for algo in ("met", "greedy"):
            res = e[algo]
            if "error" in res:
                continue
            ref = Schedule(batches=tuple(
                ScheduledBatch(task=b[0], device=b[1], size=b[2],
                               inputs=tuple(b[3]), start=float.fromhex(b[4]))
                for b in res["batches"]), objective=0.0, input_count=L)
            genes = hs.batched_genes_from_schedule(ref, g, hw, t, L)
            s = hs.decode_batched(genes, g, hw, t, L)
            assert fhex(s.objective) == res["objective"], (e["name"], algo)
            got = [[b.task, b.device, b.size, list(b.inputs), fhex(b.start)]
                   for b in s.batches]
            assert got == res["batches"], (e["name"], algo)
    assert served >= 3


@pytest.mark.parametrize("name", ["ws30", "rn50f", "iv3f", "ws200"])
@pytest.mark.parametrize("L", [2, 4, 8])
def test_specialised_batched_equals_plan_walker(name, L):
    """Differential: specialised K8 against the plan-walking K8 (pinned to
    the reference above) on 60,000 random extended genomes, a few of them
    out of the option range."""
    from conftest import instance_doc
    from paper_2308_00127_b200.plan import Plan
    g, hw, t = hs.load_instance(instance_doc(name))
    jit = Plan(g, hw, t, L, batched=())
    aot = Plan(g, hw, t, L, batched=())
    if not jit.jit_eligible():
        pytest.skip("too many live part end times for the specialised K8")
    jit.specialize()
    no = len(jit.options)
    rng = np.random.default_rng(L)
    genes = rng.integers(no, size=(60_000, jit.pref_ld), dtype=np.uint8)
    genes[::997, 3] = no + 1  # out of range: status 5 on both
    d = torch.from_numpy(genes).cuda()
    out = []
    for plan in (jit, aot):
        ms = torch.empty(len(genes), dtype=torch.float64, device="cuda")
        st = torch.empty(len(genes), dtype=torch.uint8, device="cuda")
        plan.eval(d, ms, st, None)
        out.append((ms.cpu().numpy(), st.cpu().numpy()))
    assert np.array_equal(out[0][1], out[1][1])
    ok = out[0][1] < N.ST_MISSING
    assert np.array_equal(out[0][0][ok].view(np.uint64),
                          out[1][0][ok].view(np.uint64))
