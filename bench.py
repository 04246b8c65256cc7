"""Benchmark of the batched candidate-mapping evaluator (driver contract).

Workload (BASELINE.json north star): the 200-node randomly wired
Watts-Strogatz graph `gen_module("ws", 200, seed=0, k=4, p=0.75)` with
`synth_profile(DEFAULT3, seed=0)` (V=202, E=457, K=3, L=1), frozen from the
reference's own generator in tests/golden/instances/ws200.json. A step is one
pass of the evaluator over a batch of N synthetic uint8 candidate mappings
(explicit genomes resident in HBM, N*204 B >> 126 MB L2, so no L2 flush is
needed), producing every makespan plus the fused first-index argmin; with
--gpus N each rank evaluates its own N (weak scaling) and the global best
(cost, index) is combined on the device by hs_best_allreduce (one NCCL
all-gather of 16 B per rank + merge kernel). `--gpus N` without torchrun
re-launches itself under torch.distributed.run with N ranks.

`e2e` is the same metric through the public C ABI with HOST buffers in the
reference's layout (hs_eval_host: pinned uint8 genomes in, every makespan +
best out, copies inside the timed region); packed-genome variants are
reported beside it. The north_star's other configurations (WS30, RN50f /
IV3f at L in {1,2,4,8} incl. the batched variant, WS1000 and WS stacks, the
96-layer transformer, the split heuristic with its lower-bound gap, the
1e6..1e9 on-device sweep, search time-to-solution) are measured in the same
run. `cpu_baseline` runs the reference's own `hetsched.heuristics.fitness`
(imported unmodified from oracle/_ref) on the host cores, on a subset of the
very genomes the GPU scored, and checks them bit for bit; it also holds
every other CPU-side comparison. `--impl reference` is the reference arm.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from typing import Optional

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = "ws200"
METRIC = "candidate mappings scored/sec"
UNIT = "candidates/s"


def _load_doc():
    with open(os.path.join(ROOT, "tests", "golden", "instances",
                           WORKLOAD + ".json")) as f:
        return json.load(f)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _config(n, world):
    return {"workload": "ws200: gen_module('ws',200,seed=0,k=4,p=0.75) + "
                        "synth_profile(DEFAULT3,seed=0), V=202 E=457 K=3 L=1",
            "candidates_per_gpu_per_step": n,
            "genome_layout": "uint8 [N x 204] row-major (sorted-device index "
                             "per BFS position)",
            "l2": "inputs larger than L2 (N*204 B >> 126 MB); no flush",
            "parallelism": f"dp{world} (candidate shards, NCCL 16 B best "
                           "all-gather)"}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [],
                    "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if r[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# --------------------------------------------------------------- CPU legs
# The reference's own CPU path: hetsched.heuristics.fitness (heuristics.py:
# 127-148), imported unmodified through oracle/ref.py (oracle/_ref on the GPU
# box), in a warm fork pool -- workers are started, the instance is loaded
# and a few genomes are evaluated before any timed window opens.
_REF: dict = {}


def _ref_init(doc, L):
    from oracle import ref
    if ref.import_reference() is None:
        raise ImportError("reference hetsched not available")
    RC = sys.modules["hetsched.core"]
    RH = sys.modules["hetsched.heuristics"]
    g, hw, t = ref.load_instance(doc)
    _REF.update(g=g, hw=hw, t=t, L=L, RH=RH,
                order=tuple(RC.bfs_topological_order(g)))


def _ref_eval(args):
    import numpy as np
    buf, n, V = args
    genes = np.frombuffer(buf, np.uint8).reshape(n, V)
    RH, g, hw, t, L, order = (_REF[k] for k in ("RH", "g", "hw", "t", "L",
                                                "order"))
    out = np.empty(n, np.float64)
    t0 = time.perf_counter()
    for r in range(n):
        out[r] = RH.fitness(RH.MappingGenome(genes=tuple(genes[r].tolist()),
                                             order=order), g, hw, t, L)
    return out.tobytes(), time.perf_counter() - t0


class RefPool:
    """Warm pool of `cores` forked workers running the reference's fitness."""

    def __init__(self, doc, L: int = 1, cores: Optional[int] = None):
        import multiprocessing as mp
        import numpy as np
        self.cores = cores or len(os.sched_getaffinity(0))
        self.pool = mp.get_context("fork").Pool(
            self.cores, initializer=_ref_init, initargs=(doc, L))
        self.V = len(doc["order"])
        K = len(doc["devices_sorted"])
        warm = np.random.default_rng(99).integers(
            K, size=(4 * self.cores, self.V), dtype=np.uint8)
        _, wall, busy = self.fitness(warm)
        self.rate_per_core = 4 / max(busy / self.cores, 1e-9)

    def fitness(self, genes):
        """(makespans f64[n], wall s of the dispatch, summed worker s)."""
        import numpy as np
        genes = np.ascontiguousarray(genes[:, :self.V], np.uint8)
        n = len(genes)
        cuts = [n * k // self.cores for k in range(self.cores + 1)]
        jobs = [(genes[a:b].tobytes(), b - a, self.V)
                for a, b in zip(cuts, cuts[1:]) if b > a]
        t0 = time.perf_counter()
        res = self.pool.map(_ref_eval, jobs, chunksize=1)
        wall = time.perf_counter() - t0
        out = np.frombuffer(b"".join(r[0] for r in res), np.float64).copy()
        return out, wall, sum(r[1] for r in res)

    def close(self):
        self.pool.terminate()
        self.pool.join()


def c_port_rate(doc, cores):
    """The C restatement of the decoder (oracle/hs_oracle.c) on all host
    cores: the native CPU comparator."""
    import numpy as np
    from oracle import hs_oracle as O
    from oracle.hs_oracle_c import CTables, load
    tb = O.build_tables(O.Instance.from_doc(doc), 1)
    ct, lib = CTables(tb), load()
    genes = np.random.default_rng(5).integers(3, size=(400_000, tb.V),
                                              dtype=np.uint8)
    t0 = time.perf_counter()
    ct.fitness(lib, genes, cores)
    return len(genes) / (time.perf_counter() - t0)


def _inst(name):
    with open(os.path.join(ROOT, "tests", "golden", "instances",
                           name + ".json")) as f:
        return json.load(f)


def run_reference(args):
    """The reference arm: hetsched.heuristics.fitness itself (unmodified,
    oracle/_ref) on all host cores, warm pool, on this arm's workload and
    metric. Each step scores a fresh bounded sample of uniform WS200
    genomes sized so that warmup + steps take about a minute."""
    import numpy as np
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    doc = _load_doc()
    pool = RefPool(doc)
    cores, V, K = pool.cores, pool.V, len(doc["devices_sorted"])
    step_s = min(4.0, max(0.5, 60.0 / max(1, args.steps + args.warmup)))
    per_step = max(cores, int(pool.rate_per_core * cores * step_s))
    rng = np.random.default_rng(2024)
    vals, walls = [], []
    for s in range(args.warmup + args.steps):
        genes = rng.integers(K, size=(per_step, V), dtype=np.uint8)
        _, wall, _ = pool.fitness(genes)
        if s >= args.warmup:
            walls.append(wall)
            vals.append(per_step / wall)
    pool.close()
    v = per_step * len(walls) / sum(walls)
    out = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * sum(walls) / len(walls),
           "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (uniform random genomes; reference benchgen "
                   "graph frozen as JSON)",
           # the same workload description as the GPU arm (each timed step
           # here scores a bounded sample of it: cpu_baseline.sample)
           "config": _config(args.n, args.gpus),
           "evaluator": "hetsched.heuristics.fitness (the reference, "
                        "unmodified), warm fork pool on the host cores",
           "cpu_baseline": {
               "value": v, "unit": UNIT, "cores": cores, "kind": "reference",
               "sample": f"{per_step} uniform WS200 genomes per step, "
                         "hetsched.heuristics.fitness (reference, unmodified, "
                         f"oracle/_ref) in a warm fork pool x{cores}; pool "
                         "start-up and instance load outside the timed "
                         "window",
               "per_step_values": vals},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


# ------------------------------------------------------------- launching
def _free_port():
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    return port


def _spawn_ranks(args):
    """`bench.py --gpus N` outside torchrun: re-run this command under
    torch.distributed.run with N ranks (one per GPU) and exit with its
    status; the ranks then find WORLD_SIZE == N."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    # torchrun's parser prefix-matches every "--x" token, so pass the
    # ambiguous alias --n under its full name
    argv = ["--candidates" + a[3:] if a == "--n" or a.startswith("--n=")
            else a for a in sys.argv[1:]]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__),
           *argv]
    sys.exit(subprocess.call(cmd))


def _world(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE "
                         f"{world}")
    return world, rank, local


def plumbing_only(args):
    """The multi-rank plumbing of the GPU arm without a GPU (gloo): each rank
    takes its contiguous shard of a synthetic batch, reduces it to a
    first-index (cost, index) best, and the ranks merge with the same
    all-gather + lexicographic rule as hs_best_allreduce. The per-candidate
    cost is a fixed integer hash (not an evaluation); this mode exists so
    the launch / rank / merge / report path is testable on CPU
    (tests/test_bench_dist.py)."""
    import numpy as np
    import torch.distributed as dist

    from paper_2308_00127_b200.dist import allgather_best, shard_range
    world, rank, _ = _world(args)
    if world > 1:
        dist.init_process_group("gloo")
    n = args.n
    lo, hi = shard_range(n, world, rank)
    idx = np.arange(lo, hi, dtype=np.uint64)
    cost = ((idx * np.uint64(0x9E3779B97F4A7C15)) >> np.uint64(54)) \
        .astype(np.float64)
    k = int(np.argmin(cost)) if hi > lo else -1
    local = (float(cost[k]), lo + k) if k >= 0 else (float("inf"), -1)
    best = allgather_best(local) if world > 1 else local
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT,
                          "n_gpus": world, "plumbing_only": True,
                          "candidates": n, "best": {"cost": best[0],
                                                    "index": best[1]}}))
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------- GPU arm
def _timed(stream, fn, reps):
    """Device time (ms) of `reps` calls of fn on `stream` (CUDA events)."""
    import torch
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for r in range(reps):
        fn(r)
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1)


def _ncu_profile():
    """Per-candidate DRAM bytes and warp instructions of the headline
    kernel, from the ncu capture of this very bench command committed under
    profiles/ (tools/ncu_summary.py writes it); None if absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "bench_kernel_ncu.json")) as f:
            return json.load(f)
    except Exception:
        return None


def graph_rates(stream, gen, world):
    """Device throughput of the same evaluator on the north_star's other
    graph families (explicit uint8 genomes resident in HBM)."""
    import torch

    import paper_2308_00127_b200 as hs
    from paper_2308_00127_b200.batched import _plan
    from paper_2308_00127_b200.plan import get_plan
    out = {}

    def rate(plan, nopt, on, jit=True):
        if jit and plan.jit_eligible():
            plan.specialize()
        genes = torch.randint(0, nopt, (on, plan.pref_ld), dtype=torch.uint8,
                              device="cuda", generator=gen)
        ms = torch.empty(on, dtype=torch.float64, device="cuda")
        b = torch.empty(2, dtype=torch.int64, device="cuda")
        for _ in range(2):
            plan.eval(genes, ms, None, b, stream=stream)
        t = _timed(stream, lambda r: plan.eval(genes, ms, None, b,
                                               stream=stream), 5)
        bb = b.cpu()
        best = float(bb[:1].view(torch.float64).item())
        del genes, ms
        return {"value": world * on * 5 / (t / 1e3), "unit": UNIT,
                "V": plan.V, "K": plan.K, "L": plan.L, "candidates": on,
                "kernel": ("hs_jit_eval" if plan.specialized_ms is not None
                           else ("hs::beval_kernel" if plan.batched
                                 else "hs::eval_kernel")),
                "best_makespan_ms": best,
                "best_throughput_per_s": (1000.0 * plan.L / best
                                          if best > 0 else None)}

    cases = [("ws30", 1), ("ws1000", 1), ("ws_stack_10x20", 1),
             ("ws_stack_10x100", 1), ("tf96", 1)]
    cases += [(nm, L) for nm in ("rn50f", "iv3f") for L in (1, 2, 4, 8)]
    for name, L in cases:
        key = f"{name}_L{L}"
        try:
            g, hw, t = hs.load_instance(_inst(name))
            plan = get_plan(g, hw, t, L)
            on = 1 << (20 if plan.V > 512 else 22)
            out[key] = rate(plan, plan.K, on)
            if plan.specialized_ms is not None:
                out[key]["specialise_ms_not_timed"] = plan.specialized_ms
        except Exception as exc:  # reported, never fatal for the bench
            out[key] = {"error": repr(exc)}
    # batched variant (K8): extended genomes, throughput objective
    for name in ("rn50f", "iv3f", "ws200"):
        for L in (2, 4, 8):
            key = f"{name}_batched_L{L}"
            try:
                g, hw, t = hs.load_instance(_inst(name))
                plan = _plan(g, hw, t, L, None)
                out[key] = rate(plan, len(plan.options), 1 << 22)
                out[key]["options"] = len(plan.options)
                out[key]["parts"] = plan.max_parts
            except Exception as exc:
                out[key] = {"error": repr(exc)}
    torch.cuda.empty_cache()
    return out


def n_sweep(stream, world, rank, comm):
    """Config 5: 1e6 .. 1e9 on-device generated WS200 candidates
    (hs_eval_gen: oracle.gen_genes's counter hash, genomes never
    touch HBM), this rank's contiguous shard, best merged over ranks on the
    device; a few sampled candidates' genomes and makespans are kept for the
    CPU re-scoring in cpu_baseline."""
    import numpy as np
    import torch

    import paper_2308_00127_b200 as hs
    from paper_2308_00127_b200 import _native as N
    from paper_2308_00127_b200.dist import (best_allreduce_device, merge_best,
                                            shard_range)
    from paper_2308_00127_b200.plan import get_plan
    g, hw, t = hs.load_instance(_inst("ws200"))
    plan = get_plan(g, hw, t, 1)
    plan.specialize()
    best = torch.empty(2, dtype=torch.int64, device="cuda")
    gbest = torch.empty(2, dtype=torch.int64, device="cuda")
    seed = 2308
    chunk = 1 << 28
    plan.eval_gen(N.GEN_RANDOM, seed, 0, 1 << 20, best=best, stream=stream)
    out = {}
    for total in (10**6, 10**7, 10**8, 10**9):
        lo, hi = shard_range(total, world, rank)

        def run(_r):
            parts = []
            for c in range(lo, hi, chunk):
                m = min(chunk, hi - c)
                plan.eval_gen(N.GEN_RANDOM, seed, c, m, best=best,
                              stream=stream)
                bb = best.cpu()
                parts.append((float(bb[:1].view(torch.float64).item()),
                              int(bb[1].item())))
            # this rank's chunk bests, same rule as the device merge
            c, i = merge_best(parts)
            bits = int(np.array([c], np.float64).view(np.int64)[0])
            best.copy_(torch.tensor([bits, i], dtype=torch.int64))
            if comm is not None:
                best_allreduce_device(best, gbest, comm, stream)
            else:
                gbest.copy_(best)

        torch.cuda.synchronize()
        # the whole shard incl. the host-side chunk merge; median of 5 runs
        # below 1e9 (a 1e6 run is ~0.3 ms, within host jitter)
        runs = [_timed(stream, run, 1) for _ in range(5 if total < 10**9 else 1)]
        ms = sorted(runs)[len(runs) // 2]
        gb = gbest.cpu()
        out[f"n_{total:.0e}"] = {
            "candidates": total, "ms": ms, "runs_ms": runs,
            "value": total / (ms / 1e3), "unit": UNIT,
            "best": {"cost_ms": float(gb[:1].view(torch.float64).item()),
                     "index": int(gb[1].item())}}
    # device makespans + genomes of sampled indices (checked on the CPU)
    samples = [0, 1, 12345, 10**6 - 1, 10**8 + 7, 10**9 - 1]
    samples.append(out["n_1e+09"]["best"]["index"])
    rows = torch.empty((len(samples), plan.V), dtype=torch.uint8,
                       device="cuda")
    mk = torch.empty(len(samples), dtype=torch.float64, device="cuda")
    for k, c in enumerate(samples):
        plan.eval_gen(N.GEN_RANDOM, seed, c, 1, makespan=mk[k:k + 1],
                      genes_out=rows[k:k + 1], stream=stream)
    torch.cuda.synchronize()
    return out, {"seed": seed, "index": samples,
                 "genes": rows.cpu().numpy(), "makespan": mk.cpu().numpy()}


def split_config3():
    """Config 3: the split heuristic on the WS 10x20 stack -- the module
    decomposition (native k-edge components), the DP over endpoint pinnings
    with the GPU module solver, every returned schedule validated on the
    GPU -- and the lower-bound gap (critical-path recursion, subgraph_cap=0:
    no MILP in this package)."""
    import paper_2308_00127_b200 as hs
    g, hw, t = hs.load_instance(_inst("ws_stack_10x20"))
    out = {}
    t0 = time.perf_counter()
    dec = hs.k_edge_components(g, 1)
    t1 = time.perf_counter()
    sched = hs.milp_split(g, hw, t, 1, dec,
                          module_solver=hs.gpu_module_solver(), workers=8)
    t2 = time.perf_counter()
    mk = hs.validate_schedule(g, hw, t, sched)
    lb = hs.lower_bound(g, hw, t, 1, dec, subgraph_cap=0)
    t3 = time.perf_counter()
    q1 = hs.decomposition_modularity(g, dec)
    dq, qq = hs.modularity_split(g, 1)
    out["modularity"] = {"k_edge_components_c1": q1,
                         "after_modularity_merges": qq,
                         "modules_after_merges": len(dq.modules)}
    out.update({
        "instance": "ws_stack_10x20 (V=220, 10 modules)",
        "modules": len(dec.modules), "decompose_s": t1 - t0,
        "split_s": t2 - t1, "objective_ms": sched.objective,
        "validated_makespan_ms": mk, "flags": list(sched.flags),
        "lower_bound_ms": lb.lower_bound_ms, "lower_bound_s": t3 - t2,
        "gap": sched.objective / lb.lower_bound_ms - 1.0
        if lb.lower_bound_ms > 0 else None,
        "context": {"reference_milp_split_ms": 3685.67,
                    "reference_milp_split_s": 50.2,
                    "reference_heft_ms": 2263.1,
                    "reference_lower_bound_cap40_ms": 1878.24,
                    "source": "SURVEY.md 3(3) / 6 (survey-measured, CPU)"}})
    # the 1000-node stack (V=1020): split with sampled module sweeps
    g, hw, t = hs.load_instance(_inst("ws_stack_10x100"))
    t0 = time.perf_counter()
    dec = hs.k_edge_components(g, 1)
    sched = hs.milp_split(g, hw, t, 1, dec,
                          module_solver=hs.gpu_module_solver(), workers=8)
    t1 = time.perf_counter()
    mk = hs.validate_schedule(g, hw, t, sched)
    lb = hs.lower_bound(g, hw, t, 1, dec, subgraph_cap=0)
    out["ws_stack_10x100"] = {
        "instance": "ws_stack_10x100 (V=1020, 10 modules)",
        "modules": len(dec.modules), "split_s": t1 - t0,
        "objective_ms": sched.objective, "validated_makespan_ms": mk,
        "lower_bound_ms": lb.lower_bound_ms,
        "gap": sched.objective / lb.lower_bound_ms - 1.0
        if lb.lower_bound_ms > 0 else None}
    return out


def _genome_sha(s, hw):
    import hashlib
    devs = sorted(hw.devices)
    return hashlib.sha1(bytes(devs.index(b.device) for b in s.batches)
                        ).hexdigest()[:16]


def search_tts(names=("ws_stack_10x20", "ws200", "tf96"), budget=2000,
               seed=0):
    """Heuristic time-to-solution on the GPU: SA (K10) and (1+1) EA (K9) as
    trajectory-exact device launches, whole runs (start heuristic and final
    decode included), warm, 10 runs each; the CPU comparisons (the
    reference's own SA / EA) are in cpu_baseline."""
    import paper_2308_00127_b200 as hs
    from paper_2308_00127_b200.heuristics import _last_chain_stats
    out = {}
    for name in names:
        g, hw, t = hs.load_instance(_inst(name))
        spec_ms = hs.specialize(g, hw, t, 1)
        for algo in ("sa", "ea"):
            fn = hs.simulated_annealing if algo == "sa" else \
                hs.one_plus_one_ea
            s = fn(g, hw, t, 1, seed=seed, budget=budget)  # warm
            runs = []
            for _ in range(10):
                t0 = time.perf_counter()
                s2 = fn(g, hw, t, 1, seed=seed, budget=budget)
                runs.append(time.perf_counter() - t0)
                assert s2 == s
            out[f"{algo}_{name}_budget{budget}"] = {
                "gpu_s": statistics.median(runs), "gpu_runs_s": runs,
                "max_over_median": max(runs) / statistics.median(runs),
                "objective_ms": s.objective,
                "genome_sha1": _genome_sha(s, hw),
                "device_rounds": _last_chain_stats.get(f"{algo}_rounds"),
                "specialise_ms_not_timed": spec_ms}
    # multi-start: 148 independent chains (seeds 0..147), one per SM, in
    # one launch; chain c equals the single run at seed c
    for name in names:
        g, hw, t = hs.load_instance(_inst(name))
        # the graph-specialised body, like the single-chain runs above (a
        # freshly loaded instance is a new plan)
        hs.specialize(g, hw, t, 1)
        for algo in ("sa", "ea"):
            fn = hs.simulated_annealing_multi if algo == "sa" else \
                hs.one_plus_one_ea_multi
            seeds = list(range(148))
            fn(g, hw, t, 1, seeds[:2], budget=budget)  # warm
            runs = []
            for _ in range(3):
                t0 = time.perf_counter()
                res = fn(g, hw, t, 1, seeds, budget=budget)
                runs.append(time.perf_counter() - t0)
            best = min(range(len(res)), key=lambda c: (res[c].objective, c))
            out[f"{algo}_multi148_{name}_budget{budget}"] = {
                "gpu_s": statistics.median(runs), "gpu_runs_s": runs,
                "chains": len(seeds), "seeds": "0..147",
                "best_objective_ms": res[best].objective, "best_seed": best,
                "seed0_objective_ms": res[0].objective,
                "single_chain_gpu_s": out[f"{algo}_{name}_budget{budget}"]
                ["gpu_s"]}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--candidates", "--n", dest="n", type=int,
                    default=1 << 24, help="candidates per GPU per step")
    ap.add_argument("--e2e-n", type=int, default=1 << 23)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-tts", action="store_true")
    ap.add_argument("--no-others", action="store_true",
                    help="skip the other configurations")
    ap.add_argument("--no-jit", action="store_true",
                    help="time the ahead-of-time kernel instead of the "
                         "graph-specialised one")
    ap.add_argument("--plumbing-only", action="store_true",
                    help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    _spawn_ranks(args)
    if args.plumbing_only:
        plumbing_only(args)
        return
    world, rank, local = _world(args)

    import numpy as np
    import torch

    import paper_2308_00127_b200 as hs
    from paper_2308_00127_b200 import _native as N
    from paper_2308_00127_b200.dist import best_allreduce_device, nccl_comm
    from paper_2308_00127_b200.plan import get_plan

    torch.cuda.set_device(local)
    dist = None
    comm = None
    if world > 1:
        import torch.distributed as dist
        # NCCL's init log lets the driver count the ranks of the communicator
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = nccl_comm()

    doc = _load_doc()
    g, hw, table = hs.load_instance(doc)
    plan = get_plan(g, hw, table, 1)
    jit_ms = None
    if not args.no_jit:
        jit_ms = plan.specialize()  # NVRTC, once per plan (not timed)
    V, ld, n = plan.V, plan.pref_ld, args.n
    stream = torch.cuda.current_stream()
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1234 + rank)
    genes = torch.randint(0, plan.K, (n, ld), dtype=torch.uint8,
                          device="cuda", generator=gen)
    ms = torch.empty(n, dtype=torch.float64, device="cuda")
    best = torch.empty(2, dtype=torch.int64, device="cuda")
    gbest = torch.empty(2, dtype=torch.int64, device="cuda")

    def step():
        plan.eval(genes, ms, None, best, index_base=rank * n, stream=stream)
        if comm is not None:
            best_allreduce_device(best, gbest, comm, stream)

    evs = [(torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.3)  # the sampler is up before the GPU work starts
        # the warm-up steps run right before the timed ones (no idle gap in
        # which the clocks could settle lower)
        for _ in range(max(args.warmup, 3)):
            step()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t0.record(stream)
        for k in range(args.steps):
            evs[k][0].record(stream)
            plan.eval(genes, ms, None, best, index_base=rank * n,
                      stream=stream)
            evs[k][1].record(stream)
            if comm is not None:
                best_allreduce_device(best, gbest, comm, stream)
        t1.record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    total_ms = t0.elapsed_time(t1)
    kern_ms = statistics.mean(a.elapsed_time(b) for a, b in evs)
    if dist is not None:
        tt = torch.tensor([total_ms, kern_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms, kern_ms = float(tt[0]), float(tt[1])
        b = gbest.cpu()
    else:
        b = best.cpu()
    bcost, bidx = float(b[:1].view(torch.float64).item()), int(b[1].item())
    ms_step = total_ms / args.steps
    value = world * n / (ms_step / 1e3)
    clocks = clk.summary()

    # ---- roofline of the dominant kernel: algorithmic bytes per launch /
    # its CUDA-event duration (HBM), and the issue fraction from the ncu
    # warp-instruction count of the same kernel (profiles/)
    peak, peak_kind = _peaks()
    achieved = n * (V + 8) / (kern_ms / 1e3) / 1e9
    prof = _ncu_profile()
    traffic = issue = None
    if prof:
        if prof.get("dram_bytes_per_candidate"):
            traffic = prof["dram_bytes_per_candidate"] * n
        ipc_cand = prof.get("warp_inst_per_candidate")
        sm_mhz = clocks.get("sm_mhz") or 1965.0
        if ipc_cand:
            issued = ipc_cand * n / (kern_ms / 1e3)  # warp-instr / s
            cap = 4 * 148 * sm_mhz * 1e6
            issue = {"warp_inst_per_candidate": ipc_cand,
                     "achieved_warp_inst_per_s": issued,
                     "peak_warp_inst_per_s": cap, "frac": issued / cap,
                     "basis": "4 issue slots/clk x 148 SMs x median SM clock "
                              "sampled during the timed region"}

    # ---- e2e through the C ABI with host buffers (pinned): genomes in the
    # reference layout go host -> device every step, makespans + best come
    # back every step
    ne = min(args.e2e_n, n)
    hb = N.Best()
    host_rows = genes[:ne, :V].cpu().numpy()
    hm = torch.empty(ne, dtype=torch.float64, pin_memory=True)
    hmn = hm.numpy()
    variants = {}
    ref_ms = ms[:ne].cpu().numpy()
    default_packs = plan.eval_host_packs(ne)
    for kind in ("u8", "u8_dma", "u8_host_pack", "packed3", "packed2"):
        t_pack = None
        # "u8": the library's default policy; the other two force it
        os.environ.pop("HS_HOST_PACK", None)
        if kind in ("u8_dma", "u8_host_pack"):
            os.environ["HS_HOST_PACK"] = "1" if kind == "u8_host_pack" else "0"
        if kind == "packed3":
            tp = time.perf_counter()
            src = hs.pack_genes3(host_rows)
            t_pack = time.perf_counter() - tp
            call = plan.eval_host_packed3
        elif kind == "packed2":
            tp = time.perf_counter()
            src = hs.pack_genes(host_rows)
            t_pack = time.perf_counter() - tp
            call = plan.eval_host_packed
        else:  # u8, u8_dma, u8_host_pack
            src = np.zeros((ne, ld), np.uint8)
            src[:, :V] = host_rows
            call = plan.eval_host
        hp = torch.empty(src.shape, dtype=torch.uint8, pin_memory=True)
        hp.numpy()[:] = src
        hpn = hp.numpy()
        for _ in range(2):
            call(hpn, hmn, None, hb, stream=stream)
        torch.cuda.synchronize()
        els = []
        for _ in range(max(3, min(args.steps, 7))):
            w0 = time.perf_counter()
            call(hpn, hmn, None, hb, stream=stream)
            els.append(time.perf_counter() - w0)
        el = statistics.median(els)
        if dist is not None:
            tt = torch.tensor([el], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            el = float(tt[0])
        # the host path returns exactly the device path's makespans
        assert np.array_equal(hmn.view(np.uint64), ref_ms.view(np.uint64))
        variants[kind] = {"value": world * ne / el, "unit": UNIT,
                          "h2d_bytes_per_step": int(src.nbytes),
                          "d2h_bytes_per_step": ne * 8 + 16,
                          "candidates_per_step": ne}
        if kind == "u8_host_pack" or (kind == "u8" and default_packs):
            # what crosses PCIe: the 2-bit rows the call packs on the host
            variants[kind]["h2d_bytes_per_step"] = ne * plan.packed_ld()
            variants[kind]["host_input_bytes_per_step"] = int(src.nbytes)
        if t_pack is not None:
            variants[kind]["pack_included"] = False
            variants[kind]["host_pack_s_per_step"] = t_pack
            variants[kind]["value_with_host_pack"] = world * ne / (el + t_pack)
        del hp, src
    os.environ.pop("HS_HOST_PACK", None)
    e2e = dict(variants["u8"])
    e2e["api"] = ("hs_eval_host (C ABI, default policy): pinned host uint8 "
                  "genomes in the reference layout (one byte per gene) in, "
                  "every makespan + best out, chunked H2D/kernel/D2H on 2 "
                  "streams; median wall clock per call; "
                  + ("rows packed to 2 bits per gene by host threads inside "
                     "the call" if default_packs else "rows copied as bytes"))
    e2e["host_packs"] = bool(default_packs)
    e2e["host_threads"] = os.cpu_count()
    e2e["u8_dma"] = dict(
        variants["u8_dma"],
        note="HS_HOST_PACK=0: the uint8 rows cross PCIe as they are")
    e2e["u8_host_packed_in_call"] = dict(
        variants["u8_host_pack"], host_threads=os.cpu_count(),
        note="HS_HOST_PACK=1: host threads pack to 2 bits inside the call")
    e2e["packed3_genomes"] = variants["packed3"]
    e2e["packed2_genomes"] = variants["packed2"]
    del hm
    torch.cuda.empty_cache()

    # ---- the other configurations
    others, sweep, sweep_samples, split, tts = {}, None, None, None, None
    if not args.no_others:
        others = graph_rates(stream, gen, world)
        try:
            sweep, sweep_samples = n_sweep(stream, world, rank, comm)
        except Exception as exc:  # reported, never fatal for the bench
            sweep = {"error": repr(exc)}
    if rank == 0 and not args.no_others:
        try:
            split = split_config3()
        except Exception as exc:
            split = {"error": repr(exc)}
    if rank == 0 and not args.no_tts:
        try:
            tts = search_tts()
        except Exception as exc:
            tts = {"error": repr(exc)}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    cpu = None
    if not args.no_cpu:
        cpu = cpu_legs(doc, genes[:, :V], ms, sweep_samples, tts)

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (uniform random genomes; "
                                "reference benchgen graph frozen as JSON)",
        "config": _config(n, world),
        "evaluator": ("graph-specialised hs_jit_eval (NVRTC sm_100a, compiled "
                      f"once in {jit_ms:.0f} ms, not timed)")
        if jit_ms is not None else "ahead-of-time plan walker",
        "best": {"cost_ms": bcost, "index": bidx},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak,
                     "peak_kind": peak_kind, "traffic": traffic,
                     "algorithmic_bytes_per_candidate": V + 8,
                     "kernel_ms": kern_ms,
                     "kernel": "hs_jit_eval" if jit_ms is not None
                     else "hs::eval_kernel",
                     "issue": issue,
                     "ncu_source": prof.get("source") if prof else None,
                     "sm_utilisation": prof.get("sm_utilisation")
                     if prof else None},
        "cpu_baseline": cpu, "e2e": e2e,
        "n_sweep": sweep, "other_graphs": others, "split": split,
        "time_to_solution": tts,
        "gpu_launches": args.steps * (3 if comm is not None else 1),
        "clocks": clocks,
    }
    print(json.dumps(out))
    if dist is not None:
        dist.destroy_process_group()


def cpu_legs(doc, d_genes, d_ms, sweep_samples, tts):
    """Everything that runs on the host CPU, rank 0, N=1 semantics: the
    reference's own fitness on the first genomes of the timed batch (rate
    and bit-for-bit check against the GPU makespans), the C port, the
    sampled on-device-generated candidates re-scored by the reference, and
    the reference's own SA / EA against the GPU search results."""
    import numpy as np
    cores = len(os.sched_getaffinity(0))
    out = {}
    pool = RefPool(doc)
    try:
        m = int(min(len(d_genes),
                    max(10_000, pool.rate_per_core * cores * 12.0)))
        rows = d_genes[:m].cpu().numpy()
        want, wall, _ = pool.fitness(rows)
        got = d_ms[:m].cpu().numpy()
        mism = int(np.count_nonzero(want.view(np.uint64) !=
                                    got.view(np.uint64)))
        out = {"value": m / wall, "unit": UNIT, "cores": cores,
               "kind": "reference",
               "sample": f"the first {m} genomes of the timed WS200 batch, "
                         "hetsched.heuristics.fitness (the reference, "
                         "unmodified, oracle/_ref), warm fork pool "
                         f"x{cores}, {wall:.1f} s",
               "same_run_check": {"candidates": m, "mismatches": mism,
                                  "bit_exact": mism == 0,
                                  "checker": "reference fitness vs GPU "
                                             "makespans, float64 bits"}}
        if sweep_samples is not None:
            from oracle import hs_oracle as O
            gg = np.vstack([O.gen_genes(sweep_samples["seed"], c, 1, pool.V,
                                        len(doc["devices_sorted"]))
                            for c in sweep_samples["index"]])
            same_genes = bool(np.array_equal(gg, sweep_samples["genes"]))
            ref_ms, _, _ = pool.fitness(gg)
            out["n_sweep_check"] = {
                "index": sweep_samples["index"], "genes_equal": same_genes,
                "makespans_equal": bool(np.array_equal(
                    ref_ms.view(np.uint64),
                    sweep_samples["makespan"].view(np.uint64)))}
    finally:
        pool.close()
    try:
        out["c_port_all_cores"] = {"value": c_port_rate(doc, cores),
                                   "unit": UNIT, "cores": cores,
                                   "kind": "port (oracle/hs_oracle.c)"}
    except Exception as exc:
        out["c_port_all_cores"] = {"error": repr(exc)}
    if isinstance(tts, dict) and "error" not in tts:
        out["time_to_solution"] = reference_search(tts)
    try:
        out["split_comparators"] = reference_constructive()
    except Exception as exc:
        out["split_comparators"] = {"error": repr(exc)}
    return out


def reference_constructive():
    """The reference's own HEFT and greedy (heuristics.py:192-256) on the
    split instances, as the comparators of the GPU split's objective."""
    from oracle import ref
    ref.import_reference()
    RH = sys.modules["hetsched.heuristics"]
    out = {}
    for name in ("ws_stack_10x20", "ws_stack_10x100"):
        g, hw, t = ref.load_instance(_inst(name))
        row = {}
        for algo in ("heft", "greedy"):
            t0 = time.perf_counter()
            s = getattr(RH, algo)(g, hw, t, 1)
            row[algo] = {"objective_ms": s.objective,
                         "s": time.perf_counter() - t0}
        out[name] = row
    return out


def _ref_search_job(args):
    name, algo, budget, seed = args
    from oracle import ref
    ref.import_reference()
    RH = sys.modules["hetsched.heuristics"]
    g, hw, t = ref.load_instance(_inst(name))
    fn = RH.simulated_annealing if algo == "sa" else RH.one_plus_one_ea
    t0 = time.perf_counter()
    s = fn(g, hw, t, 1, seed=seed, budget=budget)
    el = time.perf_counter() - t0
    return s.objective, _genome_sha(s, hw), el


def reference_search(tts):
    """The reference's own simulated_annealing / one_plus_one_ea (one core
    each, in parallel processes) on the GPU runs' instances and seeds:
    wall time and the final schedule, which must be the GPU's."""
    import multiprocessing as mp
    jobs = []
    for key in tts:
        if "_multi" in key:
            continue
        algo, rest = key.split("_", 1)
        name, b = rest.rsplit("_budget", 1)
        jobs.append((name, algo, int(b), 0))
    with mp.get_context("fork").Pool(min(len(jobs),
                                         len(os.sched_getaffinity(0)))) as p:
        res = p.map(_ref_search_job, jobs, chunksize=1)
    out = {}
    for (name, algo, b, _), (obj, genes, el) in zip(jobs, res):
        key = f"{algo}_{name}_budget{b}"
        gpu = tts[key]
        out[key] = {"reference_s": el, "gpu_s": gpu["gpu_s"],
                    "speedup": el / gpu["gpu_s"],
                    "reference_objective_ms": obj,
                    "same_result": obj == gpu["objective_ms"]
                    and genes == gpu["genome_sha1"],
                    "cpu": "hetsched.heuristics (reference, unmodified), "
                           "1 core per run"}
    cores = len(os.sched_getaffinity(0))
    for key, v in tts.items():
        if "_multi148_" not in key:
            continue
        single = out.get(key.replace("_multi148_", "_"))
        if single:
            est = single["reference_s"] * v["chains"] / cores
            out[key] = {"gpu_s": v["gpu_s"],
                        "reference_s_estimate": est,
                        "speedup_estimate": est / v["gpu_s"],
                        "basis": f"{v['chains']} reference runs at the "
                                 f"measured single-run time on {cores} "
                                 "cores in parallel"}
    return out


if __name__ == "__main__":
    main()
