"""Generate the golden fixtures that pin parity with the reference.

Runs the REFERENCE (`hetsched`, read-only under /root/reference/pkg/src, plus
`hetsched_ingest` for the torchvision graphs) in-process and freezes its
inputs and outputs as JSON next to this script:

* ``instances/<name>.json`` -- graph / hardware / latency in the reference
  wire format (core.py:297-356), the reference's BFS order
  (core.py:82-101), the sorted device list (heuristics.py:132), and cases of
  uint8 genomes (base64, row-major [n x V]) with the reference
  ``fitness`` (heuristics.py:146-148) as float.hex() strings, "inf", or
  "GraphError"; a few genomes also carry the ``decode`` schedule starts.
* ``random_instances.json`` -- conftest.random_instance (tests/conftest.py:
  51-108) mini instances incl. missing links, tight memory, unsupported L,
  missing latency entries, out-of-range genes and non-BFS genome orders.
* ``bounds.json`` -- critical_path_bound / dep_subgraph / pre_subgraph
  (bounds.py:29-72) and lower_bound with subgraph_cap=0 (bounds.py:142-236).
* ``heuristics.json`` -- best_device / met / greedy / SA / (1+1) EA results
  (heuristics.py:151-334) at fixed seeds.

This script is test infrastructure: it is run here (where /root/reference
exists), its outputs are committed, and nothing on the GPU box runs it.
Usage: python tests/golden/make_golden.py
"""
from __future__ import annotations

import base64
import json
import math
import os
import sys
import zlib
from multiprocessing import get_context

sys.dont_write_bytecode = True
REF = "/root/reference/pkg"
sys.path[:0] = [REF + "/src", REF + "/ingest/src", REF + "/tests"]

import numpy as np  # noqa: E402

from hetsched import benchgen  # noqa: E402
from hetsched.bounds import (critical_path_bound, dep_subgraph,  # noqa: E402
                             lower_bound, pre_subgraph)
from hetsched.core import (Device, DnnGraph, GraphError,  # noqa: E402
                           HardwareSystem, LatencyTable, ScheduleError,
                           TaskNode, bfs_topological_order, save_graph,
                           save_hardware, save_latency)
from hetsched.heuristics import (MappingGenome, best_device,  # noqa: E402
                                 decode, fitness, greedy, met,
                                 one_plus_one_ea, simulated_annealing)
from hetsched.splitting import k_edge_components  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "instances")


def fhex(x: float) -> str:
    if math.isinf(x):
        return "inf" if x > 0 else "-inf"
    if math.isnan(x):
        return "nan"
    return x.hex()


def b64(a: np.ndarray) -> str:
    return base64.b64encode(np.ascontiguousarray(a, dtype=np.uint8)
                            .tobytes()).decode()


def inst_doc(name, source, g, hw, table, decomp=None):
    doc = {
        "name": name,
        "source": source,
        "graph": json.loads(save_graph(g)),
        "hardware": json.loads(save_hardware(hw)),
        "latency": json.loads(save_latency(table)),
        "order": list(bfs_topological_order(g)),
        "devices_sorted": sorted(hw.devices),
    }
    if decomp is not None:
        doc["decomposition"] = json.loads(decomp.to_json())
    return doc


# ---------------------------------------------------------------- fitness
_G = {}


def _eval_chunk(args):
    key, L, rows, order = args
    g, hw, table = _G[key]
    out = []
    for row in rows:
        try:
            v = fitness(MappingGenome(genes=tuple(int(x) for x in row),
                                      order=tuple(order)), g, hw, table, L)
            out.append(fhex(v))
        except GraphError:
            out.append("GraphError")
    return out


def eval_many(pool, key, L, genes, order):
    chunks = np.array_split(genes, max(1, min(64, len(genes) // 16 + 1)))
    res = pool.map(_eval_chunk, [(key, L, c, order) for c in chunks if len(c)])
    return [x for r in res for x in r]


def trace_doc(g, hw, table, L, row, order):
    try:
        s = decode(MappingGenome(genes=tuple(int(x) for x in row),
                                 order=tuple(order)), g, hw, table, L)
    except GraphError:
        return {"objective": "GraphError"}
    if s is None:
        return None
    return {"objective": fhex(s.objective),
            "batches": [[b.task, b.device, b.size, list(b.inputs),
                         fhex(b.start)] for b in s.batches]}


def make_cases(pool, key, Ls_counts, seed, edge=True, traces=2):
    g, hw, table = _G[key]
    order = list(bfs_topological_order(g))
    V, K = len(order), len(hw.devices)
    cases = []
    for L, n in Ls_counts:
        rng = np.random.default_rng(seed + 7919 * L)
        genes = rng.integers(K, size=(n, V), dtype=np.uint8)
        if edge:  # all-on-one-device candidates (SURVEY 8(d) edge set)
            genes = np.concatenate(
                [genes, np.repeat(np.arange(K, dtype=np.uint8)[:, None],
                                  V, axis=1)])
        exp = eval_many(pool, key, L, genes, order)
        case = {"L": L, "n": int(genes.shape[0]), "V": V,
                "genes_b64": b64(genes), "expected": exp, "traces": []}
        for r in range(min(traces, len(genes))):
            case["traces"].append({"row": r, **(trace_doc(
                g, hw, table, L, genes[r], order) or {"objective": "inf"})})
        cases.append(case)
    return cases


def big_instances():
    out = {}
    g = benchgen.gen_module("ws", 30, seed=0, k=4, p=0.75)
    t, hw = benchgen.synth_profile(g, benchgen.DEFAULT3, seed=0)
    out["ws30"] = (g, hw, t, None,
                   "gen_module('ws',30,seed=0,k=4,p=0.75); "
                   "synth_profile(DEFAULT3, seed=0)",
                   [(1, 3000), (2, 300), (8, 300)])
    g = benchgen.gen_module("ws", 200, seed=0, k=4, p=0.75)
    t, hw = benchgen.synth_profile(g, benchgen.DEFAULT3, seed=0)
    out["ws200"] = (g, hw, t, None,
                    "gen_module('ws',200,seed=0,k=4,p=0.75); "
                    "synth_profile(DEFAULT3, seed=0)",
                    [(1, 1000), (4, 200), (8, 200)])
    g = benchgen.gen_module("ws", 1000, seed=0, k=4, p=0.75)
    t, hw = benchgen.synth_profile(g, benchgen.DEFAULT3, seed=0)
    out["ws1000"] = (g, hw, t, None,
                     "gen_module('ws',1000,seed=0,k=4,p=0.75); "
                     "synth_profile(DEFAULT3, seed=0)", [(1, 100)])
    g, d, hw, t = benchgen.gen_stacked_instance("ws", 20, 10, 1, "sdep", 0)
    out["ws_stack_10x20"] = (g, hw, t, d,
                             "gen_stacked_instance('ws',20,10,1,'sdep',0)",
                             [(1, 300), (2, 100)])
    g, d, hw, t = benchgen.gen_stacked_instance("ws", 100, 10, 1, "sdep", 0)
    out["ws_stack_10x100"] = (g, hw, t, d,
                              "gen_stacked_instance('ws',100,10,1,'sdep',0)",
                              [(1, 60)])
    g, d, hw, t = benchgen.gen_stacked_instance("er", 10, 10, 1, "sdep", 0)
    out["er_stack_10x10"] = (g, hw, t, d,
                             "gen_stacked_instance('er',10,10,1,'sdep',0)",
                             [(1, 300), (4, 100)])
    g, d, hw, t = benchgen.gen_stacked_instance("er", 10, 4, 2, "sdep", 1,
                                                p=0.5)
    out["er_stack_4x10_c2"] = (g, hw, t, d,
                               "gen_stacked_instance('er',10,4,2,'sdep',1,"
                               "p=0.5)", [(1, 300)])
    # transformer case study (benchgen.py:314-367): K=30, two link classes
    g, hw = benchgen.gen_transformer_stack(96, 6, 4)
    specs = [benchgen.DeviceSpec(id=u, factor=7.10 if u.endswith("cpu")
                                 else 1.0) for u in sorted(hw.devices)]
    t, _ = benchgen.synth_profile(g, specs, seed=0)
    out["tf96"] = (g, hw, t, None,
                   "gen_transformer_stack(96,6,4); synth_profile(specs "
                   "factor 7.10 cpu / 1.0 acc, seed=0); transformer hw",
                   [(1, 300), (8, 60)])
    # torchvision graphs through the reference ingest (trace + fuse)
    try:
        import torchvision
        from hetsched.core import load_graph
        from hetsched_ingest.fusion import fuse
        from hetsched_ingest.tracing import trace_model
        for nm, ctor, shape in (
                ("rn50f", torchvision.models.resnet50, (1, 3, 224, 224)),
                ("iv3f", lambda: torchvision.models.inception_v3(
                    aux_logits=False, init_weights=False), (1, 3, 299, 299))):
            doc = fuse(trace_model(ctor(), shape))
            doc = {"tasks": [{k: v for k, v in tk.items() if k != "op"}
                             for tk in doc["tasks"]],
                   "edges": doc["edges"], "name": doc.get("name")}
            g = load_graph(json.dumps(doc))
            t, hw = benchgen.synth_profile(g, benchgen.DEFAULT3, seed=0)
            out[nm] = (g, hw, t, None,
                       f"hetsched_ingest fuse(trace_model({nm}))+"
                       "synth_profile(DEFAULT3, seed=0)",
                       [(1, 500), (2, 200), (8, 200)])
    except Exception as exc:  # pragma: no cover - generator environment
        print("ingest graphs skipped:", exc)
    return out


# ----------------------------------------------------------- random mini
def mini_entries(pool):
    from conftest import random_instance
    entries = []
    specs = ([(s, 8, 4, 1) for s in range(300)]
             + [(s, 6, 3, 2) for s in range(1000, 1150)]
             + [(s, 6, 3, 4) for s in range(2000, 2060)])
    for seed, mt, md, L in specs:
        g, hw, t = random_instance(seed, max_tasks=mt, max_devices=md, L=L)
        entries.append((f"ri_{seed}_L{L}", g, hw, t, L,
                        f"random_instance({seed}, max_tasks={mt}, "
                        f"max_devices={md}, L={L})"))
    # missing latency entries: GraphError only when reached (core.py:166-170)
    for seed in range(40):
        g, hw, t = random_instance(3000 + seed, max_tasks=6, max_devices=3,
                                   L=1, allow_tight_memory=(seed % 2 == 0))
        rng = np.random.default_rng(seed)
        ent = dict(t.entries)
        keys = sorted(k for k in ent if k[2] == 1)
        for j in rng.choice(len(keys), size=min(2, len(keys)), replace=False):
            del ent[keys[j]]
        entries.append((f"ri_missing_{seed}", g, hw, LatencyTable(ent), 1,
                        f"random_instance({3000 + seed}) minus 2 L=1 "
                        "latency entries"))
    # hand-made edge cases
    g = DnnGraph([], [])
    hw = HardwareSystem([Device("d0", 1.0, (1,))], {})
    entries.append(("empty_graph", g, hw, LatencyTable({}), 1, "no tasks"))
    g = DnnGraph([TaskNode("a", 0, 0, 2.0), TaskNode("b", 0, 0, 2.0),
                  TaskNode("c")], [("a", "b"), ("b", "c")])
    hw = HardwareSystem([Device("d0", 1e9, (1,)), Device("d1", 1e9, (1,))],
                        {("d0", "d1"): 1.0, ("d1", "d0"): 1.0})
    t = LatencyTable({(i, u, 1): {"d0": 2.0, "d1": 5.0}[u]
                      + {"a": 0, "b": 1, "c": 2}[i]
                      for i in "abc" for u in ("d0", "d1")})
    entries.append(("chain3", g, hw, t, 1, "test_heuristics._chain3"))
    # zero durations, zero-byte outputs, no links at all, inf latencies
    g = DnnGraph([TaskNode("x", 1, 1, 0.0), TaskNode("y", 0, 3, 7.0),
                  TaskNode("z", 5, 0, 0.0)], [("x", "y"), ("x", "z"),
                                              ("y", "z")])
    hw = HardwareSystem([Device("p", 100.0, (1, 2)), Device("q", 9.0, (2,))],
                        {})
    t = LatencyTable({(i, u, b): v for (i, u, b), v in {
        ("x", "p", 1): 0.0, ("x", "p", 2): 0.0, ("x", "q", 2): 1.5,
        ("y", "p", 1): float("inf"), ("y", "p", 2): 3.0, ("y", "q", 2): 0.0,
        ("z", "p", 1): 2.5, ("z", "p", 2): 4.0, ("z", "q", 2): 1.0}.items()})
    entries.append(("nolinks_zero", g, hw, t, 1, "hand-made: no links"))
    entries.append(("nolinks_zero_L2", g, hw, t, 2, "hand-made: no links"))

    out = []
    for name, g, hw, t, L, src in entries:
        _G[name] = (g, hw, t)
    for name, g, hw, t, L, src in entries:
        order = list(bfs_topological_order(g))
        V, K = len(order), len(hw.devices)
        rng = np.random.default_rng(zlib.crc32(name.encode()))
        genes = rng.integers(K, size=(24, V), dtype=np.uint8) if V else \
            np.zeros((1, 0), np.uint8)
        if V:
            genes = np.concatenate([genes, np.repeat(
                np.arange(K, dtype=np.uint8)[:, None], V, axis=1)])
        e = {"name": name, "source": src, "L": L,
             **{k: v for k, v in inst_doc(name, src, g, hw, t).items()
                if k not in ("name", "source")}}
        cases = []
        exp = _eval_chunk((name, L, genes, order))
        cases.append({"L": L, "n": int(genes.shape[0]), "V": V,
                      "genes_b64": b64(genes), "expected": exp,
                      "traces": [{"row": r, **(trace_doc(
                          g, hw, t, L, genes[r], order)
                          or {"objective": "inf"})}
                          for r in range(min(3, len(genes)))]})
        if V >= 2:  # out-of-range gene raises GraphError (heuristics.py:133)
            bad = genes[:2].copy()
            bad[0, V // 2] = K
            bad[1, 0] = 255
            cases.append({"L": L, "n": 2, "V": V, "genes_b64": b64(bad),
                          "expected": _eval_chunk((name, L, bad, order)),
                          "traces": []})
            # a non-BFS genome order: Kahn with the largest id first
            alt = _alt_order(g)
            if alt != order:
                ag = genes[:8]
                cases.append({"L": L, "n": int(ag.shape[0]), "V": V,
                              "order": alt, "genes_b64": b64(ag),
                              "expected": _eval_chunk((name, L, ag, alt)),
                              "traces": [{"row": 0, **(trace_doc(
                                  g, hw, t, L, ag[0], alt)
                                  or {"objective": "inf"})}]})
        e["cases"] = cases
        out.append(e)
    return out


def _alt_order(g):
    import heapq
    indeg = {i: len(g.pred[i]) for i in g.tasks}
    heap = [(-ord_key(i), i) for i in g.tasks if indeg[i] == 0]
    heapq.heapify(heap)
    out = []
    while heap:
        _, i = heapq.heappop(heap)
        out.append(i)
        for j in g.succ[i]:
            indeg[j] -= 1
            if indeg[j] == 0:
                heapq.heappush(heap, (-ord_key(j), j))
    return out


def ord_key(s):
    return int.from_bytes(s.encode()[:8].ljust(8, b"\0"), "big")


# ------------------------------------------------------------------ bounds
def bounds_doc(insts):
    out = []
    for name in ("ws_stack_10x20", "er_stack_10x10", "er_stack_4x10_c2",
                 "ws200", "rn50f"):
        if name not in insts:
            continue
        g, hw, t, d = insts[name][:4]
        ids = list(g.tasks)
        rng = np.random.default_rng(5)
        cp = []
        for k in range(40):
            p = [0.05, 0.2, 0.5, 1.0][k % 4]
            mask = rng.random(len(ids)) < p
            sub = [ids[i] for i in range(len(ids)) if mask[i]]
            cp.append({"tasks": sub,
                       "value": fhex(critical_path_bound(g, hw, t, sub))})
        reach = []
        for k in range(30):
            u = ids[int(rng.integers(len(ids)))]
            T = [ids[i] for i in range(len(ids)) if rng.random() < 0.5]
            reach.append({"u": u, "T": T,
                          "dep": sorted(dep_subgraph(g, u, T)),
                          "pre": sorted(pre_subgraph(g, u, T))})
        lbs = []
        if d is None:
            d = k_edge_components(g, 1)
        for L in (1, 2, 4):
            rep = lower_bound(g, hw, t, L, d, subgraph_cap=0)
            lbs.append({"L": L, "lower_bound_ms": fhex(rep.lower_bound_ms),
                        "throughput_upper_bound":
                            fhex(rep.throughput_upper_bound),
                        "terms": json.loads(json.dumps(rep.terms))})
        out.append({"instance": name, "critical_path": cp, "reach": reach,
                    "lower_bound_cap0": lbs,
                    "decomposition": json.loads(d.to_json())})
    return out


# -------------------------------------------------------------- heuristics
def heur_doc():
    from conftest import random_instance
    out = []
    cases = [(f"ri_{s}", random_instance(s, max_tasks=6, L=1,
                                         allow_tight_memory=False), 1)
             for s in range(12)]
    g = benchgen.gen_module("ws", 30, seed=0, k=4, p=0.75)
    t, hw = benchgen.synth_profile(g, benchgen.DEFAULT3, seed=0)
    cases.append(("ws30", (g, hw, t), 1))
    cases.append(("ws30_L4", (g, hw, t), 4))
    for name, (g, hw, t), L in cases:
        e = {"name": name, "L": L, **{k: v for k, v in inst_doc(
            name, "", g, hw, t).items() if k not in ("name", "source")}}
        for fn, label in ((best_device, "best_device"), (met, "met"),
                          (greedy, "greedy")):
            try:
                s = fn(g, hw, t, L)
                e[label] = {"objective": fhex(s.objective),
                            "mapping": {b.task: b.device for b in s.batches}}
            except ScheduleError as exc:
                e[label] = {"error": "ScheduleError", "msg": str(exc)}
        runs = []
        for seed in (0, 1, 2):
            for budget in (0, 50, 300):
                for algo in ("sa", "ea", "ea_unbiased"):
                    try:
                        if algo == "sa":
                            s = simulated_annealing(g, hw, t, L, seed=seed,
                                                    budget=budget)
                        else:
                            s = one_plus_one_ea(g, hw, t, L, seed=seed,
                                                budget=budget,
                                                biased=(algo == "ea"))
                        r = {"objective": fhex(s.objective),
                             "mapping": {b.task: b.device for b in s.batches}}
                    except ScheduleError as exc:
                        r = {"error": "ScheduleError", "msg": str(exc)}
                    runs.append({"algo": algo, "seed": seed,
                                 "budget": budget, **r})
        e["search"] = runs
        out.append(e)
    return out


# ----------------------------------------------------------- batched variants
def batched_doc():
    """bMET / bGreedy schedules (heuristics.py:363-433, non-insertion) whose
    per-task (decomposition, devices) choices form extended genomes."""
    from conftest import random_instance
    from hetsched.heuristics import batched_variant
    out = []
    cases = []
    for s in range(60):
        cases.append((f"ri_{s}_L2", random_instance(
            4000 + s, max_tasks=6, max_devices=3, L=2), 2))
    for s in range(30):
        cases.append((f"ri_{s}_L4", random_instance(
            5000 + s, max_tasks=6, max_devices=3, L=4), 4))
    g = benchgen.gen_module("ws", 30, seed=0, k=4, p=0.75)
    t, hw = benchgen.synth_profile(g, benchgen.DEFAULT3, seed=0)
    cases += [("ws30_L4", (g, hw, t), 4), ("ws30_L8", (g, hw, t), 8),
              ("ws30_L2", (g, hw, t), 2)]
    for name, (g, hw, t), L in cases:
        e = {"name": name, "L": L, **{k: v for k, v in inst_doc(
            name, "", g, hw, t).items() if k not in ("name", "source")}}
        for algo in ("met", "greedy"):
            try:
                s = batched_variant(algo, g, hw, t, L)
                e[algo] = {"objective": fhex(s.objective),
                           "batches": [[b.task, b.device, b.size,
                                        list(b.inputs), fhex(b.start)]
                                       for b in s.batches]}
            except (ScheduleError, GraphError) as exc:
                e[algo] = {"error": type(exc).__name__}
        out.append(e)
    return out


def dump(path, obj):
    with open(path, "w") as f:
        json.dump(obj, f, separators=(",", ":"))
    print("wrote", os.path.relpath(path, HERE),
          f"{os.path.getsize(path) / 1024:.0f} KiB")


def main():
    os.makedirs(OUT, exist_ok=True)
    insts = big_instances()
    for name, (g, hw, t, *_r) in insts.items():
        _G[name] = (g, hw, t)
    ctx = get_context("fork")
    with ctx.Pool(os.cpu_count()) as pool:
        for name, (g, hw, t, d, src, lc) in insts.items():
            if os.path.exists(os.path.join(OUT, name + ".json")) \
                    and "--force" not in sys.argv:
                continue
            doc = inst_doc(name, src, g, hw, t, d)
            doc["cases"] = make_cases(pool, name, lc, seed=len(name))
            dump(os.path.join(OUT, name + ".json"), doc)
        dump(os.path.join(HERE, "random_instances.json"), mini_entries(pool))
    dump(os.path.join(HERE, "bounds.json"), bounds_doc(insts))
    dump(os.path.join(HERE, "heuristics.json"), heur_doc())
    dump(os.path.join(HERE, "batched.json"), batched_doc())


if __name__ == "__main__":
    main()
