"""Round-2 golden fixtures: run the REFERENCE (`hetsched`, read-only under
/root/reference/pkg/src) and freeze what it returns for

* ``decomp.json`` -- ``find_bridges_and_articulation_points`` and
  ``k_edge_components(g, c)`` for c = 1, 2, 3 (splitting.py:36-81,
  178-219) on every golden instance and on random ER / WS / BA modules,
  random DAGs and stacked instances;
* ``validate.json`` -- ``validate_schedule`` (core.py:206-291) on schedules
  the reference produced (decode of random genomes, greedy, met, the batched
  variants at L > 1) and on mutated copies of them, with the reference's
  return value (makespan hex) or exception class and message;
* ``bounds_cap40.json`` -- ``lower_bound`` with its DEFAULT subgraph cap of
  40 (the MILP terms, bounds.py:91-131) on the small stacked instances;
* ``search_big.json`` -- ``simulated_annealing`` / ``one_plus_one_ea`` at the
  north star's scale (budget 2000, seeds 0-2) on the WS 10x20 stack, WS200
  and the 96-layer transformer (heuristics.py:259-334).

Test infrastructure, run here (where /root/reference exists); its outputs
are committed and nothing on the GPU box runs it.
Usage: python tests/golden/make_golden_r2.py [decomp|validate|bounds|search]
"""
from __future__ import annotations

import json
import os
import sys
from multiprocessing import get_context

sys.dont_write_bytecode = True
REF = "/root/reference/pkg"
sys.path[:0] = [REF + "/src", REF + "/tests"]
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402

from hetsched import benchgen  # noqa: E402
from hetsched.bounds import lower_bound  # noqa: E402
from hetsched.core import (DnnGraph, GraphError, ScheduledBatch,  # noqa: E402
                           Schedule, ScheduleError, TaskNode, load_graph,
                           load_hardware, load_latency, save_graph,
                           validate_schedule)
from hetsched.heuristics import (MappingGenome, batched_variant,  # noqa: E402
                                 decode, greedy, met, one_plus_one_ea,
                                 simulated_annealing)
from hetsched.splitting import (find_bridges_and_articulation_points,  # noqa
                                k_edge_components)

INSTANCES = ["ws30", "ws200", "ws1000", "ws_stack_10x20", "ws_stack_10x100",
             "er_stack_10x10", "er_stack_4x10_c2", "tf96", "rn50f", "iv3f"]


def fhex(x: float) -> str:
    if x != x:
        return "nan"
    if x in (float("inf"), float("-inf")):
        return "inf" if x > 0 else "-inf"
    return float(x).hex()


def load(name):
    with open(os.path.join(HERE, "instances", name + ".json")) as f:
        doc = json.load(f)
    return (load_graph(json.dumps(doc["graph"])),
            load_hardware(json.dumps(doc["hardware"])),
            load_latency(json.dumps(doc["latency"])))


def dump(name, obj):
    path = os.path.join(HERE, name)
    with open(path, "w") as f:
        json.dump(obj, f, separators=(",", ":"))
    print("wrote", name, f"{os.path.getsize(path) / 1024:.0f} KiB")


# ------------------------------------------------------------ decompositions
def _decomp_entry(g, label):
    bridges, artic, conn = find_bridges_and_articulation_points(g)
    e = {"name": label, "bridges": [list(x) for x in bridges],
         "articulation": sorted(artic), "connected": conn, "k_edge": {}}
    for c in (1, 2, 3):
        d = k_edge_components(g, c)
        e["k_edge"][str(c)] = {
            "modules": [sorted(m) for m in d.modules],
            "cuts": [[a, b, [list(x) for x in es]]
                     for (a, b), es in d.cut_edges.items()],
            "is_chain": d.is_chain}
    return e


def _random_dag(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 40))
    p = float(rng.uniform(0.03, 0.4))
    ids = [f"n{int(x)}" for x in rng.permutation(n * 3)[:n]]
    tasks = [TaskNode(id=i, wm=0.0, im=0.0, om=1.0) for i in ids]
    edges = [(ids[a], ids[b]) for a in range(n) for b in range(a + 1, n)
             if rng.random() < p]
    return DnnGraph(tasks, edges, name=f"dag{seed}")


def decomp_doc():
    out = []
    for name in INSTANCES:
        g, _hw, _t = load(name)
        out.append(_decomp_entry(g, name))
    extra = []
    for s in range(12):
        for model, kw in (("er", {"p": 0.15}), ("ws", {"k": 4, "p": 0.3}),
                          ("ba", {"m": 2})):
            n = 8 + 3 * s
            extra.append(benchgen.gen_module(model, n, seed=s, **kw))
    for s in range(60):
        extra.append(_random_dag(s))
    for s in range(6):
        for model in ("er", "ws"):
            try:
                g, _d, _hw, _t = benchgen.gen_stacked_instance(
                    model, 8, 4, 1 + s % 2, "sdep" if s % 3 else "dep", s,
                    **({"p": 0.5} if model == "er" else {}))
            except GraphError:
                continue
            extra.append(g)
    for k, g in enumerate(extra):
        e = _decomp_entry(g, f"extra{k}")
        e["graph"] = json.loads(save_graph(g))
        out.append(e)
    return out


# ------------------------------------------------------------- validation
def _sched_doc(s):
    return {"objective": fhex(s.objective), "input_count": s.input_count,
            "batches": [[b.task, b.device, b.size, list(b.inputs),
                         fhex(b.start)] for b in s.batches]}


def _outcome(g, hw, t, s):
    try:
        return {"ok": fhex(validate_schedule(g, hw, t, s))}
    except (ScheduleError, GraphError) as exc:
        return {"error": type(exc).__name__, "msg": str(exc)}


def _mutations(s, g, hw, rng):
    """Mutated copies of a valid schedule covering every validator check."""
    bs = list(s.batches)
    devs = sorted(hw.devices)
    out = []
    if not bs:
        return out

    def put(label, batches, objective=s.objective, L=s.input_count):
        out.append((label, Schedule(batches=tuple(batches),
                                    objective=objective, input_count=L)))

    def rep(k, **kw):
        b = bs[k]
        d = dict(task=b.task, device=b.device, size=b.size,
                 inputs=b.inputs, start=b.start)
        d.update(kw)
        nb = list(bs)
        nb[k] = ScheduledBatch(**d)
        return nb

    k = int(rng.integers(len(bs)))
    put("unknown_task", rep(k, task="zz_nope"))
    put("unknown_device", rep(k, device="zz_dev"))
    put("size_mismatch", rep(k, size=bs[k].size + 1))
    put("negative_start", rep(k, start=-1.0))
    put("input_range", rep(k, inputs=tuple(x + s.input_count
                                           for x in bs[k].inputs)))
    put("dropped_batch", bs[:k] + bs[k + 1:])
    put("duplicate_batch", bs + [bs[k]])
    put("objective_off", bs, objective=s.objective * 1.001 + 1.0)
    put("objective_tiny", bs, objective=s.objective + 1e-12)
    for j in range(3):
        k = int(rng.integers(len(bs)))
        put(f"moved_device{j}", rep(k, device=devs[int(rng.integers(
            len(devs)))]))
        k = int(rng.integers(len(bs)))
        put(f"start_earlier{j}", rep(k, start=bs[k].start * 0.5))
        k = int(rng.integers(len(bs)))
        put(f"start_later{j}", rep(k, start=bs[k].start + 0.25))
    # everything shifted: no overlap change, objective mismatch only
    shifted = [ScheduledBatch(task=b.task, device=b.device, size=b.size,
                              inputs=b.inputs, start=b.start + 2.0)
               for b in bs]
    put("shifted", shifted)
    put("shifted_obj", shifted, objective=s.objective + 2.0)
    return out


def validate_doc():
    random_instance = _ref_conftest().random_instance
    out = []
    cases = []
    for s in range(30):
        cases.append((f"ri_{s}", random_instance(s, max_tasks=6, L=1), 1))
    for s in range(20):
        cases.append((f"ri_{s}_L2", random_instance(
            4000 + s, max_tasks=6, max_devices=3, L=2), 2))
    for s in range(10):
        cases.append((f"ri_{s}_L4", random_instance(
            5000 + s, max_tasks=6, max_devices=3, L=4), 4))
    for name in ("ws30", "ws_stack_10x20", "er_stack_4x10_c2", "rn50f"):
        cases.append((name, load(name), 1))
    cases.append(("ws30_L4", load("ws30"), 4))
    for name, (g, hw, t), L in cases:
        rng = np.random.default_rng(len(out))
        doc = {"name": name, "L": L,
               "graph": json.loads(save_graph(g)),
               "hardware": json.loads(_save_hw(hw)),
               "latency": json.loads(_save_lat(t)), "schedules": []}
        devs = sorted(hw.devices)
        base = []
        if L == 1:
            from hetsched.core import bfs_topological_order
            order = tuple(bfs_topological_order(g))
            for _ in range(6):
                genes = tuple(int(x) for x in rng.integers(len(devs),
                                                            size=len(order)))
                try:
                    s = decode(MappingGenome(genes=genes, order=order), g,
                               hw, t, L)
                except GraphError:
                    s = None
                if s is not None:
                    base.append(("decode", s))
            for fn, lab in ((greedy, "greedy"), (met, "met")):
                try:
                    base.append((lab, fn(g, hw, t, L)))
                except (ScheduleError, GraphError):
                    pass
        else:
            for algo in ("met", "greedy"):
                try:
                    base.append((f"b{algo}", batched_variant(algo, g, hw, t,
                                                             L)))
                except (ScheduleError, GraphError):
                    pass
        for lab, s in base[:5 if len(g.tasks) <= 40 else 1]:
            doc["schedules"].append({"label": lab, **_sched_doc(s),
                                     **_outcome(g, hw, t, s)})
            for mlab, ms in _mutations(s, g, hw, rng):
                doc["schedules"].append({"label": f"{lab}/{mlab}",
                                         **_sched_doc(ms),
                                         **_outcome(g, hw, t, ms)})
        out.append(doc)
    return out


def _ref_conftest():
    """The reference's tests/conftest.py (random_instance), loaded by path
    so that this repository's own tests/conftest.py does not shadow it."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "ref_conftest", REF + "/tests/conftest.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _save_hw(hw):
    from hetsched.core import save_hardware
    return save_hardware(hw)


def _save_lat(t):
    from hetsched.core import save_latency
    return save_latency(t)


# ------------------------------------------------------------ lower bounds
def _lb_job(args):
    from hetsched.core import save_hardware, save_latency
    name, L, workers = args
    g, d0, hw, t = benchgen.gen_stacked_instance(*name)
    d = k_edge_components(g, 1)
    rep = lower_bound(g, hw, t, L, d, workers=workers)
    return {"instance": "gen_stacked_instance%r" % (name,), "L": L,
            "subgraph_cap": 40, "graph": json.loads(save_graph(g)),
            "hardware": json.loads(save_hardware(hw)),
            "latency": json.loads(save_latency(t)),
            "lower_bound_ms": fhex(rep.lower_bound_ms),
            "throughput_upper_bound": fhex(rep.throughput_upper_bound),
            "terms": json.loads(json.dumps(rep.terms))}


def bounds_doc():
    # small stacks: the MILP sub-solves of a 24-task instance already take
    # ~80 s single-threaded (HiGHS), the 10-module stacks hours
    jobs = [(("er", 6, 3, 1, "sdep", 0), 1, 8)]
    with get_context("fork").Pool(len(jobs)) as p:
        return p.map(_lb_job, jobs, chunksize=1)


# ------------------------------------------------------- search trajectories
def _search_job(args):
    name, algo, seed, budget = args
    g, hw, t = load(name)
    if algo == "sa":
        s = simulated_annealing(g, hw, t, 1, seed=seed, budget=budget)
    else:
        s = one_plus_one_ea(g, hw, t, 1, seed=seed, budget=budget)
    return {"instance": name, "algo": algo, "seed": seed, "budget": budget,
            "objective": fhex(s.objective),
            "mapping": {b.task: b.device for b in s.batches}}


def search_doc():
    jobs = [(n, a, s, 2000) for n in ("ws_stack_10x20", "ws200", "tf96")
            for a in ("sa", "ea") for s in (0, 1, 2)]
    with get_context("fork").Pool(os.cpu_count()) as p:
        return p.map(_search_job, jobs, chunksize=1)


# ------------------------------------------------------- throughput mode
def throughput_doc():
    """test_acceptance.py:298-321: 20 random L=2 instances, the brute-force
    optimum under the throughput objective (oracle.py:96-) and the batched
    heuristics' schedules (which must never beat it)."""
    from hetsched.core import save_hardware, save_latency
    from hetsched.oracle import brute_force
    random_instance = _ref_conftest().random_instance
    out = []
    L = 2
    for seed in range(2000, 2020):
        g, hw, t = random_instance(seed, max_tasks=5, max_devices=2, L=L,
                                   allow_missing_links=False,
                                   allow_tight_memory=False)
        opt = brute_force(g, hw, t, L, objective="throughput")
        e = {"seed": seed, "L": L, "graph": json.loads(save_graph(g)),
             "hardware": json.loads(save_hardware(hw)),
             "latency": json.loads(save_latency(t)),
             "oracle_objective": fhex(opt.objective), "batched": {}}
        for algo in ("met", "greedy", "heft"):
            try:
                s = batched_variant(algo, g, hw, t, L)
            except ScheduleError:
                continue
            e["batched"][algo] = {"objective": fhex(s.objective),
                                  **_sched_doc(s)}
        out.append(e)
    return out


def main():
    # networkx's k-edge auxiliary graph recurses once per tree level
    # (RecursionError at the default limit on WS1000 with k >= 3)
    sys.setrecursionlimit(200000)
    what = sys.argv[1:] or ["decomp", "validate", "search", "throughput",
                            "bounds"]
    if "decomp" in what:
        dump("decomp.json", decomp_doc())
    if "validate" in what:
        dump("validate.json", validate_doc())
    if "search" in what:
        dump("search_big.json", search_doc())
    if "throughput" in what:
        dump("throughput.json", throughput_doc())
    if "bounds" in what:
        dump("bounds_cap40.json", bounds_doc())


if __name__ == "__main__":
    main()
