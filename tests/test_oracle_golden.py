"""Pins the CPU oracle to the reference: every golden makespan, decode trace,
critical path and reachability set produced by running the reference
(tests/golden/make_golden.py) must be reproduced bit-for-bit by the oracle's
restatements (oracle/hs_oracle.py, oracle/hs_oracle.c). CPU only."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import (INSTANCES, case_genes, fhex, golden, instance_doc,
                      random_docs)
from oracle import hs_oracle as O
from oracle.hs_oracle_c import CTables


def _check_case(inst, case, oracle_lib, slow_rows=64):
    order = case.get("order")
    tb = O.build_tables(inst, case["L"], order)
    genes = case_genes(case)
    exp = case["expected"]
    ms, st = O.fitness_np(tb, genes)
    got = ["GraphError" if s >= O.ST_MISSING else fhex(v)
           for v, s in zip(ms, st)]
    assert got == exp
    cm, cst = CTables(tb).fitness(oracle_lib, genes, threads=4)
    assert ["GraphError" if s >= 4 else fhex(v) for v, s in zip(cm, cst)] == exp
    for r in range(min(slow_rows, len(genes))):
        v, s = O.fitness_one(tb, genes[r])
        assert ("GraphError" if s >= 4 else fhex(v)) == exp[r]
    for tr in case.get("traces", []):
        v, s, starts = O.fitness_one(tb, genes[tr["row"]], trace=True)
        if tr["objective"] in ("inf", "GraphError"):
            assert s != O.OK
            continue
        assert fhex(v) == tr["objective"]
        assert [fhex(x) for x in starts] == [b[4] for b in tr["batches"]]
        assert [b[0] for b in tr["batches"]] == tb.order


@pytest.mark.parametrize("name", INSTANCES)
def test_instances(name, oracle_lib):
    doc = instance_doc(name)
    inst = O.Instance.from_doc(doc)
    assert O.bfs_order(inst) == doc["order"]
    assert sorted(inst.dev_ids) == doc["devices_sorted"]
    for case in doc["cases"]:
        _check_case(inst, case, oracle_lib, slow_rows=8)


def test_random_instances(oracle_lib):
    docs = random_docs()
    assert len(docs) > 500
    kinds = set()
    for doc in docs:
        inst = O.Instance.from_doc(doc)
        assert O.bfs_order(inst) == doc["order"]
        for case in doc["cases"]:
            _check_case(inst, case, oracle_lib)
            kinds.update(case["expected"])
    # the fixture set really exercises every outcome
    assert "inf" in kinds and "GraphError" in kinds


def test_bounds_golden():
    for entry in golden("bounds"):
        inst = O.Instance.from_doc(instance_doc(entry["instance"]))
        for c in entry["critical_path"]:
            assert fhex(O.critical_path(inst, c["tasks"])) == c["value"]
        for r in entry["reach"]:
            assert sorted(O.reach_dep(inst, r["u"], r["T"])) == r["dep"]
            assert sorted(O.reach_pre(inst, r["u"], r["T"])) == r["pre"]


def test_gen_genes_properties():
    a = O.gen_genes(7, 0, 64, 202, 3)
    b = O.gen_genes(7, 32, 32, 202, 3)
    assert a.shape == (64, 202) and a.max() < 3
    assert np.array_equal(a[32:], b)          # counter based: any sub-range
    c = O.gen_genes(8, 0, 64, 202, 3)
    assert not np.array_equal(a, c)
    hist = np.bincount(O.gen_genes(1, 0, 2000, 202, 3).ravel(), minlength=3)
    assert hist.min() > 0.3 * hist.sum() / 3 * 0.9


def test_argmin_first_semantics():
    v = np.array([np.inf, 3.0, 1.0, 1.0, np.inf])
    assert O.argmin_first(v) == (1.0, 2)
    assert O.argmin_first(np.full(4, np.inf)) == (np.inf, 0)
    assert O.argmin_first(np.array([])) == (np.inf, -1)


def test_search_oracle_golden():
    """The CPU SA / EA restatement (oracle/hs_search.py) reproduces the
    reference's recorded runs (objective + mapping)."""
    from oracle import hs_search as S
    checked = 0
    for e in golden("heuristics"):
        inst = O.Instance.from_doc(e)
        tb = O.build_tables(inst, e["L"])
        for run in e["search"]:
            if "error" in run or run["budget"] > 50:
                continue
            if run["algo"] == "sa":
                fit, genes = S.simulated_annealing(inst, e["L"], run["seed"],
                                                   run["budget"])
            else:
                fit, genes = S.one_plus_one_ea(inst, e["L"], run["seed"],
                                               run["budget"],
                                               biased=run["algo"] == "ea")
            assert fhex(fit) == run["objective"]
            assert {t: tb.devs[k] for t, k in zip(tb.order, genes)} == \
                run["mapping"]
            checked += 1
    assert checked > 50


def test_batched_oracle_golden():
    """The extended-genome restatement reproduces the reference's bMET and
    bGreedy schedules (objective and every sub-batch start)."""
    from oracle import hs_batched as B
    checked = 0
    for e in golden("batched"):
        inst = O.Instance.from_doc(e)
        opts = B.options(inst, e["L"])
        for algo in ("met", "greedy"):
            res = e[algo]
            if "error" in res:
                continue
            genes = B.genes_from_schedule(inst, e["L"], opts, res["batches"])
            ms, st, starts = B.eval_one(inst, e["L"], opts, genes, trace=True)
            assert st == 0 and fhex(ms) == res["objective"]
            got = [fhex(x) for row in starts for x in row]
            assert got == [b[4] for b in res["batches"]]
            checked += 1
    assert checked > 150
