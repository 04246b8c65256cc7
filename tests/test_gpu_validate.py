"""K11 (csrc/validate.cu, hs_validate_schedules) against the reference's
validate_schedule (core.py:206-291) on the schedules frozen in
tests/golden/validate.json: reference-produced schedules (decode, greedy,
met, bMET / bGreedy at L = 2, 4) and mutated copies of them that trip every
check. Valid ones must return the same makespan bit for bit; invalid ones
the same exception class with the same message."""
from __future__ import annotations

import json

import pytest

from conftest import fhex, golden

import paper_2308_00127_b200 as hs
from paper_2308_00127_b200.core import (GraphError, Schedule, ScheduledBatch,
                                        ScheduleError, load_graph,
                                        load_hardware, load_latency)

pytestmark = pytest.mark.gpu


def _inst(e):
    return (load_graph(json.dumps(e["graph"])),
            load_hardware(json.dumps(e["hardware"])),
            load_latency(json.dumps(e["latency"])))


def _sched(s):
    return Schedule(
        batches=tuple(ScheduledBatch(task=t, device=d, size=z,
                                     inputs=tuple(ins),
                                     start=float.fromhex(st)
                                     if st not in ("inf", "nan") else
                                     float(st))
                      for t, d, z, ins, st in s["batches"]),
        objective=float.fromhex(s["objective"]), input_count=s["input_count"])


def _check(res, s, label):
    if "ok" in s:
        assert not isinstance(res, Exception), (label, res)
        assert fhex(res) == s["ok"], label
    else:
        assert isinstance(res, Exception), (label, res)
        want = {"ScheduleError": ScheduleError, "GraphError": GraphError}
        assert type(res) is want[s["error"]], (label, res)
        assert str(res) == s["msg"], label


def test_validate_golden_batched():
    """Every schedule of a case in ONE launch."""
    n = 0
    for e in golden("validate"):
        g, hw, t = _inst(e)
        scheds = [_sched(s) for s in e["schedules"]]
        res = hs.validate_schedules(g, hw, t, scheds)
        assert len(res) == len(scheds)
        for r, s in zip(res, e["schedules"]):
            _check(r, s, (e["name"], s["label"]))
            n += 1
    assert n > 2000


def test_validate_golden_single():
    """validate_schedule returns the makespan or raises."""
    for e in golden("validate")[::7]:
        g, hw, t = _inst(e)
        for s in e["schedules"][:12]:
            try:
                res = hs.validate_schedule(g, hw, t, _sched(s))
            except (ScheduleError, GraphError) as exc:
                res = exc
            _check(res, s, (e["name"], s["label"]))


def test_validate_decode_outputs():
    """K3 trace schedules of random genomes validate to their objective."""
    import numpy as np
    from conftest import instance_doc
    for name in ("ws30", "ws200", "tf96"):
        g, hw, t = hs.load_instance(instance_doc(name))
        order = tuple(instance_doc(name)["order"])
        K = len(hw.devices)
        rng = np.random.default_rng(3)
        scheds = []
        for _ in range(20):
            genes = tuple(int(x) for x in rng.integers(K, size=len(order)))
            s = hs.decode(hs.MappingGenome(genes=genes, order=order), g, hw,
                          t, 1)
            if s is not None:
                scheds.append(s)
        res = hs.validate_schedules(g, hw, t, scheds)
        assert [fhex(r) for r in res] == [fhex(s.objective) for s in scheds]
