"""The split DP (paper_2308_00127_b200.splitting.milp_split) against the
reference's milp_split (splitting.py:259-402) run live with the SAME
deterministic module solver, so that only the DP is compared: states, tie
rules (first strict improvement by more than 1e-12), incoming-channel
delays, infeasible pinnings, missing links, flags and the assembled
schedule. Host-only (the solver here is a pure-Python stand-in, not the GPU
sweep); skipped when the reference is not importable."""
from __future__ import annotations

import hashlib
import json
import sys

import pytest

from conftest import instance_doc

import paper_2308_00127_b200 as hs


@pytest.fixture(scope="module")
def R():
    from oracle import ref
    if ref.import_reference() is None:
        pytest.skip("reference not importable")
    return (sys.modules["hetsched.core"], sys.modules["hetsched.splitting"])


def _det_solver(RC, reject_mod=None):
    """objective = a hash of (module tasks, pins) scaled to [1, 100), with
    a few exact ties; schedule = every task of the module on its pinned (else
    the first) device, back to back -- deterministic for both sides."""

    def solver(sub, hw, table, L, pins, same_device, timeout):
        tasks = sorted(sub.tasks)
        key = json.dumps([tasks, sorted(pins.items()),
                          sorted(map(list, same_device))]).encode()
        h = int(hashlib.sha1(key).hexdigest()[:8], 16)
        if reject_mod is not None and h % reject_mod == 0:
            return None, None, False
        obj = 1.0 + (h % 97) * 1.0 if h % 5 else 7.0
        dev0 = sorted(hw.devices)[0]
        t0, batches = 0.0, []
        for t in tasks:
            batches.append(RC.ScheduledBatch(
                task=t, device=pins.get(t, dev0), size=L,
                inputs=tuple(range(1, L + 1)), start=t0))
            t0 += 1.0
        return obj, RC.Schedule(batches=tuple(batches), objective=obj,
                                input_count=L), h % 3 != 0

    return solver


def _same(a, b):
    assert a.objective == b.objective
    assert tuple(a.flags) == tuple(b.flags)
    assert a.input_count == b.input_count
    assert [(x.task, x.device, x.size, tuple(x.inputs), x.start)
            for x in a.batches] == \
        [(x.task, x.device, x.size, tuple(x.inputs), x.start)
         for x in b.batches]


def _ref_objs(R, name):
    RC, _ = R
    doc = instance_doc(name)
    return (RC.load_graph(json.dumps(doc["graph"])),
            RC.load_hardware(json.dumps(doc["hardware"])),
            RC.load_latency(json.dumps(doc["latency"])))


@pytest.mark.parametrize("name,c,L", [("ws_stack_10x20", 1, 1),
                                      ("er_stack_10x10", 1, 1),
                                      ("er_stack_10x10", 1, 2),
                                      ("er_stack_4x10_c2", 2, 1),
                                      ("er_stack_4x10_c2", 1, 4),
                                      ("ws30", 1, 1)])
@pytest.mark.parametrize("reject", [None, 4])
def test_split_dp_matches_reference(R, name, c, L, reject):
    RC, RS = R
    rg, rhw, rt = _ref_objs(R, name)
    g, hw, t = hs.load_instance(instance_doc(name))
    rd, d = RS.k_edge_components(rg, c), hs.k_edge_components(g, c)
    solver = _det_solver(RC, reject)
    try:
        want = RS.milp_split(rg, rhw, rt, L, rd, module_solver=solver)
    except RC.ScheduleError as exc:
        with pytest.raises(hs.ScheduleError) as got:
            hs.milp_split(g, hw, t, L, d, module_solver=solver)
        assert str(got.value) == str(exc)
        return
    got = hs.milp_split(g, hw, t, L, d, module_solver=solver, workers=4)
    _same(got, want)


def test_split_dp_same_device_and_pin_cap(R):
    RC, RS = R
    name = "er_stack_4x10_c2"
    rg, rhw, rt = _ref_objs(R, name)
    g, hw, t = hs.load_instance(instance_doc(name))
    rd, d = RS.k_edge_components(rg, 1), hs.k_edge_components(g, 1)
    ids = sorted(g.tasks)
    pairs = [(ids[0], ids[5]), (ids[3], ids[9])]
    solver = _det_solver(RC)
    for max_pins in (1, 2, 4):
        want = RS.milp_split(rg, rhw, rt, 1, rd, module_solver=solver,
                             same_device=pairs, max_pins=max_pins)
        got = hs.milp_split(g, hw, t, 1, d, module_solver=solver,
                            same_device=pairs, max_pins=max_pins)
        _same(got, want)
