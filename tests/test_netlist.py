"""Netlist ingest / DAG levelling of the host mirror vs the reference (no GPU)."""
import ctypes
import json

import numpy as np
import pytest

from oracle import pyoracle
from paper_2010_09410_b200 import netlist as N

has_ref = pytest.mark.skipif(not pyoracle.available("ref"), reason="reference not built")


def ref_levels(text):
    L = pyoracle._lib("ref")
    nl = N.parse_netlist(text)
    lv = np.zeros(len(nl.cells) + 1, np.int32)
    cells = np.zeros(len(nl.cells) + 1, np.int32)
    gmax, depth, nodes = ctypes.c_int(), ctypes.c_int(), ctypes.c_size_t()
    rc = L.ref_netlist_levels(text.encode(), lv.ctypes.data_as(ctypes.c_void_p),
                              cells.ctypes.data_as(ctypes.c_void_p), ctypes.byref(gmax),
                              ctypes.byref(depth), ctypes.byref(nodes))
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    return lv[:nodes.value], gmax.value, depth.value


HALF_ADDER = {
    "name": "half_adder",
    "ports": {"in": [{"name": "A", "bits": [0]}, {"name": "B", "bits": [1]}],
              "out": [{"name": "S", "bits": [5]}, {"name": "C", "bits": [6]}]},
    "cells": [
        {"id": 1, "kind": "NAND", "pins": {"a": 0, "b": 1, "y": 2}},
        {"id": 2, "kind": "NAND", "pins": {"a": 0, "b": 2, "y": 3}},
        {"id": 3, "kind": "NAND", "pins": {"a": 2, "b": 1, "y": 4}},
        {"id": 4, "kind": "NAND", "pins": {"a": 3, "b": 4, "y": 5}},
        {"id": 5, "kind": "NOT", "pins": {"a": 2, "y": 6}},
    ],
}


def test_half_adder_stats():
    nl = N.parse_netlist(json.dumps(HALF_ADDER))
    st = N.netlist_stats(nl)
    assert st["count_by_kind"]["NAND"] == 4 and st["count_by_kind"]["NOT"] == 1
    assert st["depth"] == 3 and st["dff_count"] == 0


def test_plain_half_adder():
    nl = N.parse_netlist(json.dumps(HALF_ADDER))
    for a in (0, 1):
        for b in (0, 1):
            ev = N.PlainEvaluator(nl)
            ev.set_input("A", 0, a)
            ev.set_input("B", 0, b)
            ev.run(1)
            assert ev.output("S", 0) == a ^ b and ev.output("C", 0) == a & b


@pytest.mark.parametrize("bad,msg", [
    ({"kind": "FOO"}, "unknown cell kind"),
    ({"pins": {"a": 0, "y": 2}}, "missing pin 'b'"),
    ({"pins": {"a": 0, "b": 1, "y": 3}}, "multiple drivers"),
    ({"pins": {"a": 0, "b": 99, "y": 2}}, "dangling input net"),
])
def test_validation_errors_match_reference_text(bad, msg):
    j = json.loads(json.dumps(HALF_ADDER))
    j["cells"][0].update(bad)
    with pytest.raises(RuntimeError, match=msg):
        N.parse_netlist(json.dumps(j))


def test_combinational_cycle_rejected():
    j = json.loads(json.dumps(HALF_ADDER))
    j["cells"][0]["pins"]["b"] = 5  # NAND1 <- NAND4 <- NAND2 <- NAND1
    with pytest.raises(RuntimeError, match="combinational cycle"):
        N.parse_netlist(json.dumps(j))


@has_ref
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_levels_gmax_depth_match_reference(seed):
    nl = N.synthetic_netlist(seed=seed, scale=0.05, levels=9, dffs=48, ram=(3, 4))
    text = N.netlist_to_json(nl)
    lv, gmax, depth = ref_levels(text)
    d = N.build_dag(N.parse_netlist(text))
    assert list(lv) == d["level"] and gmax == d["gmax"] and depth == d["depth"]


def test_synthetic_ruby_shape():
    nl = N.synthetic_netlist(seed=7)
    st = N.netlist_stats(nl)
    for k, v in N.RUBY_MIX.items():
        assert st["count_by_kind"][k] == v
    assert st["count_by_kind"]["ROM"] == 1 and st["count_by_kind"]["RAM"] == 1
    assert st["dff_count"] == 256
    # JSON round trip (netlistToJson / parseNetlist)
    again = N.parse_netlist(N.netlist_to_json(nl))
    assert N.netlist_to_json(again) == N.netlist_to_json(nl)


# ---- the engine's launch schedule (vsp_netlist_schedule: host-only C ABI, no device) ----

def _tasks(kind):
    return 2 if kind == "MUX" else 0 if kind in ("NOT", "ROM", "RAM", "CONST0", "CONST1") else 1


def _waves(nodes, lv, sms):
    t = {}
    for i, c in enumerate(nodes):
        t[lv[i]] = t.get(lv[i], 0) + _tasks(c.kind)
    return sum(-(-x // sms) for x in t.values())


def _check_schedule(nl, sms):
    nodes = [c for c in nl.cells if c.kind != "DFF"]
    asap, launch, depth = N.schedule(nl, sms)
    assert len(asap) == len(nodes)
    assert np.array_equal(asap, np.asarray(N.build_dag(nl)["level"]))  # buildDag semantics
    assert np.all(launch >= asap) and depth == int(asap.max()) + 1 and launch.max() < depth
    producer = {b: i for i, c in enumerate(nodes) for b in c.outputs}
    for i, c in enumerate(nodes):
        for b in c.inputs:
            if b in producer:
                assert launch[producer[b]] < launch[i]
        if c.kind in ("ROM", "RAM", "CONST0", "CONST1"):
            assert launch[i] == asap[i]
    return _waves(nodes, asap, sms), _waves(nodes, launch, sms)


@pytest.mark.parametrize("sms", [148, 132, 64])
@pytest.mark.parametrize("seed", range(1, 9))
def test_launch_schedule_properties(seed, sms):
    """Level balancing never evaluates a gate before a producer or after a consumer, never
    moves memory ports or constants, never deepens the cycle and never adds a latency
    wave; on netlists with levels just over one wave it removes waves."""
    rng = np.random.default_rng(seed)
    nl = N.synthetic_netlist(seed=seed, scale=float(rng.uniform(0.05, 0.3)),
                             levels=int(rng.integers(3, 8)), dffs=48, ram=(3, 4))
    w_asap, w_launch = _check_schedule(nl, sms)
    assert w_launch <= w_asap


def test_launch_schedule_removes_waves():
    """Netlists whose ASAP levels sit just above one wave of 148 SMs: the bench's cycle
    netlist (one 149-task level: 34 -> 33 waves) and a small one (7 -> 5)."""
    assert _check_schedule(N.synthetic_netlist(seed=1, levels=32), 148) == (34, 33)
    small = N.synthetic_netlist(seed=3, scale=0.134, levels=4, dffs=48, ram=(3, 4))
    assert _check_schedule(small, 148) == (7, 5)


def test_launch_schedule_rejects_invalid_netlists():
    nl = N.synthetic_netlist(seed=2, scale=0.02, levels=3, dffs=8, rom=False, ram=None)
    nl.cells[-1].inputs = [nl.net_count + 5]  # dangling input
    with pytest.raises(RuntimeError, match="dangling input net"):
        N.schedule(nl, 148)
