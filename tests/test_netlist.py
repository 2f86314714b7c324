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
