"""Netlist layer: JSON ingest/validation, the Evaluator facade over the native
level-batched runner, a plaintext backend, and a synthetic Ruby-shaped generator.

Mirrors hvp::netlist (netlist.hpp / netlist.cpp / engine.hpp):
* parse_netlist / validate_netlist / netlist_to_json follow netlist.cpp:106-346 with the
  same error texts (raised as RuntimeError, the reference's std::runtime_error);
* Evaluator keeps the reference Evaluator surface (engine.hpp:107-405): set_input,
  set_input_bool, output, dff_names, dff_state, set_dff_state_raw, set_dff_by_name,
  set_rom, set_ram, rom/ram, run(cycles, RunOptions) with CycleStats;
* PlainEvaluator is the PlainBackend (engine.hpp:48-71, engine.cpp:65-111).
The per-cycle evaluation itself runs in libvsp_b200.so (vsp_netlist_*).
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass, field

import numpy as np

from . import _check, _ptr, lib

# hvp::netlist::CellKind order (netlist.hpp:12-28)
CELL_KINDS = ["AND", "ANDNOT", "MUX", "NAND", "NOR", "NOT", "OR", "ORNOT", "XNOR", "XOR",
              "DFF", "ROM", "RAM", "CONST0", "CONST1"]
KIND_ID = {k: i for i, k in enumerate(CELL_KINDS)}
GATES = set(CELL_KINDS[:10])


def _fail(msg: str):
    raise RuntimeError("netlist: " + msg)


@dataclass
class Cell:
    id: int
    kind: str
    inputs: list
    outputs: list
    name: str = ""


@dataclass
class Port:
    name: str
    bits: list


@dataclass
class Netlist:
    name: str = ""
    inputs: list = field(default_factory=list)
    outputs: list = field(default_factory=list)
    cells: list = field(default_factory=list)
    net_count: int = 0


def parse_netlist(text: str) -> Netlist:
    """parseNetlist (netlist.cpp:106-199)."""
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        _fail(f"JSON syntax error: {e}")
    nl = Netlist(name=j.get("name", ""))
    ports = j.get("ports", {})
    for p in ports.get("in", []):
        nl.inputs.append(Port(p["name"], [int(x) for x in p["bits"]]))
    for p in ports.get("out", []):
        nl.outputs.append(Port(p["name"], [int(x) for x in p["bits"]]))
    for c in j.get("cells", []):
        cid = int(c["id"])
        kind = c["kind"]
        if kind not in KIND_ID:
            _fail(f"unknown cell kind '{kind}'")
        pins = c["pins"]

        def one(pin):
            if pin not in pins:
                _fail(f"cell {cid} ({kind}) is missing pin '{pin}'")
            return int(pins[pin])

        if kind == "NOT":
            ins, outs = [one("a")], [one("y")]
        elif kind == "MUX":
            ins, outs = [one("s"), one("a"), one("b")], [one("y")]
        elif kind == "DFF":
            ins, outs = [one("d")], [one("q")]
        elif kind in ("CONST0", "CONST1"):
            ins, outs = [], [one("y")]
        elif kind == "ROM":
            ins, outs = [int(x) for x in pins["addr"]], [int(x) for x in pins["rdata"]]
        elif kind == "RAM":
            ins = [int(x) for x in pins["addr"]] + [int(x) for x in pins["wdata"]] + [one("wflag")]
            outs = [int(x) for x in pins["rdata"]]
        else:
            ins, outs = [one("a"), one("b")], [one("y")]
        nl.cells.append(Cell(cid, kind, ins, outs, c.get("name", "")))
    nets = [b for p in nl.inputs + nl.outputs for b in p.bits]
    nets += [b for c in nl.cells for b in c.inputs + c.outputs]
    nl.net_count = (max(nets) + 1) if nets else 0
    validate_netlist(nl)
    return nl


def netlist_to_json(nl: Netlist) -> str:
    """netlistToJson (netlist.cpp:201-263)."""
    cells = []
    for c in nl.cells:
        k = c.kind
        if k == "NOT":
            pins = {"a": c.inputs[0], "y": c.outputs[0]}
        elif k == "MUX":
            pins = {"s": c.inputs[0], "a": c.inputs[1], "b": c.inputs[2], "y": c.outputs[0]}
        elif k == "DFF":
            pins = {"d": c.inputs[0], "q": c.outputs[0]}
        elif k in ("CONST0", "CONST1"):
            pins = {"y": c.outputs[0]}
        elif k == "ROM":
            pins = {"addr": c.inputs, "rdata": c.outputs}
        elif k == "RAM":
            w = len(c.outputs)
            v = len(c.inputs) - w - 1
            pins = {"addr": c.inputs[:v], "wdata": c.inputs[v:v + w], "wflag": c.inputs[v + w],
                    "rdata": c.outputs}
        else:
            pins = {"a": c.inputs[0], "b": c.inputs[1], "y": c.outputs[0]}
        jc = {"id": c.id, "kind": k, "pins": pins}
        if c.name:
            jc["name"] = c.name
        cells.append(jc)
    return json.dumps({"name": nl.name,
                       "ports": {"in": [{"name": p.name, "width": len(p.bits), "bits": p.bits}
                                        for p in nl.inputs],
                                 "out": [{"name": p.name, "width": len(p.bits), "bits": p.bits}
                                         for p in nl.outputs]},
                       "cells": cells})


def validate_netlist(nl: Netlist):
    """validateNetlist (netlist.cpp:265-346)."""
    ids = set()
    for c in nl.cells:
        if c.id in ids:
            _fail(f"duplicate cell id {c.id}")
        ids.add(c.id)
    driver = [-1] * nl.net_count
    for p in nl.inputs:
        for b in p.bits:
            if b < 0 or b >= nl.net_count:
                _fail(f"input port '{p.name}' references bad net {b}")
            if driver[b] != -1:
                _fail(f"multiple drivers on net {b}")
            driver[b] = -2
    for i, c in enumerate(nl.cells):
        arity = {"NOT": 1, "DFF": 1, "MUX": 3, "CONST0": 0, "CONST1": 0}.get(c.kind, 2)
        if c.kind in ("ROM", "RAM"):
            arity = len(c.inputs)
        if len(c.inputs) != arity:
            _fail(f"cell {c.id} ({c.kind}) has wrong input count")
        for b in c.outputs:
            if b < 0 or b >= nl.net_count:
                _fail(f"cell {c.id} drives bad net {b}")
            if driver[b] != -1:
                _fail(f"multiple drivers on net {b} (cell {c.id})")
            driver[b] = i
    for c in nl.cells:
        for b in c.inputs:
            if b < 0 or b >= nl.net_count or driver[b] == -1:
                _fail(f"dangling input net {b} on cell {c.id}")
    for p in nl.outputs:
        for b in p.bits:
            if b < 0 or b >= nl.net_count or driver[b] == -1:
                _fail(f"output port '{p.name}' reads undriven net {b}")
    rom = ram = 0
    for c in nl.cells:
        if c.kind == "ROM":
            rom += 1
            if len(c.outputs) != 32:
                _fail("ROM port must have 32 rdata bits")
            if not c.inputs:
                _fail("ROM port needs address bits")
        if c.kind == "RAM":
            ram += 1
            w = len(c.outputs)
            if w == 0 or len(c.inputs) < w + 2:
                _fail("RAM port pin widths are inconsistent")
    if rom > 1 or ram > 1:
        _fail("at most one ROM port and one RAM port are supported")
    build_dag(nl)


def build_dag(nl: Netlist) -> dict:
    """buildDag (netlist.cpp:348-432): levels, heights, gMax, depth (host-side copy used
    for validation and statistics; the runner rebuilds it natively)."""
    node_of = {}
    dag_cells, dffs = [], []
    for i, c in enumerate(nl.cells):
        if c.kind == "DFF":
            dffs.append(i)
            continue
        node_of[i] = len(dag_cells)
        dag_cells.append(i)
    producer = [-1] * nl.net_count
    for i in node_of:
        for net in nl.cells[i].outputs:
            producer[net] = node_of[i]
    n = len(dag_cells)
    consumers = [[] for _ in range(n)]
    indeg = [0] * n
    for node, ci in enumerate(dag_cells):
        for net in nl.cells[ci].inputs:
            p = producer[net]
            if p >= 0:
                consumers[p].append(node)
                indeg[node] += 1
    level = [0] * n
    deg = list(indeg)
    q = [i for i in range(n) if deg[i] == 0]
    topo = []
    h = 0
    while h < len(q):
        node = q[h]
        h += 1
        topo.append(node)
        for c2 in consumers[node]:
            level[c2] = max(level[c2], level[node] + 1)
            deg[c2] -= 1
            if deg[c2] == 0:
                q.append(c2)
    if len(topo) != n:
        for i in range(n):
            if deg[i] > 0:
                _fail(f"combinational cycle through cell {nl.cells[dag_cells[i]].id}")
    widths = {}
    for lv in level:
        widths[lv] = widths.get(lv, 0) + 1
    return {"dag_cells": dag_cells, "dff_cells": dffs, "level": level,
            "gmax": max(widths.values()) if widths else 0,
            "depth": (max(level) + 1) if level else 0}


def netlist_stats(nl: Netlist) -> dict:
    """netlistStats (netlist.cpp:434-450)."""
    counts = {k: 0 for k in CELL_KINDS}
    for c in nl.cells:
        counts[c.kind] += 1
    d = build_dag(nl) if nl.cells else {"gmax": 0, "depth": 0}
    return {"count_by_kind": counts, "dff_count": counts["DFF"],
            "comb_cell_count": len(nl.cells) - counts["DFF"], "gmax": d["gmax"],
            "depth": d["depth"]}


@dataclass
class CycleStats:
    """CycleStats (engine.hpp:22-35)."""
    evaluated_total: int
    gmax: int
    depth: int
    seconds: float


@dataclass
class RunOptions:
    """RunOptions (engine.hpp:37-43).  workers/shuffle_seed are accepted for API parity;
    the level-batched runner is deterministic by construction."""
    workers: int = 1
    shuffle_seed: int = 0
    stats: list | None = None


def _bind():
    L = lib()
    vp, i32, u32, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint64
    if getattr(L, "_nl_bound", False):
        return L
    L.vsp_netlist_create.restype = vp
    L.vsp_netlist_create.argtypes = [vp, i32, i32, vp, vp, vp, vp, vp, vp, vp, i32]
    L.vsp_netlist_destroy.argtypes = [vp]
    L.vsp_netlist_info.argtypes = [vp, vp, vp]
    L.vsp_netlist_launch_levels.argtypes = [vp, vp]
    L.vsp_netlist_schedule.argtypes = [i32, i32, vp, vp, vp, vp, vp, vp, vp, i32, i32, vp, vp, vp]
    L.vsp_netlist_set_input.argtypes = [vp, i32, vp]
    L.vsp_netlist_get_net.argtypes = [vp, i32, vp]
    L.vsp_netlist_dff.argtypes = [vp, vp, vp]
    L.vsp_netlist_set_rom.argtypes = [vp, u32, vp, u32]
    L.vsp_netlist_ram.argtypes = [vp, u32, u32, vp, vp]
    L.vsp_netlist_run.argtypes = [vp, u64, vp]
    L.vsp_netlist_cycle.argtypes = [vp]
    L.vsp_netlist_cycle.restype = u64
    L.vsp_netlist_set_cycle.argtypes = [vp, u64]
    L.vsp_netlist_set_name.argtypes = [vp, ctypes.c_char_p]
    L.vsp_netlist_ram_geometry.argtypes = [vp, ctypes.POINTER(u32), ctypes.POINTER(u32)]
    L.vsp_netlist_snapshot_save.argtypes = [vp, ctypes.c_char_p, vp, ctypes.c_size_t,
                                            ctypes.POINTER(ctypes.c_size_t)]
    L.vsp_netlist_snapshot_load.argtypes = [vp, ctypes.c_char_p, vp, ctypes.c_size_t]
    L.vsp_snapshot_peek.argtypes = [vp, ctypes.c_size_t, vp, vp, vp, ctypes.c_size_t]
    L._nl_bound = True
    return L


def _flat(nl: Netlist):
    """The flat C-ABI arrays of a netlist (vsp_netlist_create / vsp_netlist_schedule)."""
    kinds = np.array([KIND_ID[c.kind] for c in nl.cells], np.int32)
    ids = np.array([c.id for c in nl.cells], np.int32)
    in_off = np.zeros(len(nl.cells) + 1, np.int32)
    out_off = np.zeros(len(nl.cells) + 1, np.int32)
    for i, c in enumerate(nl.cells):
        in_off[i + 1] = in_off[i] + len(c.inputs)
        out_off[i + 1] = out_off[i] + len(c.outputs)
    in_nets = np.array([x for c in nl.cells for x in c.inputs] or [0], np.int32)
    out_nets = np.array([x for c in nl.cells for x in c.outputs] or [0], np.int32)
    inp = [b for p in nl.inputs for b in p.bits]
    return kinds, ids, in_off, in_nets, out_off, out_nets, inp


def schedule(nl: Netlist, sms: int = 148):
    """The engine's launch schedule without a device (vsp_netlist_schedule): per DAG node
    (non-DFF cells, in cell order) the ASAP level and the launch level on an `sms`-SM GPU,
    and the depth."""
    L = _bind()
    kinds, ids, in_off, in_nets, out_off, out_nets, inp = _flat(nl)
    nodes = sum(1 for c in nl.cells if c.kind != "DFF")
    asap = np.zeros(max(nodes, 1), np.int32)
    launch = np.zeros(max(nodes, 1), np.int32)
    depth = np.zeros(1, np.int32)
    inp_arr = np.array(inp or [0], np.int32)
    _check(L.vsp_netlist_schedule(nl.net_count, len(nl.cells), _ptr(kinds), _ptr(ids),
                                  _ptr(in_off), _ptr(in_nets), _ptr(out_off), _ptr(out_nets),
                                  _ptr(inp_arr), len(inp), sms, _ptr(asap), _ptr(launch),
                                  _ptr(depth)))
    return asap[:nodes], launch[:nodes], int(depth[0])


class Evaluator:
    """hvp::netlist::Evaluator<TfheBackend> on the GPU engine."""

    def __init__(self, nl: Netlist, engine):
        self.nl = nl
        self.engine = engine
        self.n = engine.params.n
        L = _bind()
        kinds, ids, in_off, in_nets, out_off, out_nets, inp = _flat(nl)
        self._input_index = {b: i for i, b in enumerate(inp)}
        inp_arr = np.array(inp or [0], np.int32)
        h = L.vsp_netlist_create(engine.h, nl.net_count, len(nl.cells), _ptr(kinds), _ptr(ids),
                                 _ptr(in_off), _ptr(in_nets), _ptr(out_off), _ptr(out_nets),
                                 _ptr(inp_arr), len(inp))
        if not h:
            from . import _raise
            _raise(3, L.vsp_last_error())
        self.h = ctypes.c_void_p(h)
        _check(L.vsp_netlist_set_name(self.h, nl.name.encode()))
        info = np.zeros(6, np.int32)
        _check(L.vsp_netlist_info(self.h, _ptr(info), None))
        self.dag_nodes, self.n_dffs, self.gmax, self.depth, self.rom_cell, self.ram_cell = \
            (int(x) for x in info)
        self._dff_cells = [i for i, c in enumerate(nl.cells) if c.kind == "DFF"]
        self._cell_by_name = {c.name: i for i, c in enumerate(nl.cells) if c.name}
        self._ram_geom = None

    def close(self):
        if getattr(self, "h", None):
            lib().vsp_netlist_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def levels(self) -> np.ndarray:
        lv = np.zeros(max(self.dag_nodes, 1), np.int32)
        info = np.zeros(6, np.int32)
        _check(lib().vsp_netlist_info(self.h, _ptr(info), _ptr(lv)))
        return lv[:self.dag_nodes]

    def launch_levels(self) -> np.ndarray:
        """The level each DAG node is evaluated in (vsp_netlist_launch_levels): ASAP, with
        slack gates moved out of levels wider than one latency wave."""
        lv = np.zeros(max(self.dag_nodes, 1), np.int32)
        _check(lib().vsp_netlist_launch_levels(self.h, _ptr(lv)))
        return lv[:self.dag_nodes]

    @staticmethod
    def _port_bit(ports, name, idx):
        for p in ports:
            if p.name == name:
                if idx >= len(p.bits):
                    raise RuntimeError(f"port '{name}' bit out of range")
                return p.bits[idx]
        raise RuntimeError(f"no port named '{name}'")

    @property
    def cycle(self) -> int:
        return int(lib().vsp_netlist_cycle(self.h))

    def set_cycle(self, c: int):
        _check(lib().vsp_netlist_set_cycle(self.h, c))

    def set_input(self, port: str, idx: int, ct: np.ndarray):
        net = self._port_bit(self.nl.inputs, port, idx)
        ct = np.ascontiguousarray(ct, np.uint32)
        if ct.size != self.n + 1:
            raise ValueError(f"setInput: a TLWE has {self.n + 1} words, got {ct.size}")
        _check(lib().vsp_netlist_set_input(self.h, self._input_index[net], _ptr(ct)))

    def set_input_bool(self, port: str, idx: int, v: bool):
        t = np.zeros(self.n + 1, np.uint32)
        t[-1] = (1 << 29) if v else (2**32 - (1 << 29))
        self.set_input(port, idx, t)

    def output(self, port: str, idx: int) -> np.ndarray:
        net = self._port_bit(self.nl.outputs, port, idx)
        return self.net(net)

    def net(self, net: int) -> np.ndarray:
        out = np.zeros(self.n + 1, np.uint32)
        _check(lib().vsp_netlist_get_net(self.h, net, _ptr(out)))
        return out

    def dff_names(self) -> list:
        return [self.nl.cells[i].name for i in self._dff_cells]

    def dff_state(self) -> np.ndarray:
        out = np.zeros((self.n_dffs, self.n + 1), np.uint32)
        _check(lib().vsp_netlist_dff(self.h, _ptr(out), None))
        return out

    def set_dff_state_raw(self, state: np.ndarray):
        state = np.ascontiguousarray(state, np.uint32)
        if state.shape != (self.n_dffs, self.n + 1):
            raise RuntimeError("DFF state size mismatch")
        _check(lib().vsp_netlist_dff(self.h, None, _ptr(state)))

    def set_dff_by_name(self, name: str, ct: np.ndarray):
        i = self._cell_by_name.get(name)
        if i is None or self.nl.cells[i].kind != "DFF":
            raise RuntimeError(f"no DFF named '{name}'")
        st = self.dff_state()
        st[self._dff_cells.index(i)] = ct
        self.set_dff_state_raw(st)

    def set_rom(self, luts: np.ndarray, depth_bytes: int):
        luts = np.ascontiguousarray(luts, np.uint32)
        if luts.ndim != 2 or luts.shape[1] != 2 * self.engine.params.N1:
            raise ValueError("setRom: LUTs must be (nluts, 2*N1) TRLWEs")
        _check(lib().vsp_netlist_set_rom(self.h, depth_bytes, _ptr(luts), luts.shape[0]))

    def set_ram(self, cells: np.ndarray, v: int, w: int):
        cells = np.ascontiguousarray(cells, np.uint32)
        if cells.size != (w << v) * 2 * self.engine.params.N1:
            raise ValueError("setRam: image must hold w * 2^v TRLWE cells")
        _check(lib().vsp_netlist_ram(self.h, v, w, None, _ptr(cells)))
        self._ram_geom = (v, w)

    def ram(self) -> np.ndarray:
        if self._ram_geom is None:
            raise RuntimeError("RAM image not bound")
        v, w = self._ram_geom
        out = np.zeros(((w << v), 2 * self.engine.params.N1), np.uint32)
        _check(lib().vsp_netlist_ram(self.h, v, w, _ptr(out), None))
        return out

    def snapshot_save(self, param_name: str | None = None) -> bytes:
        """snapshotSave (snapshot.cpp:84-101): the reference's HVPS bytes."""
        L = lib()
        name = (param_name or self.engine.params.name).encode()
        n = ctypes.c_size_t()
        _check(L.vsp_netlist_snapshot_save(self.h, name, None, 0, ctypes.byref(n)))
        buf = np.zeros(n.value, np.uint8)
        _check(L.vsp_netlist_snapshot_save(self.h, name, _ptr(buf), buf.size, ctypes.byref(n)))
        return buf.tobytes()

    def snapshot_load(self, data: bytes, param_name: str | None = None):
        """snapshotLoad (snapshot.cpp:124-158) into this runner: cycle, DFFs, RAM, ROM."""
        buf = np.frombuffer(bytes(data), np.uint8).copy()
        name = (param_name or self.engine.params.name).encode()
        _check(lib().vsp_netlist_snapshot_load(self.h, name, _ptr(buf), buf.size))
        if self.ram_cell >= 0:
            v, w = ctypes.c_uint32(), ctypes.c_uint32()
            if lib().vsp_netlist_ram_geometry(self.h, ctypes.byref(v), ctypes.byref(w)) == 0:
                self._ram_geom = (int(v.value), int(w.value))

    def run(self, cycles: int, opt: RunOptions | None = None):
        """Evaluator::run (engine.hpp:238-247)."""
        opt = opt or RunOptions()
        st = np.zeros(max(4 * cycles, 4), np.float64)
        _check(lib().vsp_netlist_run(self.h, cycles, _ptr(st)))
        if opt.stats is not None:
            for i in range(cycles):
                opt.stats.append(CycleStats(int(st[4 * i]), int(st[4 * i + 1]),
                                            int(st[4 * i + 2]), float(st[4 * i + 3])))


def snapshot_peek(data: bytes) -> dict:
    """snapshotPeek (snapshot.cpp:165-176): backend tag, parameter set, netlist name."""
    L = _bind()
    buf = np.frombuffer(bytes(data), np.uint8).copy()
    outs = [ctypes.create_string_buffer(256) for _ in range(3)]
    _check(L.vsp_snapshot_peek(_ptr(buf), buf.size, *[ctypes.addressof(o) for o in outs], 256))
    return {"backend": outs[0].value.decode(), "param": outs[1].value.decode(),
            "netlist": outs[2].value.decode()}


class PlainEvaluator:
    """PlainBackend + Evaluator over plaintext bits (engine.hpp:48-71, engine.cpp:65-111):
    the backend-equivalence oracle of SPEC.md:364."""

    def __init__(self, nl: Netlist):
        self.nl = nl
        self.dag = build_dag(nl)
        self.dff = {i: 0 for i in self.dag["dff_cells"]}
        self.inputs = {b: 0 for p in nl.inputs for b in p.bits}
        self.values = [0] * nl.net_count
        self.rom = None
        self.ram = None  # (v, w, words)
        order = sorted(range(len(self.dag["dag_cells"])), key=lambda k: self.dag["level"][k])
        self.order = [self.dag["dag_cells"][k] for k in order]

    def set_input(self, port, idx, v):
        self.inputs[Evaluator._port_bit(self.nl.inputs, port, idx)] = int(v)

    def output(self, port, idx):
        net = Evaluator._port_bit(self.nl.outputs, port, idx)
        for i, q in ((i, self.nl.cells[i].outputs[0]) for i in self.dff):
            if q == net:
                return self.dff[i]
        if net in self.inputs:
            return self.inputs[net]
        return self.values[net]

    def run(self, cycles=1):
        for _ in range(cycles):
            vals = self.values
            for b, v in self.inputs.items():
                vals[b] = v
            for i, v in self.dff.items():
                vals[self.nl.cells[i].outputs[0]] = v
            for ci in self.order:
                c = self.nl.cells[ci]
                if c.kind in GATES:
                    vals[c.outputs[0]] = plain_gate(c.kind, [vals[b] for b in c.inputs])
                else:
                    self._eval_port(c, vals)
            for i in self.dff:
                self.dff[i] = vals[self.nl.cells[i].inputs[0]]

    def _eval_port(self, c, vals):
        """Constants and memory ports (PlainBackend::romRead / ramCycle, engine.cpp:83-111)."""
        x = [vals[b] for b in c.inputs]
        if c.kind == "CONST0":
            vals[c.outputs[0]] = 0
        elif c.kind == "CONST1":
            vals[c.outputs[0]] = 1
        elif c.kind == "ROM":
            blk = sum(b << i for i, b in enumerate(x))
            word = int.from_bytes(bytes(self.rom[4 * blk:4 * blk + 4]), "little")
            for k, o in enumerate(c.outputs):
                vals[o] = (word >> k) & 1
        elif c.kind == "RAM":
            v, w, words = self.ram
            a = sum(b << i for i, b in enumerate(x[:v]))
            old = words[a]
            if x[v + w]:
                words[a] = sum(b << i for i, b in enumerate(x[v:v + w]))
            for k, o in enumerate(c.outputs):
                vals[o] = (old >> k) & 1


class ShardedPlainEvaluator(PlainEvaluator):
    """The multi-GPU runner's schedule on plaintext bits (CPU, any torch.distributed
    backend, e.g. gloo): every ASAP level's gates are split with the runner's own
    task-balanced partition (level_partition with the level's kinds, multi.cuh) and each
    rank evaluates only its slice; the padded slices are all-gathered (the runner's
    all-gather) and repacked before the next level.  The RAM is sharded by bit-block like
    ram_cycle_dev: rank r reads and writes only bits [r w/world, (r+1) w/world) of each
    word and the read-out bits are all-gathered.  The ROM and constants are evaluated on
    every rank, DFFs latch locally.  Must equal PlainEvaluator exactly
    (tests/test_multi_cpu.py)."""

    def __init__(self, nl: Netlist, group=None):
        super().__init__(nl)
        import torch.distributed as dist
        from . import level_partition
        self._dist, self._part, self.group = dist, level_partition, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        lv = self.dag["level"]
        depth = self.dag["depth"]
        self.levels = [[] for _ in range(depth)]
        for node, ci in enumerate(self.dag["dag_cells"]):  # runner order: DAG node order
            self.levels[lv[node]].append(ci)
        self.gate_evals = 0  # gates this rank evaluated (the shard)

    def run(self, cycles=1):
        dist = self._dist
        for _ in range(cycles):
            vals = self.values
            for b, v in self.inputs.items():
                vals[b] = v
            for i, v in self.dff.items():
                vals[self.nl.cells[i].outputs[0]] = v
            for cells in self.levels:
                gates = [ci for ci in cells if self.nl.cells[ci].kind in GATES]
                kinds = [self.nl.cells[ci].kind for ci in gates]
                cut = [self._part(len(gates), self.world, r, kinds)[0] for r in range(self.world)]
                lo, hi, per = self._part(len(gates), self.world, self.rank, kinds)
                mine = [plain_gate(self.nl.cells[ci].kind,
                                   [vals[b] for b in self.nl.cells[ci].inputs])
                        for ci in gates[lo:hi]]
                self.gate_evals += len(mine)
                if gates:
                    box = [None] * self.world
                    dist.all_gather_object(box, mine + [0] * (per - len(mine)), group=self.group)
                    cut.append(len(gates))
                    flat = [x for r in range(self.world) for x in box[r][:cut[r + 1] - cut[r]]]
                    for ci, v in zip(gates, flat):
                        vals[self.nl.cells[ci].outputs[0]] = v
                for ci in cells:
                    c = self.nl.cells[ci]
                    if c.kind in GATES:
                        continue
                    if c.kind == "RAM":
                        self._eval_ram_sharded(c, vals)
                    else:
                        self._eval_port(c, vals)
            for i in self.dff:
                self.dff[i] = vals[self.nl.cells[i].inputs[0]]


    def _eval_ram_sharded(self, c, vals):
        """ramCycle with the RAM sharded by bit-block (ram_cycle_dev, multi.cuh
        ram_blocks): this rank owns bits [j0, j1) of every word."""
        v, w, words = self.ram
        if w % self.world:
            return self._eval_port(c, vals)
        x = [vals[b] for b in c.inputs]
        j0, j1 = self.rank * w // self.world, (self.rank + 1) * w // self.world
        a = sum(b << i for i, b in enumerate(x[:v]))
        mine = [(words[a] >> j) & 1 for j in range(j0, j1)]  # read-before-write
        if x[v + w]:
            for j in range(j0, j1):
                words[a] = (words[a] & ~(1 << j)) | (x[v + j] << j)
        box = [None] * self.world
        self._dist.all_gather_object(box, mine, group=self.group)
        for k, o in enumerate(c.outputs):
            vals[o] = box[k // (w // self.world)][k % (w // self.world)]

    def owned_ram_bits(self) -> int:
        """Mask of the word bits this rank keeps current (its bit-blocks)."""
        v, w, _ = self.ram
        if w % self.world:
            return (1 << w) - 1
        j0, j1 = self.rank * w // self.world, (self.rank + 1) * w // self.world
        return ((1 << j1) - 1) ^ ((1 << j0) - 1)


def plain_gate(kind, x):
    """plainGate (engine.cpp:17-43); MUX inputs {s, a, b}."""
    a = x[0]
    b = x[1] if len(x) > 1 else 0
    return {"AND": a & b, "ANDNOT": a & (1 - b), "NAND": 1 - (a & b), "NOR": 1 - (a | b),
            "OR": a | b, "ORNOT": a | (1 - b), "XNOR": 1 - (a ^ b), "XOR": a ^ b, "NOT": 1 - a,
            "MUX": (x[1] if x[0] else x[2]) if kind == "MUX" else 0}[kind]


# Ruby gate mix of the paper's processor
RUBY_MIX = {"AND": 651, "ANDNOT": 223, "MUX": 996, "NAND": 1025, "NOR": 90, "NOT": 15,
            "OR": 215, "ORNOT": 195, "XNOR": 51, "XOR": 36}


def synthetic_netlist(seed: int = 1, mix: dict | None = None, levels: int = 24, dffs: int = 256,
                      rom: bool = True, ram: tuple | None = (8, 16), rom_addr_bits: int = 7,
                      n_inputs: int = 8, scale: float = 1.0) -> Netlist:
    """Seeded synthetic pipelined-processor netlist in the reference JSON schema: the
    gate mix of CAHP-Ruby spread over `levels` DFF-bounded logic levels, one ROM port and
    one RAM port fed from DFF outputs, RAM/ROM read data latched into DFFs."""
    rng = np.random.default_rng(seed)
    mix = dict(mix or RUBY_MIX)
    kinds = [k for k, c in mix.items() for _ in range(int(round(c * scale)))]
    rng.shuffle(kinds)
    net = 0

    def new():
        nonlocal net
        net += 1
        return net - 1

    cells, cid = [], 0
    nl = Netlist(name=f"synthetic-ruby-{seed}")
    in_bits = [new() for _ in range(n_inputs)]
    nl.inputs.append(Port("in", in_bits))
    q = [new() for _ in range(dffs)]  # DFF outputs (sources)
    sources = list(q) + in_bits
    # memory ports read addresses/data from DFF outputs
    mem_out = []
    if rom:
        rd = [new() for _ in range(32)]
        cells.append(Cell(cid, "ROM", [q[i] for i in range(rom_addr_bits)], rd))
        cid += 1
        mem_out += rd
    if ram:
        v, w = ram
        rd = [new() for _ in range(w)]
        ins = [q[(rom_addr_bits + i) % dffs] for i in range(v)]
        ins += [q[(rom_addr_bits + v + i) % dffs] for i in range(w)] + [q[-1]]
        cells.append(Cell(cid, "RAM", ins, rd))
        cid += 1
        mem_out += rd
    per_level = max(1, len(kinds) // levels)
    prev = sources + mem_out
    avail = list(prev)
    gate_outs = []
    k = 0
    for L in range(levels):
        cur = []
        take = kinds[k:k + per_level] if L < levels - 1 else kinds[k:]
        k += len(take)
        for kind in take:
            ar = 1 if kind == "NOT" else 3 if kind == "MUX" else 2
            # at least one input from the previous level keeps the level structure
            ins = [prev[int(rng.integers(len(prev)))]]
            ins += [avail[int(rng.integers(len(avail)))] for _ in range(ar - 1)]
            y = new()
            cells.append(Cell(cid, kind, ins, [y]))
            cid += 1
            cur.append(y)
        gate_outs += cur
        avail += cur
        prev = cur if cur else prev
    # DFF D inputs: the deepest gates first, then memory read data
    d_src = list(reversed(gate_outs)) + mem_out
    for i in range(dffs):
        d = d_src[i % len(d_src)]
        cells.append(Cell(cid, "DFF", [d], [q[i]], name=f"r{i}"))
        cid += 1
    nl.cells = cells
    nl.outputs.append(Port("out", q[:16]))
    nl.net_count = net
    validate_netlist(nl)
    return nl
