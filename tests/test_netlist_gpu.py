"""GPU netlist runner vs the reference Evaluator<TfheBackend> (oracle/_ref) and vs the
plaintext backend: bit-exact DFF state and outputs on test-det, decrypted equality on
tfhe-80 (SPEC.md:363-368 backend equivalence)."""
import ctypes

import numpy as np
import pytest

import paper_2010_09410_b200 as vsp
from oracle import pyoracle
from oracle.pyoracle import CpuTfhe
from paper_2010_09410_b200 import netlist as N
from tests.helpers import oracle_keys

pytestmark = pytest.mark.gpu


def words_to_image(words, v, w):
    img = np.zeros((w << v) // 8, np.uint8)
    for A, x in enumerate(words):
        for j in range(w):
            if (x >> j) & 1:
                b = A * w + j
                img[b // 8] |= 1 << (b % 8)
    return img


class RefEval:
    """The reference's own Evaluator<TfheBackend> (oracle/_ref, ref_shim.cpp)."""

    def __init__(self, r: CpuTfhe, text: str, threads: int = 4):
        self.r, self.L = r, r.L
        self.threads = threads
        self.h = ctypes.c_void_p(self.L.ref_eval_new(r.h, text.encode(), threads))
        assert self.h.value, self.L.ref_last_error()

    def set_input(self, port, idx, ct):
        assert self.L.ref_eval_set_input(self.h, port.encode(), idx, ct.ctypes.data, self.r.n) == 0

    def output(self, port, idx):
        out = np.zeros(self.r.n + 1, np.uint32)
        assert self.L.ref_eval_output(self.h, port.encode(), idx, out.ctypes.data) == 0
        return out

    def dff(self):
        cnt = self.L.ref_eval_dff_count(self.h)
        out = np.zeros((cnt, self.r.n + 1), np.uint32)
        assert self.L.ref_eval_get_dff(self.h, out.ctypes.data_as(ctypes.c_void_p),
                                       ctypes.c_uint32(self.r.n)) == 0
        return out

    def set_ram(self, ram, v, w):
        assert self.L.ref_eval_set_ram(self.h, v, w, ram.ctypes.data_as(ctypes.c_void_p),
                                       self.r.N1) == 0

    def get_ram(self, shape):
        out = np.zeros(shape, np.uint32)
        assert self.L.ref_eval_get_ram(self.h, out.ctypes.data_as(ctypes.c_void_p)) == 0
        return out

    def set_rom(self, luts, depth):
        assert self.L.ref_eval_set_rom(self.h, depth, luts.ctypes.data_as(ctypes.c_void_p),
                                       luts.shape[0], self.r.N1) == 0

    def run(self, cycles):
        assert self.L.ref_eval_run(self.h, cycles, self.threads, 0, None) == 0, \
            self.L.ref_last_error()

    def set_dff(self, state):
        state = np.ascontiguousarray(state, np.uint32)
        assert self.L.ref_eval_set_dff(self.h, state.ctypes.data_as(ctypes.c_void_p),
                                       ctypes.c_uint32(self.r.n)) == 0


@pytest.mark.skipif(not pyoracle.available("ref"), reason="reference not built")
def test_runner_matches_reference_evaluator_testdet():
    seed = 515253
    r = CpuTfhe("ref", "test-det", seed=seed)
    r.keygen(True)
    e = vsp.Engine("test-det")
    e.upload_keys(oracle_keys("test-det", seed, True))
    nl = N.synthetic_netlist(seed=3, scale=0.03, levels=6, dffs=40, ram=(3, 4))
    text = N.netlist_to_json(nl)
    ev = N.Evaluator(nl, e)
    rev = RefEval(r, text)
    rng = np.random.default_rng(1)
    v, w = 3, 4
    words = [int(x) for x in rng.integers(0, 16, 8)]
    ram = r.encrypt_ram(words_to_image(words, v, w), v, w)
    ev.set_ram(ram, v, w)
    rev.set_ram(ram, v, w)
    rom_img = rng.integers(0, 256, 512).astype(np.uint8)
    luts = r.encrypt_rom(rom_img)
    ev.set_rom(luts, 512)
    rev.set_rom(luts, 512)
    for i in range(len(nl.inputs[0].bits)):
        ct = r.encrypt(int(rng.integers(0, 2)))
        ev.set_input("in", i, ct)
        rev.set_input("in", i, ct)
    init = np.stack([r.encrypt(int(b)) for b in rng.integers(0, 2, ev.n_dffs)])
    ev.set_dff_state_raw(init)
    assert rev.L.ref_eval_set_dff(rev.h, init.ctypes.data_as(ctypes.c_void_p),
                                  ctypes.c_uint32(r.n)) == 0
    stats = []
    for cyc in range(2):
        ev.run(1, N.RunOptions(stats=stats))
        rev.run(1)
        assert np.array_equal(ev.dff_state(), rev.dff()), f"DFF state differs at cycle {cyc}"
        for k in range(16):
            assert np.array_equal(ev.output("out", k), rev.output("out", k))
    assert np.array_equal(ev.ram(), rev.get_ram(ram.shape))
    assert stats[0].evaluated_total == ev.dag_nodes and stats[0].depth == ev.depth
    assert ev.cycle == 2


def _launch_schedule_ok(nl, ev, sms):
    """Launch levels vs the ASAP levels: never earlier, every gate before all of its
    consumers (gates and memory ports), memory ports unmoved.  Returns the latency-kernel
    waves (ceil(tasks / SMs) per level) of the ASAP and of the launch schedule."""
    nodes = [c for c in nl.cells if c.kind != "DFF"]
    asap, launch = ev.levels(), ev.launch_levels()
    assert np.all(launch >= asap) and launch.max() == asap.max()
    producer = {b: i for i, c in enumerate(nodes) for b in c.outputs}
    for i, c in enumerate(nodes):
        for b in c.inputs:
            if b in producer:
                assert launch[producer[b]] < launch[i], (producer[b], i)
        if c.kind in ("ROM", "RAM", "CONST0", "CONST1"):
            assert launch[i] == asap[i]

    def waves(lv):
        t = {}
        for i, c in enumerate(nodes):
            cost = 2 if c.kind == "MUX" else 0 if c.kind in ("NOT", "ROM", "RAM", "CONST0", "CONST1") else 1
            t[lv[i]] = t.get(lv[i], 0) + cost
        return sum(-(-x // sms) for x in t.values())
    return waves(asap), waves(launch)


def test_level_balancing_schedule_matches_reference_evaluator_testdet():
    """Levels wider than one latency wave (more blind-rotation tasks than SMs) hand their
    gates with slack to the next level (vsp_netlist_launch_levels); the runner's DFF state,
    outputs and RAM stay word-for-word equal to the reference Evaluator<TfheBackend>,
    which evaluates the ASAP levels."""
    if not pyoracle.available("ref"):
        pytest.skip("reference not built")
    seed = 515253
    r = CpuTfhe("ref", "test-det", seed=seed)
    r.keygen(True)
    e = vsp.Engine("test-det")
    e.upload_keys(oracle_keys("test-det", seed, True))
    nl = N.synthetic_netlist(seed=3, scale=0.134, levels=4, dffs=48, ram=(3, 4))
    ev = N.Evaluator(nl, e)
    w_asap, w_launch = _launch_schedule_ok(nl, ev, e.sms)
    assert w_launch <= w_asap
    if e.sms == 148:
        assert w_launch < w_asap, (w_asap, w_launch)
    rev = RefEval(r, N.netlist_to_json(nl))
    rng = np.random.default_rng(4)
    v, w = 3, 4
    ram = r.encrypt_ram(words_to_image([int(x) for x in rng.integers(0, 16, 8)], v, w), v, w)
    ev.set_ram(ram, v, w)
    rev.set_ram(ram, v, w)
    luts = r.encrypt_rom(rng.integers(0, 256, 512).astype(np.uint8))
    ev.set_rom(luts, 512)
    rev.set_rom(luts, 512)
    for i in range(len(nl.inputs[0].bits)):
        ct = r.encrypt(int(rng.integers(0, 2)))
        ev.set_input("in", i, ct)
        rev.set_input("in", i, ct)
    init = np.stack([r.encrypt(int(b)) for b in rng.integers(0, 2, ev.n_dffs)])
    ev.set_dff_state_raw(init)
    rev.set_dff(init)
    for cyc in range(2):
        ev.run(1)
        rev.run(1)
        assert np.array_equal(ev.dff_state(), rev.dff()), f"DFF state differs at cycle {cyc}"
        for k in range(16):
            assert np.array_equal(ev.output("out", k), rev.output("out", k))
    assert np.array_equal(ev.ram(), rev.get_ram(ram.shape))


def test_level_balancing_on_the_bench_netlist():
    """The bench's cycle netlist (one ASAP level of 149 tasks) launches every level in a
    single latency wave on a 148-SM B200."""
    e = vsp.Engine("test-det")
    e.upload_keys(oracle_keys("test-det", 515253, True))
    nl = N.synthetic_netlist(seed=1, levels=32)
    ev = N.Evaluator(nl, e)
    w_asap, w_launch = _launch_schedule_ok(nl, ev, e.sms)
    assert w_launch <= w_asap
    if e.sms == 148:
        assert (w_asap, w_launch) == (ev.depth + 1, ev.depth), (w_asap, w_launch)


def test_runner_backend_equivalence_tfhe80():
    """Decrypted TFHE outputs == PlainBackend outputs every cycle (no memory ports)."""
    p = vsp.ParameterSet("tfhe-80")
    k = vsp.keygen(p, 31, False)
    e = vsp.Engine(p)
    e.upload_keys(k)
    nl = N.synthetic_netlist(seed=5, scale=0.04, levels=8, dffs=32, rom=False, ram=None)
    ev = N.Evaluator(nl, e)
    pe = N.PlainEvaluator(nl)
    rng = np.random.default_rng(2)
    bits = rng.integers(0, 2, ev.n_dffs)
    ev.set_dff_state_raw(vsp.encrypt(p, k["lv0"], bits, 3))
    for i, di in enumerate(pe.dff):
        pe.dff[di] = int(bits[i])
    for cyc in range(3):
        ib = rng.integers(0, 2, len(nl.inputs[0].bits))
        cts = vsp.encrypt(p, k["lv0"], ib, 100 + cyc)
        for i, b in enumerate(ib):
            ev.set_input("in", i, cts[i])
            pe.set_input("in", i, int(b))
        ev.run(1)
        pe.run(1)
        got = vsp.decrypt(k["lv0"], ev.dff_state())
        want = np.array([pe.dff[i] for i in sorted(pe.dff)], np.uint8)
        assert np.array_equal(got, want), f"cycle {cyc}"
        outs = vsp.decrypt(k["lv0"], np.stack([ev.output("out", j) for j in range(16)]))
        assert list(outs) == [pe.output("out", j) for j in range(16)]


def test_runner_errors():
    e = vsp.Engine("test-det")
    e.upload_keys(oracle_keys("test-det", 515253, True))
    nl = N.synthetic_netlist(seed=4, scale=0.01, levels=3, dffs=16, ram=(2, 2))
    ev = N.Evaluator(nl, e)
    with pytest.raises(RuntimeError, match="needs an evaluated cycle|ROM image not bound"):
        ev.output("out", 0) if False else ev.run(1)
    with pytest.raises(RuntimeError):
        ev.set_input("nope", 0, np.zeros(17, np.uint32))


@pytest.mark.parametrize("bad, match", [
    # a 3-input AND would overflow the runner's 3-slot gather (advisor finding r01)
    (lambda nl: nl.cells.append(N.Cell(90, "AND", [0, 1, 2], [5])), "wrong input count"),
    (lambda nl: nl.cells.append(N.Cell(91, "NAND", [0, 1], [])), "exactly one net"),
    (lambda nl: nl.cells.append(N.Cell(92, "XOR", [0, 1], [5, 6])), "exactly one net"),
    (lambda nl: nl.inputs.append(N.Port("x", [999])), "bad net 999"),
    (lambda nl: nl.cells.append(N.Cell(93, "OR", [0, 77], [5])), "dangling input net 77"),
    (lambda nl: nl.cells.append(N.Cell(0, "OR", [0, 1], [5])), "duplicate cell id 0"),
    (lambda nl: nl.cells.append(N.Cell(94, "OR", [0, 1], [3])), "multiple drivers on net 3"),
])
def test_flat_netlist_validated_by_c_abi(bad, match):
    """vsp_netlist_create validates the flat arrays like validateNetlist (netlist.cpp:
    265-345) before anything indexes them -- the Python parser is bypassed here."""
    e = vsp.Engine("test-det")
    nl = N.Netlist(name="v", inputs=[N.Port("in", [0, 1])], outputs=[N.Port("out", [3])],
                   cells=[N.Cell(0, "AND", [0, 1], [2]), N.Cell(1, "NOT", [2], [3])],
                   net_count=8)
    N.Evaluator(nl, e).close()  # the valid base netlist is accepted
    bad(nl)
    with pytest.raises(RuntimeError, match=match):
        N.Evaluator(nl, e)


def test_runner_ram_overlap_equals_inline():
    """ram_overlap (write bars deferred to a low-priority stream beside the later levels,
    narrow levels at two tasks per SM, joined before the next RAM access) gives the same
    words as the inline schedule: DFF state, outputs and RAM image over 3 cycles, and the
    RAM getter joins the deferred write."""
    p = vsp.ParameterSet("tfhe-80")
    k = vsp.keygen(p, 2207, True, device=0)
    nl = N.synthetic_netlist(seed=9, scale=0.05, levels=6, dffs=48, ram=(4, 8))
    rng = np.random.default_rng(9)
    v, w = 4, 8
    ram = vsp.encrypt_ram(p, k, rng.integers(0, 256, (w << v) // 8).astype(np.uint8), v, w, 1)
    luts = vsp.encrypt_rom(p, k, rng.integers(0, 256, 512).astype(np.uint8), 2)
    dff0 = vsp.encrypt(p, k["lv0"], rng.integers(0, 2, 48).astype(np.uint8), 3)
    ins = vsp.encrypt(p, k["lv0"], rng.integers(0, 2, len(nl.inputs[0].bits)).astype(np.uint8), 4)
    res = []
    for overlap in (0, 1):
        e = vsp.Engine(p)
        e.upload_keys(k)
        e.set_option("ram_overlap", overlap)
        ev = N.Evaluator(nl, e)
        ev.set_ram(ram, v, w)
        ev.set_rom(luts, 512)
        ev.set_dff_state_raw(dff0)
        for i, ct in enumerate(ins):
            ev.set_input("in", i, ct)
        trace = []
        for _ in range(3):
            ev.run(1)
            trace.append((ev.dff_state(), np.stack([ev.output("out", j) for j in range(16)])))
        res.append((trace, ev.ram()))
        ev.close()
        e.close()
    (t0, r0), (t1, r1) = res
    for (d0, o0), (d1, o1) in zip(t0, t1):
        assert np.array_equal(d0, d1) and np.array_equal(o0, o1)
    assert np.array_equal(r0, r1)
