"""Word-exact parity at the production parameters (tfhe-80 with n = 630, BASELINE.json),
through the C ABI, against the reference itself (oracle/_ref: hvp compiled from its
sources) on identical keys and ciphertexts.

* the headline workload (4,096 NAND/XOR gates) word for word against the reference's
  homGate, with the launch plan asserted (whole W=8 waves + a W=4 remainder, key switch
  forked under the remainder, host pipeline);
* every CMUX-memory unit on client-encrypted selectors (ramReadUnit, ramControlUnit,
  ramWriteUnit at the full 4,096-cell geometry, romRead) against the reference's units --
  this runs the production cmux_chain1024 kernel in both modes, the key switch and the
  write-bar blind rotations;
* circuitBootstrap: the level-2 blind rotation against the restatement's exact mode
  (MulBackend::Exact semantics, Karatsuba products) at full n = 630, and the private key
  switches + row assembly against the reference's privateKeySwitch on the same level-2
  samples.

The reference's level-2 FFT (fft.hpp:67-69) is inexact (it accepts 2^30 of error,
test_tfhe.cpp:142-175), so a GPU circuit bootstrap cannot equal the reference's FFT one
word for word; it equals the Exact backend's.  tests/test_noise_gpu.py bounds its noise
against the reference's.
"""
import os

import numpy as np
import pytest

import paper_2010_09410_b200 as vsp
from oracle.pyoracle import CpuTfhe, GATE_KINDS, available
from tests.helpers import TRUTH, keys_with_cb

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")]

N630 = 630
THREADS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def prod630():
    p = vsp.ParameterSet("tfhe-80", n_override=N630)
    k = keys_with_cb(N630, 630)
    e = vsp.Engine(p)
    e.upload_keys(k)
    ref = CpuTfhe("ref", "tfhe-80", n_override=N630, seed=630)
    ref.import_keys(k)
    return e, ref, k, p


def enc_bits(p, k, bits, seed):
    return vsp.encrypt(p, k["lv0"], np.asarray(bits, np.uint8), seed)


def test_headline_4096_gates_word_exact_vs_reference(prod630):
    """BASELINE configs[0] exactly as bench.py runs it: 4,096 random NAND/XOR gates at
    n = 630 (three whole W=8 waves + a 544-task remainder on the two-warps-per-task
    kernel, key switch as one INT8 GEMM).  Every output word equals the reference's homGate (ops.cpp:839-896) on the
    same keys and ciphertexts, through both the host-pipelined C-ABI call and the
    device-resident call."""
    import torch
    e, ref, k, p = prod630
    if e.sms == 148:
        assert e.br_plan(4096) == {"lat": False, "full": 3552, "w_rem": 4, "rem_kernel": "br1024p"}
    rng = np.random.default_rng(4096)
    G = 4096
    kid = rng.choice([GATE_KINDS.index("NAND"), GATE_KINDS.index("XOR")], G).astype(np.int32)
    bits = rng.integers(0, 2, size=(G, 2)).astype(np.uint8)
    ins = np.zeros((G, 3, p.n + 1), np.uint32)
    ins[:, :2] = enc_bits(p, k, bits.reshape(-1), 4097).reshape(G, 2, p.n + 1)
    out = e.hom_gate_batch(kid, ins)
    d_in = torch.from_numpy(ins.view(np.int32)).cuda()
    d_out = torch.empty((G, p.n + 1), dtype=torch.int32, device="cuda")
    e.hom_gate_batch_dev(kid, d_in.data_ptr(), d_out.data_ptr(), G)
    torch.cuda.synchronize()
    want = ref.hom_gate_batch(kid, ins, threads=THREADS)
    assert np.array_equal(out, want)
    assert np.array_equal(d_out.cpu().numpy().view(np.uint32), want)
    truth = np.array([TRUTH[GATE_KINDS[g]](int(a), int(b), 0) for g, (a, b) in zip(kid, bits)])
    assert np.array_equal(vsp.decrypt(k["lv0"], out), truth)


def test_all_gate_kinds_mixed_batch_word_exact_vs_reference(prod630):
    """All ten kinds (MUX = two blind rotations, NOT = none) in one batch wide enough for
    a whole W=8 wave + remainder, word for word against the reference."""
    e, ref, k, p = prod630
    rng = np.random.default_rng(2100)
    G = 2100
    kid = rng.integers(0, len(GATE_KINDS), G).astype(np.int32)
    bits = rng.integers(0, 2, size=(G, 3)).astype(np.uint8)
    ins = enc_bits(p, k, bits.reshape(-1), 2101).reshape(G, 3, p.n + 1)
    tasks = int(sum(2 if g == 2 else 0 if g == 5 else 1 for g in kid))
    if e.sms == 148:
        assert not e.br_plan(tasks)["lat"]
    out = e.hom_gate_batch(kid, ins)
    assert np.array_equal(out, ref.hom_gate_batch(kid, ins, threads=THREADS))


def _selectors(ref, bits):
    return np.stack([ref.trgsw_encrypt(int(b)) for b in bits])


def words_to_image(words, v, w):
    img = np.zeros((w << v) // 8, np.uint8)
    for A, x in enumerate(words):
        for j in range(w):
            if (x >> j) & 1:
                b = A * w + j
                img[b // 8] |= 1 << (b % 8)
    return img


@pytest.fixture(scope="module")
def ram630(prod630):
    e, ref, k, p = prod630
    rng = np.random.default_rng(512)
    v, w = 8, 16
    words = [int(x) for x in rng.integers(0, 1 << w, 1 << v)]
    ram = vsp.encrypt_ram(p, k, words_to_image(words, v, w), v, w, 513)
    return v, w, words, ram


def test_ram_read_unit_full_size_word_exact(prod630, ram630):
    """ramReadUnit (mem.cpp:49-72) at v=8, w=16: 16 trees x 255 CMUXes on the production
    cmux_chain1024 kernel (mode 0, one step per task), client-encrypted selectors."""
    e, ref, k, p = prod630
    v, w, words, ram = ram630
    A = 0b10110101
    sel = _selectors(ref, [(A >> d) & 1 for d in range(v)])
    got = e.ram_read_unit(ram, v, w, sel)
    want = ref.ram_read_unit(ram, v, w, sel, threads=THREADS)
    assert np.array_equal(got, want)
    dec = vsp.trlwe_decrypt_at(k["lv1"], got, 0)
    assert sum(int(b) << j for j, b in enumerate(dec)) == words[A]


def test_ram_control_unit_word_exact(prod630, ram630):
    """ramControlUnit (mem.cpp:74-90): 16 key switches + 16 homMuxNoSeIks (32 blind
    rotations on the narrow-level kernel)."""
    e, ref, k, p = prod630
    v, w, words, ram = ram630
    rng = np.random.default_rng(74)
    rbits = np.zeros((w, p.N1), np.uint8)
    rbits[:, 0] = rng.integers(0, 2, w)
    read = vsp.trlwe_encrypt(p, k["lv1"], rbits, 75)
    for wf in (0, 1):
        wflag = enc_bits(p, k, [wf], 76 + wf)[0]
        wdata = enc_bits(p, k, rng.integers(0, 2, w), 78 + wf)
        ro, ctl = e.ram_control_unit(read, wflag, wdata)
        ro_r, ctl_r = ref.ram_control_unit(read, wflag, wdata, threads=THREADS)
        assert np.array_equal(ro, ro_r)
        assert np.array_equal(ctl, ctl_r)


def test_ram_write_unit_full_size_word_exact(prod630, ram630):
    """ramWriteUnit (mem.cpp:92-120) at the full 4,096-cell geometry: 32,768 address-match
    CMUXes (cmux_chain1024, 8-step chains), 4,096 key switches and 4,096 write-bar blind
    rotations (whole W=8 waves + remainder, key switch under the remainder wave).  Every
    word of the new RAM image equals the reference's."""
    e, ref, k, p = prod630
    v, w, words, ram = ram630
    if e.sms == 148:
        assert e.br_plan(w << v) == {"lat": False, "full": 3552, "w_rem": 4, "rem_kernel": "br1024p"}
    A, X = 77, 0xC0DE
    sel = _selectors(ref, [(A >> d) & 1 for d in range(v)])
    bits = np.zeros((w, p.N1), np.uint8)
    bits[:, 0] = [(X >> j) & 1 for j in range(w)]
    controlled = vsp.trlwe_encrypt(p, k["lv1"], bits, 79)
    got = e.ram_write_unit(ram, v, w, sel, controlled)
    want = ref.ram_write_unit(ram, v, w, sel, controlled, threads=THREADS)
    assert np.array_equal(got, want)
    model = list(words)
    model[A] = X
    assert np.array_equal(vsp.decrypt_ram(k, got, v, w), words_to_image(model, v, w))


@pytest.mark.parametrize("blk", [0, 45, 99, 127])
def test_rom_read_word_exact(prod630, blk):
    """romRead (mem.cpp:137-177) of a 512 B ROM on client-encrypted selectors: the tree
    CMUXes (mode 0) and the low-bit rotation chain (cmux_chain1024 mode 1), then 32
    sample-extract + key switches at indices 0..31."""
    e, ref, k, p = prod630
    rng = np.random.default_rng(377)
    img = rng.integers(0, 256, 512).astype(np.uint8)
    luts = vsp.encrypt_rom(p, k, img, 378)
    sel = _selectors(ref, [(blk >> d) & 1 for d in range(7)])
    got = e.rom_read_sel(luts, 512, sel)
    assert np.array_equal(got, ref.rom_read_sel(luts, 512, sel, threads=THREADS))
    dec = vsp.decrypt(k["lv0"], got)
    assert sum(int(b) << i for i, b in enumerate(dec)) == \
        int.from_bytes(bytes(img[4 * blk:4 * blk + 4]), "little")


def test_cmux_chain_255_production_word_exact(prod630):
    """test_tfhe.cpp:363-380 on the GPU: 255 chained CMUXes with a selector encrypting 1 at
    production parameters; every intermediate equals the reference's cmux and the result
    still decrypts to p."""
    e, ref, k, p = prod630
    rng = np.random.default_rng(12)
    pb = rng.integers(0, 2, p.N1).astype(np.uint8)
    qb = rng.integers(0, 2, p.N1).astype(np.uint8)
    acc = vsp.trlwe_encrypt(p, k["lv1"], pb, 13)[0]
    other = vsp.trlwe_encrypt(p, k["lv1"], qb, 14)[0]
    sel = ref.trgsw_encrypt(1)
    acc_r = acc.copy()
    for i in range(255):
        acc = e.cmux(sel[None], acc[None], other[None])[0]
        acc_r = ref.cmux(sel, acc_r, other)
        assert np.array_equal(acc, acc_r), f"step {i}"
    dec = np.array([vsp.trlwe_decrypt_at(k["lv1"], acc, kk)[0] for kk in range(p.N1)])
    assert np.array_equal(dec, pb)


def _sample_extract64(acc, N):
    a, b = acc[:N], acc[N:]
    out = np.zeros(N + 1, np.uint64)
    out[0] = a[0]
    out[1:N] = (np.uint64(0) - a[N - np.arange(1, N)])
    out[N] = b[0]
    return out


def test_circuit_bootstrap_n630_word_exact(prod630):
    """circuitBootstrap (ops.cpp:914-935) at n = 630, both halves word-exact:
    (1) the level-2 blind rotation (br2q, four-CTA clusters) == the restatement's exact
        mode (MulBackend::Exact semantics) for both gadget levels;
    (2) SE + b += h/2 + privateKeySwitch(pksNegS / pksId) of those samples, computed by the
        reference, == the rows of the GPU's TRGSW (pks_kernel)."""
    e, ref, k, p = prod630
    bits = [1, 0, 1]
    x = enc_bits(p, k, bits, 915)
    cb = e.circuit_bootstrap(x)
    orc = CpuTfhe("orc", "tfhe-80", n_override=N630, seed=630)
    orc.import_keys({**k, "pks_negs": None, "pks_id": None})
    orc.set_exact(True)
    l = p.l1
    for lev in range(l):
        h = 1 << (64 - (lev + 1) * p.Bg1Bits)
        acc = e.blind_rotate_lvl2(x, h)
        assert np.array_equal(acc, orc.blind_rotate_lvl2_batch(x, h, threads=THREADS)), lev
        for c in range(len(bits)):
            t2 = _sample_extract64(acc[c], p.N2)
            t2[p.N2] += np.uint64(h // 2)
            assert np.array_equal(cb[c, lev].reshape(-1), ref.private_key_switch(t2, 0))
            assert np.array_equal(cb[c, l + lev].reshape(-1), ref.private_key_switch(t2, 1))


def _runner_pair(prod630, nl, threads=THREADS):
    from paper_2010_09410_b200 import netlist as N
    from tests.test_netlist_gpu import RefEval
    e, ref, k, p = prod630
    return N.Evaluator(nl, e), RefEval(ref, N.netlist_to_json(nl), threads)


def test_runner_gate_only_word_exact_vs_reference_evaluator_n630(prod630):
    """The level-batched runner vs the reference's Evaluator<TfheBackend> (engine.hpp:
    263-351) at n = 630 on a gate-only netlist: DFF state and outputs word for word after
    every cycle."""
    from paper_2010_09410_b200 import netlist as N
    e, ref, k, p = prod630
    nl = N.synthetic_netlist(seed=7, scale=0.06, levels=5, dffs=48, rom=False, ram=None)
    ev, rev = _runner_pair(prod630, nl)
    rng = np.random.default_rng(70)
    init = enc_bits(p, k, rng.integers(0, 2, ev.n_dffs), 71)
    ev.set_dff_state_raw(init)
    rev.set_dff(init)
    for cyc in range(2):
        cts = enc_bits(p, k, rng.integers(0, 2, len(nl.inputs[0].bits)), 72 + cyc)
        for i, ct in enumerate(cts):
            ev.set_input("in", i, ct)
            rev.set_input("in", i, np.ascontiguousarray(ct))
        ev.run(1)
        rev.run(1)
        assert np.array_equal(ev.dff_state(), rev.dff()), f"cycle {cyc}"
        for j in range(16):
            assert np.array_equal(ev.output("out", j), rev.output("out", j))


def test_runner_with_memory_ports_matches_reference_evaluator_n630(prod630):
    """Same with a ROM port (512 B) and a RAM port (v=4, w=8) at n = 630.  The memory ports'
    circuit bootstraps are exact on the GPU and inexact (FFT) in the reference, so
    ciphertexts differ after the first memory access; decrypted DFF state, outputs and RAM
    image must be equal every cycle (and the gate-only parts word-exact, above)."""
    from paper_2010_09410_b200 import netlist as N
    e, ref, k, p = prod630
    nl = N.synthetic_netlist(seed=8, scale=0.05, levels=5, dffs=40, ram=(4, 8))
    ev, rev = _runner_pair(prod630, nl)
    rng = np.random.default_rng(80)
    v, w = 4, 8
    words = [int(x) for x in rng.integers(0, 256, 16)]
    ram = vsp.encrypt_ram(p, k, words_to_image(words, v, w), v, w, 81)
    luts = vsp.encrypt_rom(p, k, rng.integers(0, 256, 512).astype(np.uint8), 82)
    for x in (ev, rev):
        x.set_ram(ram, v, w)
        x.set_rom(luts, 512)
    init = enc_bits(p, k, rng.integers(0, 2, ev.n_dffs), 83)
    ev.set_dff_state_raw(init)
    rev.set_dff(init)
    for cyc in range(3):
        cts = enc_bits(p, k, rng.integers(0, 2, len(nl.inputs[0].bits)), 84 + cyc)
        for i, ct in enumerate(cts):
            ev.set_input("in", i, ct)
            rev.set_input("in", i, np.ascontiguousarray(ct))
        ev.run(1)
        rev.run(1)
        dec = lambda x: vsp.decrypt(k["lv0"], x)
        assert np.array_equal(dec(ev.dff_state()), dec(rev.dff())), f"cycle {cyc}"
        assert np.array_equal(dec(np.stack([ev.output("out", j) for j in range(16)])),
                              dec(np.stack([rev.output("out", j) for j in range(16)])))
        assert np.array_equal(vsp.decrypt_ram(k, ev.ram(), v, w),
                              vsp.decrypt_ram(k, rev.get_ram(ram.shape), v, w))


def test_write_bar_backfill_equals_inline_write_unit_n630(prod630):
    """The runner's write-bar backfill (the RAM write unit's remainder blind rotations run in
    the idle SMs of later narrow levels) at the bench's RAM geometry (v=8, w=16: 4,096
    cells, three whole waves + a 544-cell remainder) gives the same DFF state, outputs and
    RAM image, word for word, as the write unit run inline (backfill off) -- which the other
    runner tests pin to the reference Evaluator."""
    from paper_2010_09410_b200 import netlist as N
    e, ref, k, p = prod630
    nl = N.synthetic_netlist(seed=12, scale=0.1, levels=6, dffs=48, ram=(8, 16))
    rng = np.random.default_rng(120)
    v, w = 8, 16
    words = [int(x) for x in rng.integers(0, 1 << w, 1 << v)]
    ram = vsp.encrypt_ram(p, k, words_to_image(words, v, w), v, w, 121)
    luts = vsp.encrypt_rom(p, k, rng.integers(0, 256, 512).astype(np.uint8), 122)
    init = enc_bits(p, k, rng.integers(0, 2, 48), 123)
    ins = [enc_bits(p, k, rng.integers(0, 2, len(nl.inputs[0].bits)), 124 + c) for c in range(2)]

    def run(backfill):
        e.set_option("backfill", backfill)
        try:
            ev = N.Evaluator(nl, e)
            ev.set_ram(ram, v, w)
            ev.set_rom(luts, 512)
            ev.set_dff_state_raw(init)
            before = e.get_option("bars_backfilled")
            outs = []
            for cts in ins:
                for i, ct in enumerate(cts):
                    ev.set_input("in", i, ct)
                ev.run(1)
                outs.append(np.stack([ev.output("out", j) for j in range(16)]))
            return ev.dff_state(), np.stack(outs), ev.ram(), e.get_option("bars_backfilled") - before
        finally:
            e.set_option("backfill", 1)

    dff_a, out_a, ram_a, bars_a = run(1)
    dff_b, out_b, ram_b, bars_b = run(0)
    assert bars_b == 0 and bars_a > 0, (bars_a, bars_b)
    assert np.array_equal(dff_a, dff_b) and np.array_equal(out_a, out_b)
    assert np.array_equal(ram_a, ram_b)


def test_cycle_graph_replay_equals_eager_n630(prod630):
    """The runner's cycle as a CUDA graph (captured after one eager cycle, then replayed)
    gives the same DFF state, outputs and RAM image, word for word, every cycle, as eager
    cycles; the op counters and kernel-launch counts per cycle agree too, and a rebound ROM
    forces a new capture."""
    from paper_2010_09410_b200 import netlist as N
    e, ref, k, p = prod630
    nl = N.synthetic_netlist(seed=14, scale=0.06, levels=5, dffs=40, ram=(4, 8))
    rng = np.random.default_rng(140)
    v, w = 4, 8
    ram = vsp.encrypt_ram(p, k, words_to_image([int(x) for x in rng.integers(0, 256, 16)], v, w),
                          v, w, 141)
    luts = vsp.encrypt_rom(p, k, rng.integers(0, 256, 512).astype(np.uint8), 142)
    luts2 = vsp.encrypt_rom(p, k, rng.integers(0, 256, 512).astype(np.uint8), 143)
    init = enc_bits(p, k, rng.integers(0, 2, 40), 144)
    ins = [enc_bits(p, k, rng.integers(0, 2, len(nl.inputs[0].bits)), 145 + c) for c in range(5)]

    def run(graph):
        e.set_option("graph", graph)
        try:
            ev = N.Evaluator(nl, e)
            ev.set_ram(ram, v, w)
            ev.set_rom(luts, 512)
            ev.set_dff_state_raw(init)
            res = []
            for cyc, cts in enumerate(ins):
                if cyc == 3:
                    ev.set_rom(luts2, 512)
                for i, ct in enumerate(cts):
                    ev.set_input("in", i, ct)
                e.counters_reset()
                l0 = e.kernel_launches()
                ev.run(1)
                res.append((ev.dff_state(), np.stack([ev.output("out", j) for j in range(16)]),
                            ev.ram(), e.counters(), e.kernel_launches() - l0))
            ev.close()
            return res
        finally:
            e.set_option("graph", 1)

    eager, graph = run(0), run(1)
    for cyc, (a, b) in enumerate(zip(eager, graph)):
        for x, y in zip(a[:3], b[:3]):
            assert np.array_equal(x, y), f"cycle {cyc}"
        assert a[3] == b[3] and a[4] == b[4], (cyc, a[3:], b[3:])
