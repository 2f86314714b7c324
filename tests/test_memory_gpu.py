"""GPU parity of circuit bootstrapping and CMUX Memory (mem.cpp) against the oracle.

test-det (MulBackend::Exact on both sides): bit-exact TRGSWs, RAM cells, read-outs and
ROM outputs plus the reference's instrumented counts.  tfhe-80: the level-2 blind
rotation is exact on the GPU (lo/hi split) and is checked bit-exact against the oracle's
exact mode; the full memory path is checked functionally (decryption vs a plaintext
model, test_mem.cpp's PlainRam) because the reference's own level-2 FFT is inexact.
"""
import numpy as np
import pytest

import paper_2010_09410_b200 as vsp
from oracle.pyoracle import CpuTfhe
from tests.helpers import golden, oracle, oracle_keys

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def det():
    e = vsp.Engine("test-det")
    e.upload_keys(oracle_keys("test-det", 515253, True))
    return e, oracle("test-det", 515253, True)


def words_to_image(words, v, w):
    img = np.zeros((w << v) // 8, np.uint8)
    for A, x in enumerate(words):
        for j in range(w):
            if (x >> j) & 1:
                b = A * w + j
                img[b // 8] |= 1 << (b % 8)
    return img


def enc_word(o, x, width):
    return np.stack([o.encrypt((x >> i) & 1) for i in range(width)])


def dec_word(o, cts):
    return sum(o.decrypt(c) << i for i, c in enumerate(cts))


def test_circuit_bootstrap_golden_and_oracle(det):
    e, o = det
    g = golden("testdet_seed515253.npz")
    out = e.circuit_bootstrap(g["cb_in"])
    assert np.array_equal(out, g["cb_out"])
    x = np.stack([o.encrypt(1), o.encrypt(0), o.encrypt(1)])
    out = e.circuit_bootstrap(x)
    for i in range(3):
        assert np.array_equal(out[i], o.circuit_bootstrap(x[i]))


def test_cmux_and_hom_mux_bit_exact(det):
    e, o = det
    rng = np.random.default_rng(2)
    sels = np.stack([o.trgsw_encrypt(int(b)) for b in (1, 0, 1)])
    c1 = np.stack([o.trlwe_encrypt(rng.integers(0, 2, o.N1)) for _ in range(3)])
    c0 = np.stack([o.trlwe_encrypt(rng.integers(0, 2, o.N1)) for _ in range(3)])
    out = e.cmux(sels, c1, c0)
    for i in range(3):
        assert np.array_equal(out[i], o.cmux(sels[i], c1[i], c0[i]))
    s = np.stack([o.encrypt(b) for b in (0, 1, 1, 0)])
    a = np.stack([o.encrypt(b) for b in (1, 1, 0, 0)])
    b = np.stack([o.encrypt(b) for b in (0, 0, 1, 1)])
    out = e.hom_mux_no_se_iks(s, a, b)
    for i in range(4):
        assert np.array_equal(out[i], o.hom_mux_no_se_iks(s[i], a[i], b[i]))


def test_ram_cycle_bit_exact_and_counts(det):
    e, o = det
    rng = np.random.default_rng(4)
    v, w = 3, 4
    words = [int(x) for x in rng.integers(0, 1 << w, 1 << v)]
    ram = o.encrypt_ram(words_to_image(words, v, w), v, w)
    for A, wf, X in [(5, 1, 9), (2, 0, 3), (5, 1, 1)]:
        addr = enc_word(o, A, v)
        f = o.encrypt(wf)
        d = enc_word(o, X, w)
        e.counters_reset()
        o.counters_reset()
        ro_g, ram_g = e.ram_cycle(ram, v, w, addr, f, d)
        ro_o, ram_o = o.ram_cycle(ram, v, w, addr, f, d)
        assert np.array_equal(ro_g, ro_o)
        assert np.array_equal(ram_g, ram_o)
        assert dec_word(o, ro_g) == words[A]
        if wf:
            words[A] = X
        c, oc = e.counters(), o.counters()
        assert [c[k] for k in ("cmux", "blindRotate", "identityKeySwitch", "privateKeySwitch",
                               "circuitBootstrap")] == [int(x) for x in oc]
        ram = ram_g
    img = o.decrypt_ram(ram, v, w)
    assert np.array_equal(img, words_to_image(words, v, w))


def test_ram_cycle_matches_plain_model_v2(det):
    """test_mem.cpp:306-328 style: random ops against PlainRam."""
    e, o = det
    rng = np.random.default_rng(5)
    v, w = 2, 4
    model = [int(x) for x in rng.integers(0, 16, 4)]
    ram = o.encrypt_ram(words_to_image(model, v, w), v, w)
    for _ in range(6):
        A, wf, X = int(rng.integers(0, 4)), int(rng.integers(0, 2)), int(rng.integers(0, 16))
        ro, ram = e.ram_cycle(ram, v, w, enc_word(o, A, v), o.encrypt(wf), enc_word(o, X, w))
        assert dec_word(o, ro) == model[A]
        if wf:
            model[A] = X
    assert np.array_equal(o.decrypt_ram(ram, v, w), words_to_image(model, v, w))


def test_rom_read_bit_exact(det):
    e, o = det
    rng = np.random.default_rng(6)
    img = rng.integers(0, 256, 512).astype(np.uint8)
    luts = o.encrypt_rom(img)
    for blk in (0, 77, 127):
        addr = enc_word(o, blk, 7)
        got = e.rom_read(luts, 512, addr)
        assert np.array_equal(got, o.rom_read(luts, 512, addr))
        want = int.from_bytes(bytes(img[4 * blk:4 * blk + 4]), "little")
        assert dec_word(o, got) == want


def test_memory_errors(det):
    e, o = det
    with pytest.raises(ValueError):
        e.rom_read(np.zeros((64, 2 * o.N1), np.uint32), 512, enc_word(o, 0, 6))
    with pytest.raises(ValueError):
        e.ram_cycle(np.zeros((16, 2 * o.N1), np.uint32), 2, 4, enc_word(o, 0, 3), o.encrypt(0),
                    enc_word(o, 0, 4))
    plain = vsp.Engine("test-det")
    plain.upload_keys(oracle_keys("test-det", 20200729, False))
    with pytest.raises(RuntimeError):
        plain.circuit_bootstrap(o.encrypt(1)[None])


@pytest.mark.parametrize("h_lev", [0, 1])
def test_level2_blind_rotation_exact_tfhe80(h_lev):
    """GPU level-2 FFT path (exact lo/hi split) == oracle schoolbook, bit for bit
    (n reduced to 6 so the O(N^2) oracle stays fast; the kernel is n-agnostic)."""
    p = vsp.ParameterSet("tfhe-80", 6)
    k = vsp.keygen(p, 99, 2)
    e = vsp.Engine(p)
    e.upload_keys(k)
    o = CpuTfhe("orc", "tfhe-80", n_override=6, seed=99)
    o.import_keys(k)
    o.set_exact(True)
    rng = np.random.default_rng(h_lev)
    x = vsp.encrypt(p, k["lv0"], rng.integers(0, 2, 2), 5)
    h = 1 << (64 - (h_lev + 1) * p.Bg1Bits)
    got = e.blind_rotate_lvl2(x, h)
    for i in range(2):
        assert np.array_equal(got[i], o.blind_rotate_lvl2(x[i], h))


@pytest.fixture(scope="module")
def prod_cb():
    p = vsp.ParameterSet("tfhe-80")
    k = vsp.keygen(p, 2020, True)
    e = vsp.Engine(p)
    e.upload_keys(k)
    o = CpuTfhe("orc", "tfhe-80", seed=2020)   # client side only (encrypt/decrypt)
    o.import_keys({**k, "bk2": None, "pks_negs": None, "pks_id": None})
    return e, o, k, p


def test_tfhe80_circuit_bootstrap_selectors(prod_cb):
    e, o, k, p = prod_cb
    rng = np.random.default_rng(9)
    bits = [1, 0, 1, 0]
    sel = e.circuit_bootstrap(vsp.encrypt(p, k["lv0"], bits, 77))
    c1 = np.stack([o.trlwe_encrypt(rng.integers(0, 2, p.N1), 3.73e-9) for _ in bits])
    c0 = np.stack([o.trlwe_encrypt(rng.integers(0, 2, p.N1), 3.73e-9) for _ in bits])
    out = e.cmux(sel, c1, c0)
    for i, b in enumerate(bits):
        want = c1[i] if b else c0[i]
        for kk in range(0, p.N1, 97):
            assert o.trlwe_decrypt_at(out[i], kk) == o.trlwe_decrypt_at(want, kk)


def test_tfhe80_ram_and_rom_functional(prod_cb):
    e, o, k, p = prod_cb
    rng = np.random.default_rng(10)
    v, w = 3, 2
    model = [int(x) for x in rng.integers(0, 4, 8)]
    ram = o.encrypt_ram(words_to_image(model, v, w), v, w)
    for A, wf, X in [(3, 1, 2), (3, 0, 1), (6, 1, 3)]:
        ro, ram = e.ram_cycle(ram, v, w, enc_word(o, A, v), o.encrypt(wf), enc_word(o, X, w))
        assert dec_word(o, ro) == model[A]
        if wf:
            model[A] = X
    assert np.array_equal(o.decrypt_ram(ram, v, w), words_to_image(model, v, w))
    img = rng.integers(0, 256, 512).astype(np.uint8)
    luts = o.encrypt_rom(img)
    for blk in (0, 45, 127):
        got = e.rom_read(luts, 512, enc_word(o, blk, 7))
        assert dec_word(o, got) == int.from_bytes(bytes(img[4 * blk:4 * blk + 4]), "little")


def test_mem_ports_dev_equals_separate_calls_and_oracle(det):
    """vsp_mem_ports_dev (ROM read + RAM cycle with one batched address bootstrap, RAM in
    HBM) == the oracle's romRead and ramCycle, bit for bit, and the device-resident RAM
    evolves like the host-API RAM over consecutive accesses."""
    import torch
    e, o = det
    rng = np.random.default_rng(8)
    v, w = 3, 4
    words = [int(x) for x in rng.integers(0, 1 << w, 1 << v)]
    ram = o.encrypt_ram(words_to_image(words, v, w), v, w)
    img = rng.integers(0, 256, 512).astype(np.uint8)
    luts = o.encrypt_rom(img)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).cuda()
    d_ram, d_luts = t(ram), t(luts)
    n1 = o.n + 1
    ram_o = ram
    for A, wf, X, blk in [(5, 1, 9, 77), (2, 0, 3, 0), (5, 1, 1, 127)]:
        addr, f, d, raddr = enc_word(o, A, v), o.encrypt(wf), enc_word(o, X, w), enc_word(o, blk, 7)
        d_ro = torch.empty((w, n1), dtype=torch.int32, device="cuda")
        d_rout = torch.empty((32, n1), dtype=torch.int32, device="cuda")
        keep = [t(raddr), t(addr), t(f), t(d)]  # live until the asynchronous call is done
        e.mem_ports_dev(d_luts.data_ptr(), luts.shape[0], 512, keep[0].data_ptr(), 7,
                        d_rout.data_ptr(), d_ram.data_ptr(), v, w, keep[1].data_ptr(),
                        keep[2].data_ptr(), keep[3].data_ptr(), d_ro.data_ptr())
        torch.cuda.synchronize()
        rom_o = o.rom_read(luts, 512, raddr)
        ro_o, ram_o = o.ram_cycle(ram_o, v, w, addr, f, d)
        assert np.array_equal(d_rout.cpu().numpy().view(np.uint32), rom_o)
        assert np.array_equal(d_ro.cpu().numpy().view(np.uint32), ro_o)
        assert np.array_equal(d_ram.cpu().numpy().view(np.uint32), ram_o)
        assert dec_word(o, ro_o) == words[A]
        if wf:
            words[A] = X


def test_mem_ports_host_call_equals_oracle_and_updates_ram_in_place(det):
    """vsp_mem_ports (host buffers: the drop-in form of one memory stage) == the oracle's
    romRead and ramCycle bit for bit over consecutive accesses; a C-contiguous uint32 RAM
    image is updated in place (EncryptedRam&), any other input is copied and returned."""
    e, o = det
    rng = np.random.default_rng(18)
    v, w = 3, 4
    words = [int(x) for x in rng.integers(0, 1 << w, 1 << v)]
    ram = np.ascontiguousarray(o.encrypt_ram(words_to_image(words, v, w), v, w), np.uint32)
    luts = o.encrypt_rom(rng.integers(0, 256, 512).astype(np.uint8))
    ram_o = ram.copy()
    for A, wf, X, blk in [(6, 1, 5, 33), (6, 0, 2, 100), (1, 1, 15, 127)]:
        addr, f, d, raddr = enc_word(o, A, v), o.encrypt(wf), enc_word(o, X, w), enc_word(o, blk, 7)
        rom, ro, out = e.mem_ports(luts, 512, raddr, ram, v, w, addr, f, d)
        assert out is ram  # in place
        rom_o = o.rom_read(luts, 512, raddr)
        ro_o, ram_o = o.ram_cycle(ram_o, v, w, addr, f, d)
        assert np.array_equal(rom, rom_o) and np.array_equal(ro, ro_o)
        assert np.array_equal(ram, ram_o)
        assert dec_word(o, ro_o) == words[A]
        if wf:
            words[A] = X
    as_list = ram.astype(np.int64)  # not uint32: copied, the caller's array untouched
    _, _, out = e.mem_ports(luts, 512, enc_word(o, 0, 7), as_list, v, w, enc_word(o, 0, v),
                            o.encrypt(1), enc_word(o, 0, w))
    assert out is not as_list and np.array_equal(as_list, ram.astype(np.int64))


def test_tfhe80_full_size_ram_cycles(prod_cb):
    """BASELINE configs[1] geometry (v=8, w=16: 4,096 cells) on the FFT path, where the
    write unit key-switches the whole-wave cells under the remainder blind-rotation wave:
    two cycles against the plain model, every cell of the decrypted image checked."""
    e, o, k, p = prod_cb
    rng = np.random.default_rng(12)
    v, w = 8, 16
    model = [int(x) for x in rng.integers(0, 1 << w, 1 << v)]
    ram = o.encrypt_ram(words_to_image(model, v, w), v, w)
    for A, wf, X in [(200, 1, 0xBEEF), (200, 0, 0x1234), (17, 1, 0x0F0F)]:
        ro, ram = e.ram_cycle(ram, v, w, enc_word(o, A, v), o.encrypt(wf), enc_word(o, X, w))
        assert dec_word(o, ro) == model[A]
        if wf:
            model[A] = X
    assert np.array_equal(o.decrypt_ram(ram, v, w), words_to_image(model, v, w))
