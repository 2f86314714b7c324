"""Client-side key generation/encryption of the product (libvsp_b200.so, host code)
against the reference (golden key hashes)."""
import hashlib

import pytest

import numpy as np

import paper_2010_09410_b200 as vsp
from tests.helpers import golden


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_client_keygen_matches_reference_testdet():
    g = golden("testdet_seed515253.npz")
    k = vsp.keygen(vsp.ParameterSet("test-det"), 515253, True)
    names = ["lv0", "lv1", "lv2", "bk1", "ksk", "bk2", "pks_negs", "pks_id"]
    assert [sha(k[x]) for x in names] == list(g["key_sha"])


def test_client_keygen_matches_reference_tfhe80():
    g = golden("tfhe80_seed20200729.npz")
    k = vsp.keygen(vsp.ParameterSet("tfhe-80"), 20200729, False)
    assert [sha(k[x]) for x in ["lv0", "lv1", "lv2", "bk1", "ksk"]] == list(g["key_sha"])


def test_client_encrypt_decrypt_roundtrip():
    p = vsp.ParameterSet("tfhe-80")
    k = vsp.keygen(p, 3, False)
    bits = np.random.default_rng(1).integers(0, 2, 1000).astype(np.uint8)
    ct = vsp.encrypt(p, k["lv0"], bits, 99)
    assert np.array_equal(vsp.decrypt(k["lv0"], ct), bits)
    ph = vsp.phase(k["lv0"], ct).astype(np.int64)
    ph = np.where(ph >= 2**31, ph - 2**32, ph)
    assert np.all(np.abs(np.abs(ph) - vsp.MU32) < 2**29 // 8)


def test_client_ram_rom_encryption_layout_matches_reference():
    """encryptRam / encryptRom layouts (mem.cpp:202-263) against the restatement."""
    from oracle.pyoracle import CpuTfhe
    p = vsp.ParameterSet("test-det")
    k = vsp.keygen(p, 3, False)
    o = CpuTfhe("orc", "test-det", seed=3)
    o.keygen(False)
    img = np.random.default_rng(1).integers(0, 256, 64).astype(np.uint8)
    ram = vsp.encrypt_ram(p, k, img, 6, 8, 9)
    assert np.array_equal(vsp.decrypt_ram(k, ram, 6, 8), img)
    assert np.array_equal(o.decrypt_ram(ram, 6, 8), img)
    rimg = np.random.default_rng(2).integers(0, 256, 512).astype(np.uint8)
    rom = vsp.encrypt_rom(p, k, rimg, 3)
    ref = o.encrypt_rom(rimg, trivial=True)
    assert rom.shape == ref.shape
    for t in range(rom.shape[0]):
        for c in range(0, p.N1, 7):
            assert vsp.trlwe_decrypt_at(k["lv1"], rom[t], c)[0] == o.trlwe_decrypt_at(ref[t], c)


@pytest.mark.gpu
def test_client_keygen_on_gpu_equals_host_keygen_with_cb():
    """vsp_client_keygen_dev (b = a*s products of bk1, bk2 and both private key-switching
    tables on the GPU) yields the host keygen's keys bit for bit at n = 630 with
    circuit-bootstrapping material; the host keygen is itself pinned to the reference's
    BootstrappingKey::generate by the golden key hashes above."""
    import time
    from tests.helpers import keys_with_cb
    p = vsp.ParameterSet("tfhe-80", n_override=630)
    host = keys_with_cb(630, 630)
    t0 = time.perf_counter()
    dev = vsp.keygen(p, 630, True, device=0)
    dt = time.perf_counter() - t0
    for name in ["lv0", "lv1", "lv2", "bk1", "ksk", "bk2", "pks_negs", "pks_id"]:
        assert np.array_equal(dev[name], host[name]), name
    print(f"GPU keygen with CB at n=630: {dt:.1f} s")
