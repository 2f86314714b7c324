"""HVP1 file ingestion (serialize.cpp, mem.cpp:331-403): keys and ciphertext containers
written by the REFERENCE's serializers load straight into the engine; gates after an
HVP1 key upload are bit-exact with the reference on the same inputs."""
import ctypes

import numpy as np
import pytest

import paper_2010_09410_b200 as vsp
from oracle import pyoracle
from oracle.pyoracle import CpuTfhe, GATE_KINDS, ref_bytes

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not pyoracle.available("ref"), reason="reference not built")]


def _p(a):
    return np.ascontiguousarray(a).ctypes.data_as(ctypes.c_void_p)


@pytest.mark.parametrize("params,cb", [("test-det", True), ("tfhe-80", False)])
def test_hvp1_key_upload_gates_bit_exact(params, cb):
    r = CpuTfhe("ref", params, seed=20200729)
    r.keygen(cb)
    e = vsp.Engine(params)
    e.upload_keys_hvp1(ref_bytes("ref_serialize_bk", r.h))
    rng = np.random.default_rng(3)
    G = 24
    kinds = np.array([i % len(GATE_KINDS) for i in range(G)], np.int32)
    ins = np.zeros((G, 3, r.n + 1), np.uint32)
    for g in range(G):
        for k in range(3):
            ins[g, k] = r.encrypt(int(rng.integers(0, 2)))
    assert np.array_equal(e.hom_gate_batch(kinds, ins), r.hom_gate_batch(kinds, ins, threads=4))


def test_hvp1_ciphertext_containers():
    r = CpuTfhe("ref", "test-det", seed=515253)
    r.keygen(True)
    e = vsp.Engine("test-det")
    e.upload_keys_hvp1(ref_bytes("ref_serialize_bk", r.h))
    ct = r.encrypt(1)
    meta, got = e.read_hvp1(ref_bytes("ref_serialize_tlwe", r.h, _p(ct)))
    assert meta["tag"] == 3 and np.array_equal(got, ct)
    v, w = 3, 4
    ram = r.encrypt_ram(np.arange((w << v) // 8, dtype=np.uint8), v, w)
    meta, got = e.read_hvp1(ref_bytes("ref_serialize_ram", r.h, v, w, _p(ram)))
    assert (meta["tag"], meta["v"], meta["w"], meta["count"]) == (6, v, w, w << v)
    assert np.array_equal(got, ram.reshape(got.shape))
    luts = r.encrypt_rom(np.arange(512, dtype=np.uint8) % 251)
    meta, got = e.read_hvp1(ref_bytes("ref_serialize_rom", r.h, 512, _p(luts), luts.shape[0]))
    assert (meta["tag"], meta["depth_bytes"]) == (7, 512)
    assert np.array_equal(got, luts.reshape(got.shape))


def test_hvp1_rejections():
    r = CpuTfhe("ref", "tfhe-80", seed=1)
    r.keygen(False)
    data = ref_bytes("ref_serialize_bk", r.h)
    e = vsp.Engine("test-det")
    with pytest.raises(RuntimeError, match="does not match parameter set"):
        e.upload_keys_hvp1(data)
    with pytest.raises(RuntimeError, match="bad file magic"):
        e.upload_keys_hvp1(b"HVP2" + data[4:])
    e80 = vsp.Engine("tfhe-80")
    with pytest.raises(RuntimeError, match="truncated"):
        e80.upload_keys_hvp1(data[: len(data) // 3])
    with pytest.raises(RuntimeError, match="unexpected file type tag"):
        e80.read_hvp1(data)
