"""B200-native engine for the VSP (arXiv 2010.09410) TFHE hot path.

Python host mirror of the reference's gate-evaluation API (hvp::tfhe, ops.hpp:149-221)
over the C ABI in include/vsp_b200.h (libvsp_b200.so, built in-tree by
``python -m paper_2010_09410_b200.build``).  The CUDA library is mandatory: there is
no CPU fallback; importing the engine without the built .so raises.

Error behaviour mirrors the reference's exception types:
std::invalid_argument -> ValueError, std::out_of_range -> IndexError,
std::runtime_error -> RuntimeError.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libvsp_b200.so")

# hvp::tfhe::GateKind order (ops.hpp:183-194)
GATE_KINDS = ["AND", "ANDNOT", "MUX", "NAND", "NOR", "NOT", "OR", "ORNOT", "XNOR", "XOR"]
GATE_ARITY = {k: (1 if k == "NOT" else 3 if k == "MUX" else 2) for k in GATE_KINDS}
_KIND_ID = {k: i for i, k in enumerate(GATE_KINDS)}
MU32 = 1 << 29

_lib = None
_XCHG_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                            ctypes.c_void_p)


class VspParams(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint32) for f in
                ("n", "N1", "l1", "Bg1Bits", "N2", "l2", "Bg2Bits", "ksBaseBits", "ksLen",
                 "pksBaseBits", "pksLen")] + [("fft", ctypes.c_int32)]


def lib() -> ctypes.CDLL:
    """Load libvsp_b200.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2010_09410_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        vp, sz, u32, u64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_uint64
        L.vsp_last_error.restype = ctypes.c_char_p
        L.vsp_client_last_error.restype = ctypes.c_char_p
        L.vsp_params_by_name.argtypes = [ctypes.c_char_p, u32, ctypes.POINTER(VspParams)]
        L.vsp_create.restype = vp
        L.vsp_create.argtypes = [ctypes.POINTER(VspParams), ctypes.c_int]
        L.vsp_destroy.argtypes = [vp]
        L.vsp_upload_keys.argtypes = [vp, vp, vp, vp, vp, vp, ctypes.c_int]
        L.vsp_hom_gate_batch.argtypes = [vp, vp, vp, vp, sz]
        L.vsp_hom_gate_batch_dev.argtypes = [vp, vp, vp, vp, sz, vp]
        L.vsp_ram_cycle_dev.argtypes = [vp, u32, u32, vp, vp, vp, vp, vp, vp]
        L.vsp_rom_read_dev.argtypes = [vp, u32, vp, u32, vp, u32, vp, vp]
        L.vsp_mem_ports.argtypes = [vp, u32, vp, u32, vp, u32, vp, u32, u32, vp, vp, vp, vp, vp]
        L.vsp_mem_ports_dev.argtypes = [vp, u32, vp, u32, vp, u32, vp, u32, u32, vp, vp, vp, vp,
                                        vp, vp]
        L.vsp_bootstrap_to_trlwe_batch.argtypes = [vp, vp, vp, sz]
        L.vsp_gate_bootstrap_batch.argtypes = [vp, vp, vp, sz]
        L.vsp_identity_key_switch_batch.argtypes = [vp, vp, vp, sz]
        L.vsp_circuit_bootstrap_batch.argtypes = [vp, vp, vp, sz]
        L.vsp_cmux_batch.argtypes = [vp, vp, vp, vp, vp, sz]
        L.vsp_hom_mux_no_se_iks_batch.argtypes = [vp, vp, vp, vp, vp, sz]
        L.vsp_ram_cycle.argtypes = [vp, u32, u32, vp, vp, vp, vp, vp]
        L.vsp_rom_read.argtypes = [vp, u32, vp, u32, vp, u32, vp]
        L.vsp_blind_rotate_lvl2_batch.argtypes = [vp, vp, vp, vp, sz]
        L.vsp_ram_read_unit.argtypes = [vp, u32, u32, vp, vp, vp]
        L.vsp_ram_control_unit.argtypes = [vp, u32, vp, vp, vp, vp, vp]
        L.vsp_ram_write_unit.argtypes = [vp, u32, u32, vp, vp, vp]
        L.vsp_rom_read_sel.argtypes = [vp, u32, vp, u32, vp, u32, vp]
        L.vsp_counters.argtypes = [vp, vp]
        L.vsp_counters_reset.argtypes = [vp]
        L.vsp_kernel_launches.argtypes = [vp]
        L.vsp_kernel_launches.restype = u64
        L.vsp_synchronize.argtypes = [vp]
        L.vsp_profile_enable.argtypes = [vp, ctypes.c_int]
        L.vsp_profile_read.argtypes = [vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(ctypes.c_uint64)]
        L.vsp_profile_reset.argtypes = [vp]
        L.vsp_br_plan.argtypes = [vp, sz, vp]
        L.vsp_sm_count.argtypes = [vp]
        L.vsp_set_option.argtypes = [vp, ctypes.c_char_p, ctypes.c_int64]
        L.vsp_get_option.argtypes = [vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64)]
        L.vsp_fp64_peak_probe.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
        L.vsp_client_keygen.argtypes = [ctypes.POINTER(VspParams), u64, ctypes.c_int] + [vp] * 8
        L.vsp_client_keygen_dev.argtypes = [ctypes.POINTER(VspParams), u64, ctypes.c_int,
                                            ctypes.c_int] + [vp] * 8
        L.vsp_client_tlwe_encrypt.argtypes = [ctypes.POINTER(VspParams), vp, u64, vp, sz, vp]
        L.vsp_client_tlwe_decrypt.argtypes = [vp, u32, vp, sz, vp, vp]
        L.vsp_client_trlwe_encrypt.argtypes = [ctypes.POINTER(VspParams), vp, u64, vp, sz, vp]
        L.vsp_client_trlwe_phase_at.argtypes = [vp, u32, vp, sz, u32, vp]
        L.vsp_nccl_unique_id.argtypes = [vp]
        L.vsp_attach_comm.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int]
        L.vsp_level_partition.argtypes = [sz, ctypes.c_int, ctypes.c_int,
                                          ctypes.POINTER(sz), ctypes.POINTER(sz),
                                          ctypes.POINTER(sz)]
        L.vsp_hom_gate_level_dev.argtypes = [vp, vp, vp, vp, sz, vp]
        L.vsp_level_partition_kinds.argtypes = [vp, sz, ctypes.c_int, ctypes.c_int,
                                                ctypes.POINTER(sz), ctypes.POINTER(sz),
                                                ctypes.POINTER(sz)]
        L.vsp_attach_exchange.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, vp]
        L.vsp_upload_keys_hvp1.argtypes = [vp, vp, sz]
        L.vsp_read_hvp1.argtypes = [vp, vp, sz, vp, sz, ctypes.POINTER(sz), vp]
        _lib = L
    return _lib


def _raise(rc: int, msg: bytes | None):
    text = (msg or b"").decode()
    if rc == 1:
        raise ValueError(text)
    if rc == 2:
        raise IndexError(text)
    raise RuntimeError(text)


def _check(rc: int):
    if rc != 0:
        _raise(rc, lib().vsp_last_error())


def _ccheck(rc: int):
    if rc != 0:
        _raise(rc, lib().vsp_client_last_error())


def _ptr(a: np.ndarray | None) -> ctypes.c_void_p:
    if a is None:
        return ctypes.c_void_p(0)
    assert a.flags["C_CONTIGUOUS"], "arrays passed to the engine must be C-contiguous"
    return ctypes.c_void_p(a.ctypes.data)


class ParameterSet:
    """hvp::tfhe::ParameterSet (params.hpp:23-66); ``byName`` (params.cpp:88-95)."""

    def __init__(self, name: str = "tfhe-80", n_override: int = 0):
        self.c = VspParams()
        _check(lib().vsp_params_by_name(name.encode(), n_override, ctypes.byref(self.c)))
        self.name = name
        for f, _ in VspParams._fields_:
            setattr(self, f, int(getattr(self.c, f)))

    @property
    def deterministic(self) -> bool:
        return not self.fft

    def ksk_words(self) -> int:
        return self.N1 * self.ksLen * ((1 << self.ksBaseBits) - 1) * (self.n + 1)

    def pks_words(self) -> int:
        return (self.N2 + 1) * self.pksLen * ((1 << self.pksBaseBits) - 1) * 2 * self.N1


# ---------------------------------------------------------------------------
# client side (Alice)

def keygen(params: ParameterSet, seed: int, with_cb: bool | int = False,
           device: int | None = None) -> dict:
    """genSecretKey + BootstrappingKey::generate (ops.cpp:264-385), raw arrays.
    with_cb=2 draws bk2 but not the private key-switching tables (unit tests).
    device: run the b = a*s products on that CUDA device (vsp_client_keygen_dev; the same
    keys bit for bit), else on host threads."""
    p = params
    full_cb = int(with_cb) == 1
    k = dict(
        lv0=np.zeros(p.n, np.uint32), lv1=np.zeros(p.N1, np.uint32),
        lv2=np.zeros(p.N2, np.uint32),
        bk1=np.zeros((p.n, 2 * p.l1, 2, p.N1), np.uint32),
        ksk=np.zeros(p.ksk_words(), np.uint32),
        bk2=np.zeros((p.n, 2 * p.l2, 2, p.N2), np.uint64) if with_cb else None,
        pks_negs=np.zeros(p.pks_words(), np.uint32) if full_cb else None,
        pks_id=np.zeros(p.pks_words(), np.uint32) if full_cb else None,
    )
    outs = [_ptr(k[x]) for x in ("lv0", "lv1", "lv2", "bk1", "ksk", "bk2", "pks_negs", "pks_id")]
    if device is not None:
        _check(lib().vsp_client_keygen_dev(ctypes.byref(p.c), seed, int(with_cb), int(device),
                                           *outs))
    else:
        _ccheck(lib().vsp_client_keygen(ctypes.byref(p.c), seed, int(with_cb), *outs))
    return k


def encrypt(params: ParameterSet, lv0: np.ndarray, bits, seed: int) -> np.ndarray:
    """tlweEncrypt (ops.cpp:428-440) of each bit; returns (len, n+1) u32."""
    b = np.ascontiguousarray(np.asarray(bits, np.uint8).reshape(-1))
    out = np.zeros((b.size, params.n + 1), np.uint32)
    _ccheck(lib().vsp_client_tlwe_encrypt(ctypes.byref(params.c), _ptr(lv0), seed, _ptr(b),
                                          b.size, _ptr(out)))
    return out


def decrypt(key: np.ndarray, ct: np.ndarray) -> np.ndarray:
    """tlweDecrypt (ops.cpp:452-456); ct (..., dim+1) with dim = len(key)."""
    ct = np.ascontiguousarray(ct, np.uint32)
    flat = ct.reshape(-1, ct.shape[-1])
    bits = np.zeros(flat.shape[0], np.uint8)
    _ccheck(lib().vsp_client_tlwe_decrypt(_ptr(np.ascontiguousarray(key, np.uint32)),
                                          len(key), _ptr(flat), flat.shape[0], _ptr(bits), None))
    return bits.reshape(ct.shape[:-1])


def phase(key: np.ndarray, ct: np.ndarray) -> np.ndarray:
    ct = np.ascontiguousarray(ct, np.uint32)
    flat = ct.reshape(-1, ct.shape[-1])
    ph = np.zeros(flat.shape[0], np.uint32)
    _ccheck(lib().vsp_client_tlwe_decrypt(_ptr(np.ascontiguousarray(key, np.uint32)),
                                          len(key), _ptr(flat), flat.shape[0], None, _ptr(ph)))
    return ph.reshape(ct.shape[:-1])


def trlwe_encrypt(params: ParameterSet, lv1: np.ndarray, bit_polys, seed: int) -> np.ndarray:
    """trlweEncrypt (ops.cpp:458-468) of (count, N1) bits -> (count, 2*N1)."""
    b = np.ascontiguousarray(np.asarray(bit_polys, np.uint8).reshape(-1, params.N1))
    out = np.zeros((b.shape[0], 2 * params.N1), np.uint32)
    _ccheck(lib().vsp_client_trlwe_encrypt(ctypes.byref(params.c), _ptr(lv1), seed, _ptr(b),
                                           b.shape[0], _ptr(out)))
    return out


def trlwe_phase_at(lv1: np.ndarray, ct: np.ndarray, k: int = 0) -> np.ndarray:
    """trlwePhaseAt (ops.cpp:494-505) of coefficient k for (count, 2N) TRLWEs (u32)."""
    ct = np.ascontiguousarray(np.atleast_2d(ct), np.uint32)
    N = ct.shape[1] // 2
    ph = np.zeros(ct.shape[0], np.uint32)
    _ccheck(lib().vsp_client_trlwe_phase_at(_ptr(np.ascontiguousarray(lv1, np.uint32)), N,
                                            _ptr(ct), ct.shape[0], k, _ptr(ph)))
    return ph


def trlwe_decrypt_at(lv1: np.ndarray, ct: np.ndarray, k: int = 0) -> np.ndarray:
    """trlweDecryptAt (ops.cpp:507-510) for (count, 2N) TRLWEs."""
    ct = np.ascontiguousarray(np.atleast_2d(ct), np.uint32)
    N = ct.shape[1] // 2
    ph = np.zeros(ct.shape[0], np.uint32)
    _ccheck(lib().vsp_client_trlwe_phase_at(_ptr(np.ascontiguousarray(lv1, np.uint32)), N,
                                            _ptr(ct), ct.shape[0], k, _ptr(ph)))
    return (ph.view(np.int32) >= 0).astype(np.uint8)


def encrypt_ram(params: ParameterSet, keys: dict, image: np.ndarray, v: int, w: int,
                seed: int) -> np.ndarray:
    """encryptRam (mem.cpp:202-222): cell j*2^v + A carries bit A*w + j at coefficient 0."""
    image = np.asarray(image, np.uint8)
    if image.size != (w << v) // 8:
        raise ValueError("encryptRam: image size mismatch")
    bits = np.unpackbits(image, bitorder="little")
    polys = np.zeros(((w << v), params.N1), np.uint8)
    for j in range(w):
        polys[j << v:(j + 1) << v, 0] = bits[np.arange(1 << v) * w + j]
    return trlwe_encrypt(params, keys["lv1"], polys, seed)


def decrypt_ram(keys: dict, ram: np.ndarray, v: int, w: int) -> np.ndarray:
    """decryptRam (mem.cpp:224-234)."""
    dec = trlwe_decrypt_at(keys["lv1"], ram, 0)
    bits = np.zeros(w << v, np.uint8)
    for j in range(w):
        bits[np.arange(1 << v) * w + j] = dec[j << v:(j + 1) << v]
    return np.packbits(bits, bitorder="little")


def encrypt_rom(params: ParameterSet, keys: dict, image: np.ndarray, seed: int) -> np.ndarray:
    """encryptRom (mem.cpp:236-263): LUT t coefficient c carries ROM bit t*N1 + c."""
    image = np.asarray(image, np.uint8)
    blocks = image.size // 4
    if image.size == 0 or image.size % 4 or blocks & (blocks - 1):
        raise ValueError("encryptRom: image must hold a power-of-two number of 32-bit blocks")
    vrom = blocks.bit_length() - 1
    low = min(vrom, (params.N1 // 32).bit_length() - 1)
    nluts = 1 << (vrom - low)
    bits = np.unpackbits(image, bitorder="little")
    polys = np.zeros((nluts, params.N1), np.uint8)
    flat = polys.reshape(-1)
    flat[:min(bits.size, flat.size)] = bits[:flat.size]
    return trlwe_encrypt(params, keys["lv1"], polys, seed)


# ---------------------------------------------------------------------------
# evaluation engine (Bob)

class Engine:
    """One device context holding an uploaded BootstrappingKey.

    Method names follow the reference (ops.hpp:149-221) in snake case; every method
    accepts a batch (leading axis) and is equivalent to calling the reference
    function once per element.
    """

    def __init__(self, params: ParameterSet | str = "tfhe-80", device: int = 0,
                 n_override: int = 0):
        self.params = params if isinstance(params, ParameterSet) else \
            ParameterSet(params, n_override)
        L = lib()
        self.h = L.vsp_create(ctypes.byref(self.params.c), device)
        if not self.h:
            _raise(3, L.vsp_last_error())
        self.h = ctypes.c_void_p(self.h)
        self.device = device
        self.sms = int(lib().vsp_sm_count(self.h))

    def close(self):
        if getattr(self, "h", None):
            lib().vsp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # BootstrappingKey::fromParts (ops.cpp:387-402)
    def upload_keys(self, k: dict):
        has_cb = 0 if k.get("bk2") is None else (1 if k.get("pks_id") is not None else 2)
        c = lambda a: None if a is None else np.ascontiguousarray(a)
        self._keys = {key: c(v) for key, v in k.items()}
        kk = self._keys
        _check(lib().vsp_upload_keys(self.h, _ptr(kk["bk1"]), _ptr(kk["ksk"]),
                                     _ptr(kk.get("bk2")), _ptr(kk.get("pks_negs")),
                                     _ptr(kk.get("pks_id")), int(has_cb)))
        self._keys = None

    def upload_keys_hvp1(self, data: bytes):
        """deserializeBootstrappingKey (serialize.cpp:209-230): load the reference's HVP1
        key file straight into the device."""
        buf = np.frombuffer(bytes(data), np.uint8).copy()
        _check(lib().vsp_upload_keys_hvp1(self.h, _ptr(buf), buf.size))

    def read_hvp1(self, data: bytes):
        """HVP1 TLWE / TRLWE / RAM / ROM container -> (meta, flat array) in engine layout:
        TLWE (n+1,), TRLWE (2N,), RAM (w*2^v, 2N) with meta v, w, ROM (luts, 2N)."""
        buf = np.frombuffer(bytes(data), np.uint8).copy()
        meta = np.zeros(5, np.uint32)
        words = ctypes.c_size_t()
        _check(lib().vsp_read_hvp1(self.h, _ptr(buf), buf.size, None, 0, ctypes.byref(words),
                                   _ptr(meta)))
        out = np.zeros(words.value, np.uint32)
        _check(lib().vsp_read_hvp1(self.h, _ptr(buf), buf.size, _ptr(out), out.size,
                                   ctypes.byref(words), _ptr(meta)))
        tag, count, v, w, depth = (int(x) for x in meta)
        m = {"tag": tag, "count": count, "v": v, "w": w, "depth_bytes": depth}
        return m, (out.reshape(count, -1) if tag in (6, 7) else out)

    @staticmethod
    def _kind_ids(kinds) -> np.ndarray:
        """Gate kinds as GateKind ids (ops.hpp:183-194): names, ints, or an int array (fast
        path, no per-element Python work).  Out-of-range ids are rejected by the C ABI."""
        if isinstance(kinds, np.ndarray) and kinds.dtype.kind in "iu":
            return np.ascontiguousarray(kinds, np.int32)
        out = []
        for k in kinds:
            if isinstance(k, str):
                if k not in _KIND_ID:
                    raise ValueError(f"homGate: unknown kind {k}")
                out.append(_KIND_ID[k])
            else:
                out.append(int(k))
        return np.ascontiguousarray(np.asarray(out, np.int32))

    def hom_gate(self, kind, inputs) -> np.ndarray:
        """homGate (ops.cpp:839-896) for one gate; inputs: list of TLWEs."""
        name = kind if isinstance(kind, str) else GATE_KINDS[int(kind)]
        if len(inputs) != GATE_ARITY.get(name, -1):
            raise ValueError(f"homGate: bad arity for {name}")
        x = np.zeros((1, 3, self.params.n + 1), np.uint32)
        for i, t in enumerate(inputs):
            x[0, i] = t
        return self.hom_gate_batch([name], x)[0]

    def hom_gate_batch(self, kinds, ins: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        """Batched homGate: kinds[G], ins (G, 3, n+1) -> (G, n+1).  `out` may be a
        caller-owned (e.g. pinned) (G, n+1) uint32 array to write into."""
        kid = self._kind_ids(kinds)
        ins = np.ascontiguousarray(ins, np.uint32)
        G = kid.size
        if ins.shape != (G, 3, self.params.n + 1):
            raise ValueError(f"expected inputs of shape {(G, 3, self.params.n + 1)}")
        if out is None:
            out = np.empty((G, self.params.n + 1), np.uint32)
        elif out.shape != (G, self.params.n + 1) or out.dtype != np.uint32 or \
                not out.flags["C_CONTIGUOUS"]:
            raise ValueError(f"out must be a C-contiguous uint32 array of shape {(G, self.params.n + 1)}")
        _check(lib().vsp_hom_gate_batch(self.h, _ptr(kid), _ptr(ins), _ptr(out), G))
        return out

    def hom_gate_batch_dev(self, kinds, d_in_ptr: int, d_out_ptr: int, G: int,
                           stream_ptr: int = 0):
        """Device-resident variant (pointers from torch tensors); asynchronous."""
        kid = self._kind_ids(kinds)
        if kid.size != G:
            raise ValueError(f"homGate: {kid.size} kinds for {G} gates")
        _check(lib().vsp_hom_gate_batch_dev(self.h, _ptr(kid), ctypes.c_void_p(d_in_ptr),
                                            ctypes.c_void_p(d_out_ptr), G,
                                            ctypes.c_void_p(stream_ptr)))

    def bootstrap_to_trlwe(self, cts: np.ndarray) -> np.ndarray:
        """bootstrapToTrlwe (ops.cpp:750-757); (G, n+1) -> (G, 2*N1)."""
        cts = np.ascontiguousarray(np.atleast_2d(cts), np.uint32)
        out = np.zeros((cts.shape[0], 2 * self.params.N1), np.uint32)
        _check(lib().vsp_bootstrap_to_trlwe_batch(self.h, _ptr(cts), _ptr(out), cts.shape[0]))
        return out

    def gate_bootstrap(self, cts: np.ndarray) -> np.ndarray:
        """gateBootstrap (ops.cpp:759-762); (G, n+1) -> (G, n+1)."""
        cts = np.ascontiguousarray(np.atleast_2d(cts), np.uint32)
        out = np.zeros_like(cts)
        _check(lib().vsp_gate_bootstrap_batch(self.h, _ptr(cts), _ptr(out), cts.shape[0]))
        return out

    def identity_key_switch(self, cts: np.ndarray) -> np.ndarray:
        """identityKeySwitch (ops.cpp:651-679); (G, N1+1) -> (G, n+1)."""
        cts = np.ascontiguousarray(np.atleast_2d(cts), np.uint32)
        out = np.zeros((cts.shape[0], self.params.n + 1), np.uint32)
        _check(lib().vsp_identity_key_switch_batch(self.h, _ptr(cts), _ptr(out), cts.shape[0]))
        return out

    # ---- circuit bootstrapping / CMUX memory -------------------------------
    def circuit_bootstrap(self, cts: np.ndarray) -> np.ndarray:
        """circuitBootstrap (ops.cpp:914-935); (C, n+1) -> (C, 2*l1, 2, N1)."""
        p = self.params
        cts = np.ascontiguousarray(np.atleast_2d(cts), np.uint32)
        out = np.zeros((cts.shape[0], 2 * p.l1, 2, p.N1), np.uint32)
        _check(lib().vsp_circuit_bootstrap_batch(self.h, _ptr(cts), _ptr(out), cts.shape[0]))
        return out

    def cmux(self, sel: np.ndarray, c1: np.ndarray, c0: np.ndarray) -> np.ndarray:
        """cmux (ops.cpp:606-626) batch: sel (G, 2l, 2, N1), c1/c0 (G, 2*N1)."""
        p = self.params
        sel = np.ascontiguousarray(sel.reshape(-1, 2 * p.l1, 2, p.N1), np.uint32)
        c1 = np.ascontiguousarray(c1.reshape(-1, 2 * p.N1), np.uint32)
        c0 = np.ascontiguousarray(c0.reshape(-1, 2 * p.N1), np.uint32)
        if not (sel.shape[0] == c1.shape[0] == c0.shape[0]):
            raise ValueError("cmux: selector / operand counts differ")
        out = np.zeros_like(c1)
        _check(lib().vsp_cmux_batch(self.h, _ptr(sel), _ptr(c1), _ptr(c0), _ptr(out), c1.shape[0]))
        return out

    def hom_mux_no_se_iks(self, sel, a, b) -> np.ndarray:
        """homMuxNoSeIks (ops.cpp:898-909) batch: (G, n+1) x3 -> (G, 2*N1)."""
        p = self.params
        f = lambda x: np.ascontiguousarray(np.atleast_2d(x), np.uint32)
        sel, a, b = f(sel), f(a), f(b)
        if not (sel.shape == a.shape == b.shape) or sel.shape[1] != p.n + 1:
            raise ValueError(f"homMuxNoSeIks: operands must all be (G, {p.n + 1})")
        out = np.zeros((sel.shape[0], 2 * p.N1), np.uint32)
        _check(lib().vsp_hom_mux_no_se_iks_batch(self.h, _ptr(sel), _ptr(a), _ptr(b), _ptr(out),
                                                 sel.shape[0]))
        return out

    def ram_cycle(self, ram: np.ndarray, v: int, w: int, addr, wflag, wdata):
        """mem::ramCycle (mem.cpp:122-135).  Returns (readOut (w, n+1), new ram)."""
        p = self.params
        if len(addr) != v:
            raise ValueError("ramCycle: address width mismatch")
        ram = np.ascontiguousarray(np.array(ram, np.uint32).reshape((w << v), 2 * p.N1))
        a = np.ascontiguousarray(addr, np.uint32)
        f = np.ascontiguousarray(wflag, np.uint32)
        d = np.ascontiguousarray(wdata, np.uint32)
        if a.shape != (v, p.n + 1) or f.size != p.n + 1 or d.shape != (w, p.n + 1):
            raise ValueError("ramCycle: address width mismatch")
        ro = np.zeros((w, p.n + 1), np.uint32)
        _check(lib().vsp_ram_cycle(self.h, v, w, _ptr(ram), _ptr(a), _ptr(f), _ptr(d), _ptr(ro)))
        return ro, ram

    def rom_read(self, luts: np.ndarray, depth_bytes: int, addr) -> np.ndarray:
        """addressToTrgsw + romRead (engine.cpp:133-143): 32 TLWEs."""
        p = self.params
        luts = np.ascontiguousarray(luts, np.uint32)
        a = np.ascontiguousarray(np.atleast_2d(addr), np.uint32)
        if a.shape[1] != p.n + 1 or luts.ndim != 2 or luts.shape[1] != 2 * p.N1:
            raise ValueError("romRead: address / LUT shape mismatch")
        out = np.zeros((32, p.n + 1), np.uint32)
        _check(lib().vsp_rom_read(self.h, depth_bytes, _ptr(luts), luts.shape[0], _ptr(a),
                                  a.shape[0], _ptr(out)))
        return out

    # ---- the units of ramCycle / romRead on given selectors (mem.hpp:75-124) ----------
    def _sel(self, sel) -> np.ndarray:
        p = self.params
        return np.ascontiguousarray(np.asarray(sel, np.uint32).reshape(-1, 2 * p.l1, 2, p.N1))

    def ram_read_unit(self, ram: np.ndarray, v: int, w: int, sel) -> np.ndarray:
        """mem::ramReadUnit (mem.cpp:49-72): sel = v raw TRGSWs (RamAddress, LSB first);
        returns w TRLWEs (bit j of the addressed word at coefficient 0 of output j)."""
        p = self.params
        sel = self._sel(sel)
        ram = np.ascontiguousarray(np.asarray(ram, np.uint32).reshape((w << v), 2 * p.N1))
        if sel.shape[0] != v:
            raise ValueError("ramReadUnit: address width mismatch")
        out = np.zeros((w, 2 * p.N1), np.uint32)
        _check(lib().vsp_ram_read_unit(self.h, v, w, _ptr(ram), _ptr(sel), _ptr(out)))
        return out

    def ram_control_unit(self, read: np.ndarray, wflag, wdata):
        """mem::ramControlUnit (mem.cpp:74-90): returns (readOut (w, n+1),
        controlled (w, 2*N1))."""
        p = self.params
        read = np.ascontiguousarray(np.asarray(read, np.uint32).reshape(-1, 2 * p.N1))
        w = read.shape[0]
        f = np.ascontiguousarray(wflag, np.uint32)
        d = np.ascontiguousarray(wdata, np.uint32)
        if f.size != p.n + 1 or d.shape != (w, p.n + 1):
            raise ValueError("ramControlUnit: word width mismatch")
        ro = np.zeros((w, p.n + 1), np.uint32)
        ctl = np.zeros((w, 2 * p.N1), np.uint32)
        _check(lib().vsp_ram_control_unit(self.h, w, _ptr(read), _ptr(f), _ptr(d), _ptr(ro),
                                          _ptr(ctl)))
        return ro, ctl

    def ram_write_unit(self, ram: np.ndarray, v: int, w: int, sel, controlled) -> np.ndarray:
        """mem::ramWriteUnit (mem.cpp:92-120): returns the new RAM image."""
        p = self.params
        sel = self._sel(sel)
        ram = np.array(np.asarray(ram, np.uint32).reshape((w << v), 2 * p.N1), np.uint32)
        ctl = np.ascontiguousarray(np.asarray(controlled, np.uint32).reshape(-1, 2 * p.N1))
        if sel.shape[0] != v or ctl.shape[0] != w:
            raise ValueError("ramWriteUnit: geometry mismatch")
        _check(lib().vsp_ram_write_unit(self.h, v, w, _ptr(ram), _ptr(sel), _ptr(ctl)))
        return ram

    def rom_read_sel(self, luts: np.ndarray, depth_bytes: int, sel) -> np.ndarray:
        """mem::romRead (mem.cpp:137-177) on given selectors (vrom raw TRGSWs)."""
        p = self.params
        sel = self._sel(sel)
        luts = np.ascontiguousarray(luts, np.uint32)
        out = np.zeros((32, p.n + 1), np.uint32)
        _check(lib().vsp_rom_read_sel(self.h, depth_bytes, _ptr(luts), luts.shape[0], _ptr(sel),
                                      sel.shape[0], _ptr(out)))
        return out

    def ram_cycle_dev(self, d_ram: int, v: int, w: int, d_addr: int, d_wflag: int,
                      d_wdata: int, d_readout: int, stream: int = 0):
        """Device-resident ramCycle: d_ram (w<<v, 2*N1) u32 updated in place in HBM,
        d_readout (w, n+1); asynchronous on `stream`."""
        _check(lib().vsp_ram_cycle_dev(self.h, v, w, ctypes.c_void_p(d_ram), ctypes.c_void_p(d_addr),
                                       ctypes.c_void_p(d_wflag), ctypes.c_void_p(d_wdata),
                                       ctypes.c_void_p(d_readout), ctypes.c_void_p(stream)))

    def rom_read_dev(self, d_luts: int, nluts: int, depth_bytes: int, d_addr: int, vrom: int,
                     d_out: int, stream: int = 0):
        """Device-resident addressToTrgsw + romRead: 32 TLWEs into d_out."""
        _check(lib().vsp_rom_read_dev(self.h, depth_bytes, ctypes.c_void_p(d_luts), nluts,
                                      ctypes.c_void_p(d_addr), vrom, ctypes.c_void_p(d_out),
                                      ctypes.c_void_p(stream)))

    def mem_ports(self, luts: np.ndarray, depth_bytes: int, rom_addr, ram: np.ndarray, v: int,
                  w: int, addr, wflag, wdata):
        """One memory stage with host buffers (vsp_mem_ports): romRead + ramCycle with the
        two ports' address bootstraps batched.  Returns (rom_out (32, n+1), readOut (w, n+1),
        ram).  A C-contiguous uint32 `ram` of shape (w << v, 2 N1) is updated IN PLACE (the
        reference's EncryptedRam&; pass a pinned array for link-speed copies), any other is
        copied first and the new image returned."""
        p = self.params
        luts = np.ascontiguousarray(luts, np.uint32)
        ra = np.ascontiguousarray(np.atleast_2d(rom_addr), np.uint32)
        if ra.shape[1] != p.n + 1 or luts.ndim != 2 or luts.shape[1] != 2 * p.N1:
            raise ValueError("romRead: address / LUT shape mismatch")
        shape = ((w << v), 2 * p.N1)
        if not (isinstance(ram, np.ndarray) and ram.dtype == np.uint32 and ram.shape == shape
                and ram.flags.c_contiguous and ram.flags.writeable):
            ram = np.ascontiguousarray(np.array(ram, np.uint32).reshape(shape))
        a = np.ascontiguousarray(addr, np.uint32)
        f = np.ascontiguousarray(wflag, np.uint32)
        d = np.ascontiguousarray(wdata, np.uint32)
        if len(a) != v or a.shape != (v, p.n + 1) or f.size != p.n + 1 or d.shape != (w, p.n + 1):
            raise ValueError("ramCycle: address width mismatch")
        rom_out = np.zeros((32, p.n + 1), np.uint32)
        ro = np.zeros((w, p.n + 1), np.uint32)
        _check(lib().vsp_mem_ports(self.h, depth_bytes, _ptr(luts), luts.shape[0], _ptr(ra),
                                   ra.shape[0], _ptr(rom_out), v, w, _ptr(ram), _ptr(a), _ptr(f),
                                   _ptr(d), _ptr(ro)))
        return rom_out, ro, ram

    def mem_ports_dev(self, d_luts: int, nluts: int, depth_bytes: int, d_rom_addr: int,
                      vrom: int, d_rom_out: int, d_ram: int, v: int, w: int, d_ram_addr: int,
                      d_wflag: int, d_wdata: int, d_readout: int, stream: int = 0):
        """One ROM read + one RAM cycle with batched address bootstraps (device buffers)."""
        c = ctypes.c_void_p
        _check(lib().vsp_mem_ports_dev(self.h, depth_bytes, c(d_luts), nluts, c(d_rom_addr), vrom,
                                       c(d_rom_out), v, w, c(d_ram), c(d_ram_addr), c(d_wflag),
                                       c(d_wdata), c(d_readout), c(stream)))

    def blind_rotate_lvl2(self, cts: np.ndarray, h) -> np.ndarray:
        p = self.params
        cts = np.ascontiguousarray(np.atleast_2d(cts), np.uint32)
        hv = np.ascontiguousarray(np.broadcast_to(np.asarray(h, np.uint64), (cts.shape[0],)))
        out = np.zeros((cts.shape[0], 2 * p.N2), np.uint64)
        _check(lib().vsp_blind_rotate_lvl2_batch(self.h, _ptr(cts), _ptr(hv), _ptr(out),
                                                 cts.shape[0]))
        return out

    def br_plan(self, tasks: int) -> dict:
        """The blind-rotation launch plan for `tasks` tasks: narrow-level latency kernel,
        tasks in whole W=8 waves, tasks per SM of the remainder / single launch and its
        kernel."""
        o = np.zeros(4, np.int32)
        _check(lib().vsp_br_plan(self.h, tasks, _ptr(o)))
        return {"lat": bool(o[0]), "full": int(o[1]), "w_rem": int(o[2]),
                "rem_kernel": ("none", "br1024", "br1024p", "br_lat")[int(o[3])]}

    def set_option(self, name: str, value: int):
        """Engine tuning option (vsp_set_option): "lat_tasks" (1|2), "ram_overlap",
        "iks_gemm", "br_pair", "backfill" (0|1), "iks_split" (split-K factor, 0 = automatic)."""
        _check(lib().vsp_set_option(self.h, name.encode(), int(value)))

    def get_option(self, name: str) -> int:
        """An option's value, or the statistic "bars_backfilled" (vsp_get_option)."""
        v = ctypes.c_int64()
        _check(lib().vsp_get_option(self.h, name.encode(), ctypes.byref(v)))
        return int(v.value)

    def counters(self) -> dict:
        """OpCounters (counters.hpp:11-28)."""
        o = np.zeros(5, np.uint64)
        _check(lib().vsp_counters(self.h, _ptr(o)))
        return dict(zip(["cmux", "blindRotate", "identityKeySwitch", "privateKeySwitch",
                         "circuitBootstrap"], (int(x) for x in o)))

    def counters_reset(self):
        _check(lib().vsp_counters_reset(self.h))

    def kernel_launches(self) -> int:
        return int(lib().vsp_kernel_launches(self.h))

    def synchronize(self):
        _check(lib().vsp_synchronize(self.h))

    def profile_enable(self, on: bool = True):
        _check(lib().vsp_profile_enable(self.h, int(on)))

    def profile_read(self, name: str) -> tuple[float, int]:
        ms, cnt = ctypes.c_double(), ctypes.c_uint64()
        _check(lib().vsp_profile_read(self.h, name.encode(), ctypes.byref(ms), ctypes.byref(cnt)))
        return ms.value, int(cnt.value)

    def profile_reset(self):
        _check(lib().vsp_profile_reset(self.h))

    # ---- multi-GPU --------------------------------------------------
    def attach_comm(self, uid: bytes, rank: int, world: int):
        """Join the NCCL communicator `uid` (from nccl_unique_id on rank 0) as `rank`;
        afterwards netlist levels are sharded across the ranks and all-gathered."""
        buf = np.frombuffer(bytes(uid), np.uint8).copy()
        if buf.size != 128:
            raise ValueError("attach_comm: NCCL unique id must be 128 bytes")
        _check(lib().vsp_attach_comm(self.h, _ptr(buf), int(rank), int(world)))
        self.rank, self.world = int(rank), int(world)

    def attach_exchange(self, rank: int, world: int, allgather):
        """Shard levels / the RAM over `world` ranks with a caller-provided all-gather
        instead of NCCL: allgather(send: bytes) -> list of `world` bytes objects (one per
        rank, in rank order), e.g. torch.distributed.all_gather_object over gloo."""
        def cb(send, recv, nbytes, user):
            try:
                parts = allgather(ctypes.string_at(send, nbytes))
                if len(parts) != world or any(len(x) != nbytes for x in parts):
                    return 1
                ctypes.memmove(recv, b"".join(parts), nbytes * world)
                return 0
            except Exception:  # an exception must not cross the C boundary
                return 1
        self._xchg_cb = _XCHG_FN(cb)  # keep the thunk alive while attached
        _check(lib().vsp_attach_exchange(self.h, int(rank), int(world),
                                         ctypes.cast(self._xchg_cb, ctypes.c_void_p), None))
        self.rank, self.world = int(rank), int(world)

    def connect(self, group=None):
        """attach_comm over an initialised torch.distributed group (any backend): rank 0
        creates the NCCL id, a broadcast distributes it."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        box = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        self.attach_comm(box[0], rank, world)

    def hom_gate_level_dev(self, kinds, d_in_ptr: int, d_out_ptr: int, G: int,
                           stream: int = 0):
        """homGate over one netlist level sharded across the attached ranks (device
        buffers holding ALL G gates on every rank)."""
        kid = self._kind_ids(kinds)
        if kid.size != G:
            raise ValueError(f"homGate: {kid.size} kinds for {G} gates")
        _check(lib().vsp_hom_gate_level_dev(self.h, _ptr(kid), ctypes.c_void_p(d_in_ptr),
                                            ctypes.c_void_p(d_out_ptr), G,
                                            ctypes.c_void_p(stream)))


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the engine (NCCL is dlopen'ed by the library)."""
    buf = np.zeros(128, np.uint8)
    _check(lib().vsp_nccl_unique_id(_ptr(buf)))
    return buf.tobytes()


def level_partition(G: int, world: int, rank: int, kinds=None) -> tuple[int, int, int]:
    """The runner's per-rank slice [lo, hi) of a G-gate level (slices of equal blind-
    rotation task count: MUX 2, NOT 0, others 1; kinds=None: one task per gate) and the
    all-gather's per-rank slot count (the largest slice; multi.cuh level_slice)."""
    lo, hi, per = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
    if kinds is None:
        _check(lib().vsp_level_partition(G, world, rank, ctypes.byref(lo), ctypes.byref(hi),
                                         ctypes.byref(per)))
    else:
        kid = Engine._kind_ids(kinds)
        if kid.size != G:
            raise ValueError(f"level_partition: {kid.size} kinds for {G} gates")
        _check(lib().vsp_level_partition_kinds(_ptr(kid), G, world, rank, ctypes.byref(lo),
                                               ctypes.byref(hi), ctypes.byref(per)))
    return int(lo.value), int(hi.value), int(per.value)


def fp64_peak_tflops(device: int = 0) -> float:
    """Measured DFMA throughput of the device (TFLOP/s)."""
    t = ctypes.c_double()
    _check(lib().vsp_fp64_peak_probe(device, ctypes.byref(t)))
    return t.value
