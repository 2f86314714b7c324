"""TEST INFRASTRUCTURE ONLY — ctypes front-end for the two CPU checkers.

* ``kind="orc"``: oracle/_build/liboracle.so, the plain-C restatement (hvp_oracle.c).
* ``kind="ref"``: oracle/_ref/libhvpref.so, the reference itself compiled from
  /root/reference/proj/src by oracle/Makefile (ref_shim.cpp wraps its public API).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs import this module.  The product (paper_2010_09410_b200) never does.
Both libraries share one C API (prefix ``orc_`` / ``ref_``) and flat layouts:
TLWE = (dim+1) u32, TRLWE = 2N u32, TRGSW = 2l x TRLWE.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATHS = {
    "orc": os.path.join(HERE, "_build", "liboracle.so"),
    "ref": os.path.join(HERE, "_ref", "libhvpref.so"),
}


def _stock_level() -> str:
    """ISA level of the reference's stock (-march=native) build for THIS host: x86-64-v4
    when the CPU has AVX-512, else v3 (oracle/Makefile ref-stock)."""
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        flags = ""
    return "v4" if " avx512f" in flags and " avx512vl" in flags else "v3"


# "ref_stock": the reference built like its own CMake Release (-O3 -DNDEBUG, native ISA):
# timing only, never a checker (its FP contraction differs from the parity build).
LIB_PATHS["ref_stock"] = os.path.join(HERE, "_ref", f"stock_{_stock_level()}", "libhvpref.so")


def _prefix(kind: str) -> str:
    return "orc" if kind == "orc" else "ref"

GATE_KINDS = ["AND", "ANDNOT", "MUX", "NAND", "NOR", "NOT", "OR", "ORNOT", "XNOR", "XOR"]
MU32 = 1 << 29

_libs: dict[str, ctypes.CDLL] = {}


def build(kind: str = "all") -> None:
    target = {"orc": "oracle", "ref": "ref", "all": "all"}[kind]
    subprocess.run(["make", "-s", f"-j{os.cpu_count() or 1}", "-C", HERE, target], check=True)


def available(kind: str) -> bool:
    return os.path.exists(LIB_PATHS[kind])


def _lib(kind: str) -> ctypes.CDLL:
    if kind not in _libs:
        path = LIB_PATHS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing; run `make -C oracle`")
        L = ctypes.CDLL(path)
        p = _prefix(kind)
        vp, u32, u64, sz = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_size_t
        getattr(L, f"{p}_ctx_new").restype = vp
        getattr(L, f"{p}_ctx_new").argtypes = [ctypes.c_char_p, u32, u64]
        getattr(L, f"{p}_tlwe_phase").restype = u32
        getattr(L, f"{p}_tlwe_phase").argtypes = [vp, vp, ctypes.c_int]
        getattr(L, f"{p}_trlwe_phase_at").restype = u32
        getattr(L, f"{p}_trlwe_phase_at").argtypes = [vp, vp, u32]
        getattr(L, f"{p}_ksk_words").restype = sz
        getattr(L, f"{p}_pks_words").restype = sz
        getattr(L, f"{p}_rom_luts").restype = u32
        getattr(L, f"{p}_rom_luts").argtypes = [vp, u32]
        getattr(L, f"{p}_last_error").restype = ctypes.c_char_p
        getattr(L, f"{p}_trlwe_encrypt").argtypes = [vp, vp, ctypes.c_double, vp]
        getattr(L, f"{p}_trgsw_encrypt").argtypes = [vp, ctypes.c_int, ctypes.c_double, vp]
        getattr(L, f"{p}_hom_gate_batch").argtypes = [vp, vp, vp, vp, sz, ctypes.c_uint]
        if kind == "orc":
            L.orc_blind_rotate_lvl2_batch.argtypes = [vp, vp, vp, vp, sz, ctypes.c_uint]
        if p == "ref":
            L.ref_eval_new.restype = vp
            L.ref_eval_new.argtypes = [vp, ctypes.c_char_p, ctypes.c_uint]
            L.ref_eval_run.argtypes = [vp, u64, ctypes.c_uint, u64, vp]
            L.ref_eval_set_input.argtypes = [vp, ctypes.c_char_p, sz, vp, u32]
            L.ref_eval_output.argtypes = [vp, ctypes.c_char_p, sz, vp]
            L.ref_eval_dff_count.restype = sz
            L.ref_eval_dff_count.argtypes = [vp]
            L.ref_hardware_threads.restype = ctypes.c_uint
            L.ref_eval_snapshot_save.argtypes = [vp, vp, sz, ctypes.POINTER(sz)]
            L.ref_serialize_bk.argtypes = [vp, vp, sz, ctypes.POINTER(sz)]
            L.ref_serialize_tlwe.argtypes = [vp, vp, vp, sz, ctypes.POINTER(sz)]
            L.ref_serialize_ram.argtypes = [vp, u32, u32, vp, vp, sz, ctypes.POINTER(sz)]
            L.ref_serialize_rom.argtypes = [vp, u32, vp, u32, vp, sz, ctypes.POINTER(sz)]
            L.ref_ram_read_unit.argtypes = [vp, u32, u32, vp, vp, vp, ctypes.c_uint]
            L.ref_ram_control_unit.argtypes = [vp, u32, vp, vp, vp, vp, vp, ctypes.c_uint]
            L.ref_ram_write_unit.argtypes = [vp, u32, u32, vp, vp, vp, ctypes.c_uint]
            L.ref_rom_read_sel.argtypes = [vp, u32, vp, u32, vp, u32, vp, ctypes.c_uint]
            L.ref_eval_snapshot_load.restype = vp
            L.ref_eval_snapshot_load.argtypes = [vp, ctypes.c_char_p, vp, sz, ctypes.c_uint]
        _libs[kind] = L
    return _libs[kind]


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    assert a.flags["C_CONTIGUOUS"]
    return ctypes.c_void_p(a.ctypes.data)


class CpuTfhe:
    """One parameter set + secret key (+ bootstrapping key) on a CPU checker."""

    def __init__(self, kind: str, params: str = "test-det", n_override: int = 0,
                 seed: int = 20200729):
        self.kind = kind
        self.prefix = _prefix(kind)
        self.L = _lib(kind)
        self.h = self._f("ctx_new")(params.encode(), n_override, seed)
        if not self.h:
            raise ValueError(f"cannot create {kind} context for {params}")
        self.h = ctypes.c_void_p(self.h)
        p = np.zeros(14, np.uint32)
        self._f("params")(self.h, _ptr(p))
        (self.n, self.N1, self.l1, self.Bg1Bits, self.N2, self.l2, self.Bg2Bits,
         self.ksBaseBits, self.ksLen, self.pksBaseBits, self.pksLen) = (int(x) for x in p[:11])
        self.fft = bool(p[11])
        self.params_name = params

    def _f(self, name):
        return getattr(self.L, f"{self.prefix}_{name}")

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self._f("last_error")().decode())

    def __del__(self):
        try:
            self._f("ctx_free")(self.h)
        except Exception:
            pass

    # ---- keys -----------------------------------------------------------
    def keygen(self, with_cb: bool = False):
        self._check(self._f("keygen")(self.h, int(with_cb)))
        self.has_cb = with_cb

    def export_keys(self) -> dict:
        lv0 = np.zeros(self.n, np.uint32)
        lv1 = np.zeros(self.N1, np.uint32)
        lv2 = np.zeros(self.N2, np.uint32)
        self._f("export_sk")(self.h, _ptr(lv0), _ptr(lv1), _ptr(lv2))
        bk1 = np.zeros((self.n, 2 * self.l1, 2, self.N1), np.uint32)
        self._check(self._f("export_bk1")(self.h, _ptr(bk1)))
        ksk = np.zeros(self._f("ksk_words")(self.h), np.uint32)
        self._check(self._f("export_ksk")(self.h, _ptr(ksk)))
        out = dict(lv0=lv0, lv1=lv1, lv2=lv2, bk1=bk1, ksk=ksk, bk2=None, pks_negs=None,
                   pks_id=None)
        pw = self._f("pks_words")(self.h)
        if pw:
            bk2 = np.zeros((self.n, 2 * self.l2, 2, self.N2), np.uint64)
            self._check(self._f("export_bk2")(self.h, _ptr(bk2)))
            pn = np.zeros(pw, np.uint32)
            pi = np.zeros(pw, np.uint32)
            self._check(self._f("export_pks")(self.h, 0, _ptr(pn)))
            self._check(self._f("export_pks")(self.h, 1, _ptr(pi)))
            out.update(bk2=bk2, pks_negs=pn, pks_id=pi)
        return out

    def import_keys(self, k: dict):
        has_cb = k.get("bk2") is not None
        nul = ctypes.c_void_p(0)
        has_pks = k.get("pks_id") is not None
        if self.kind == "orc":
            self._check(self.L.orc_import_keys(
                self.h, _ptr(k["lv0"]), _ptr(k["lv1"]), _ptr(k["lv2"]), _ptr(k["bk1"]),
                _ptr(k["bk2"]) if has_cb else nul, _ptr(k["ksk"]),
                _ptr(k["pks_negs"]) if has_pks else nul, _ptr(k["pks_id"]) if has_pks else nul,
                int(has_cb)))
        else:
            self.L.ref_import_sk(self.h, _ptr(k["lv0"]), _ptr(k["lv1"]), _ptr(k["lv2"]))
            self._check(self.L.ref_import_bk(
                self.h, _ptr(k["bk1"]), _ptr(k["bk2"]) if has_cb else nul, _ptr(k["ksk"]),
                _ptr(k["pks_negs"]) if has_cb else nul, _ptr(k["pks_id"]) if has_cb else nul,
                int(has_cb)))
        self.has_cb = has_cb

    def set_exact(self, exact: bool):
        assert self.kind == "orc"
        self.L.orc_set_exact(self.h, int(exact))

    # ---- client side ----------------------------------------------------
    def encrypt(self, m: int) -> np.ndarray:
        out = np.zeros(self.n + 1, np.uint32)
        self._check(self._f("tlwe_encrypt")(self.h, int(m), _ptr(out)))
        return out

    def encrypt_bits(self, bits) -> np.ndarray:
        return np.stack([self.encrypt(int(b)) for b in bits]) if len(bits) else \
            np.zeros((0, self.n + 1), np.uint32)

    def phase(self, ct: np.ndarray, level: int = 0) -> int:
        return int(self._f("tlwe_phase")(self.h, _ptr(np.ascontiguousarray(ct)), level))

    def decrypt(self, ct: np.ndarray, level: int = 0) -> int:
        return int(np.int32(np.uint32(self.phase(ct, level))) >= 0)

    def trlwe_encrypt(self, bits, alpha: float | None = None) -> np.ndarray:
        b = np.ascontiguousarray(np.asarray(bits, np.uint32))
        out = np.zeros(2 * self.N1, np.uint32)
        self._check(self._f("trlwe_encrypt")(self.h, _ptr(b), 0.0 if alpha is None else alpha,
                                             _ptr(out)))
        return out

    def trlwe_phase_at(self, ct: np.ndarray, k: int) -> int:
        return int(self._f("trlwe_phase_at")(self.h, _ptr(np.ascontiguousarray(ct)), k))

    def trlwe_decrypt_at(self, ct: np.ndarray, k: int) -> int:
        return int(np.int32(np.uint32(self.trlwe_phase_at(ct, k))) >= 0)

    def trgsw_encrypt(self, m: int) -> np.ndarray:
        out = np.zeros((2 * self.l1, 2, self.N1), np.uint32)
        self._check(self._f("trgsw_encrypt")(self.h, int(m), 0.0, _ptr(out)))
        return out

    # ---- evaluation -----------------------------------------------------
    def hom_gate(self, kind, ins) -> np.ndarray:
        k = GATE_KINDS.index(kind) if isinstance(kind, str) else int(kind)
        x = np.ascontiguousarray(np.stack(ins).astype(np.uint32))
        out = np.zeros(self.n + 1, np.uint32)
        self._check(self._f("hom_gate")(self.h, k, _ptr(x), len(ins), _ptr(out)))
        return out

    def hom_gate_batch(self, kinds: np.ndarray, ins: np.ndarray, threads: int = 1) -> np.ndarray:
        kinds = np.ascontiguousarray(kinds.astype(np.int32))
        ins = np.ascontiguousarray(ins.astype(np.uint32))
        G = len(kinds)
        assert ins.shape == (G, 3, self.n + 1)
        out = np.zeros((G, self.n + 1), np.uint32)
        self._check(self._f("hom_gate_batch")(self.h, _ptr(kinds), _ptr(ins), _ptr(out), G,
                                              threads))
        return out

    def gate_bootstrap(self, ct):
        out = np.zeros(self.n + 1, np.uint32)
        self._check(self._f("gate_bootstrap")(self.h, _ptr(np.ascontiguousarray(ct)), _ptr(out)))
        return out

    def bootstrap_to_trlwe(self, ct):
        out = np.zeros(2 * self.N1, np.uint32)
        self._check(self._f("bootstrap_to_trlwe")(self.h, _ptr(np.ascontiguousarray(ct)),
                                                  _ptr(out)))
        return out

    def identity_key_switch(self, ct1):
        out = np.zeros(self.n + 1, np.uint32)
        self._check(self._f("identity_key_switch")(self.h, _ptr(np.ascontiguousarray(ct1)),
                                                   _ptr(out)))
        return out

    def sample_extract(self, trlwe, k):
        out = np.zeros(self.N1 + 1, np.uint32)
        self._check(self._f("sample_extract")(self.h, _ptr(np.ascontiguousarray(trlwe)), k,
                                              _ptr(out)))
        return out

    def cmux(self, sel, c1, c0):
        out = np.zeros(2 * self.N1, np.uint32)
        self._check(self._f("cmux")(self.h, _ptr(np.ascontiguousarray(sel)),
                                    _ptr(np.ascontiguousarray(c1)),
                                    _ptr(np.ascontiguousarray(c0)), _ptr(out)))
        return out

    def hom_mux_no_se_iks(self, s, a, b):
        out = np.zeros(2 * self.N1, np.uint32)
        self._check(self._f("hom_mux_no_se_iks")(self.h, _ptr(s), _ptr(a), _ptr(b), _ptr(out)))
        return out

    def circuit_bootstrap(self, ct):
        out = np.zeros((2 * self.l1, 2, self.N1), np.uint32)
        self._check(self._f("circuit_bootstrap")(self.h, _ptr(np.ascontiguousarray(ct)),
                                                 _ptr(out)))
        return out

    def blind_rotate_lvl2(self, ct: np.ndarray, h: int) -> np.ndarray:
        assert self.kind == "orc"
        tv = np.zeros(2 * self.N2, np.uint64)
        tv[self.N2:] = np.uint64(h // 2)
        out = np.zeros(2 * self.N2, np.uint64)
        self._check(self.L.orc_blind_rotate_lvl2(self.h, _ptr(np.ascontiguousarray(ct)),
                                                 _ptr(tv), _ptr(out)))
        return out

    def blind_rotate_lvl2_batch(self, cts: np.ndarray, h, threads: int = 1) -> np.ndarray:
        """T level-2 blind rotations with test vectors b = h[t]/2 (restatement only)."""
        assert self.kind == "orc"
        cts = np.ascontiguousarray(np.atleast_2d(cts), np.uint32)
        hv = np.ascontiguousarray(np.broadcast_to(np.asarray(h, np.uint64), (cts.shape[0],)))
        out = np.zeros((cts.shape[0], 2 * self.N2), np.uint64)
        self._check(self.L.orc_blind_rotate_lvl2_batch(self.h, _ptr(cts), _ptr(hv), _ptr(out),
                                                       cts.shape[0], threads))
        return out

    def private_key_switch(self, t2: np.ndarray, which: int):
        out = np.zeros(2 * self.N1, np.uint32)
        self._check(self._f("private_key_switch")(self.h, _ptr(np.ascontiguousarray(t2)),
                                                  which, _ptr(out)))
        return out

    def trgsw_not(self, g):
        out = np.zeros_like(g)
        self._check(self._f("trgsw_not")(self.h, _ptr(np.ascontiguousarray(g)), _ptr(out)))
        return out

    def encrypt_ram(self, image: np.ndarray, v: int, w: int, trivial: bool = False):
        out = np.zeros(((w << v), 2 * self.N1), np.uint32)
        img = np.ascontiguousarray(image.astype(np.uint8))
        self._check(self._f("encrypt_ram")(self.h, _ptr(img), v, w, int(trivial), _ptr(out)))
        return out

    def decrypt_ram(self, ram: np.ndarray, v: int, w: int) -> np.ndarray:
        img = np.zeros((w << v) // 8, np.uint8)
        self._check(self._f("decrypt_ram")(self.h, _ptr(np.ascontiguousarray(ram)), v, w,
                                           _ptr(img)))
        return img

    def encrypt_rom(self, image: np.ndarray, trivial: bool = False):
        nl = self._f("rom_luts")(self.h, len(image))
        out = np.zeros((nl, 2 * self.N1), np.uint32)
        img = np.ascontiguousarray(image.astype(np.uint8))
        self._check(self._f("encrypt_rom")(self.h, _ptr(img), len(image), int(trivial),
                                           _ptr(out)))
        return out

    def ram_cycle(self, ram: np.ndarray, v, w, addr, wflag, wdata, threads: int = 1):
        ram = np.ascontiguousarray(ram.copy())
        ro = np.zeros((w, self.n + 1), np.uint32)
        a = np.ascontiguousarray(addr)
        f = np.ascontiguousarray(wflag)
        d = np.ascontiguousarray(wdata)
        if self.prefix == "ref":
            rc = self.L.ref_ram_cycle(self.h, v, w, _ptr(ram), _ptr(a), _ptr(f), _ptr(d),
                                      _ptr(ro), threads)
        else:
            rc = self.L.orc_ram_cycle(self.h, v, w, _ptr(ram), _ptr(a), _ptr(f), _ptr(d),
                                      _ptr(ro))
        self._check(rc)
        return ro, ram

    def rom_read(self, luts: np.ndarray, depth_bytes: int, addr: np.ndarray, threads: int = 1):
        vrom = addr.shape[0]
        out = np.zeros((32, self.n + 1), np.uint32)
        lu = np.ascontiguousarray(luts)
        a = np.ascontiguousarray(addr)
        if self.prefix == "ref":
            rc = self.L.ref_rom_read(self.h, depth_bytes, _ptr(lu), lu.shape[0], _ptr(a), vrom,
                                     _ptr(out), threads)
        else:
            rc = self.L.orc_rom_read(self.h, depth_bytes, _ptr(lu), lu.shape[0], _ptr(a), vrom,
                                     _ptr(out))
        self._check(rc)
        return out

    # ---- the units of ramCycle / romRead on given selectors (reference only) ----------
    def _need_ref(self):
        if self.prefix != "ref":
            raise NotImplementedError("memory units on selectors: reference checker only")

    def ram_read_unit(self, ram, v, w, sel, threads: int = 1) -> np.ndarray:
        self._need_ref()
        out = np.zeros((w, 2 * self.N1), np.uint32)
        self._check(self.L.ref_ram_read_unit(self.h, v, w, _ptr(np.ascontiguousarray(ram)),
                                             _ptr(np.ascontiguousarray(sel)), _ptr(out),
                                             threads))
        return out

    def ram_control_unit(self, read, wflag, wdata, threads: int = 1):
        self._need_ref()
        w = read.shape[0]
        ro = np.zeros((w, self.n + 1), np.uint32)
        ctl = np.zeros((w, 2 * self.N1), np.uint32)
        self._check(self.L.ref_ram_control_unit(
            self.h, w, _ptr(np.ascontiguousarray(read)), _ptr(np.ascontiguousarray(wflag)),
            _ptr(np.ascontiguousarray(wdata)), _ptr(ro), _ptr(ctl), threads))
        return ro, ctl

    def ram_write_unit(self, ram, v, w, sel, controlled, threads: int = 1) -> np.ndarray:
        self._need_ref()
        ram = np.array(ram, np.uint32)
        self._check(self.L.ref_ram_write_unit(self.h, v, w, _ptr(ram),
                                              _ptr(np.ascontiguousarray(sel)),
                                              _ptr(np.ascontiguousarray(controlled)), threads))
        return ram

    def rom_read_sel(self, luts, depth_bytes, sel, threads: int = 1) -> np.ndarray:
        self._need_ref()
        sel = np.ascontiguousarray(sel)
        out = np.zeros((32, self.n + 1), np.uint32)
        lu = np.ascontiguousarray(luts)
        self._check(self.L.ref_rom_read_sel(self.h, depth_bytes, _ptr(lu), lu.shape[0],
                                            _ptr(sel), sel.shape[0], _ptr(out), threads))
        return out

    def counters(self) -> np.ndarray:
        out = np.zeros(5, np.uint64)
        self._f("counters")(_ptr(out))
        return out

    def counters_reset(self):
        self._f("counters_reset")()


def ref_bytes(fn, *args) -> bytes:
    """Call a two-pass ref_serialize_* / snapshot function of the reference shim."""
    L = _lib("ref")
    n = ctypes.c_size_t()
    rc = getattr(L, fn)(*args, None, 0, ctypes.byref(n))
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    buf = np.zeros(n.value, np.uint8)
    rc = getattr(L, fn)(*args, buf.ctypes.data_as(ctypes.c_void_p), buf.size, ctypes.byref(n))
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    return buf.tobytes()

