"""Shared fixtures/helpers for the parity tests (test infrastructure)."""
import functools
import os

import numpy as np

from oracle.pyoracle import CpuTfhe, GATE_KINDS

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

TRUTH = {
    "AND": lambda a, b, c: a & b, "ANDNOT": lambda a, b, c: a & (1 - b),
    "NAND": lambda a, b, c: 1 - (a & b), "NOR": lambda a, b, c: 1 - (a | b),
    "OR": lambda a, b, c: a | b, "ORNOT": lambda a, b, c: a | (1 - b),
    "XNOR": lambda a, b, c: 1 - (a ^ b), "XOR": lambda a, b, c: a ^ b,
    "NOT": lambda a, b, c: 1 - a, "MUX": lambda s, a, b: a if s else b,
}


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


@functools.lru_cache(maxsize=None)
def oracle(params: str, seed: int, with_cb: bool, n_override: int = 0) -> CpuTfhe:
    """Oracle restatement with keygen from the seed (bit-exact with the reference)."""
    o = CpuTfhe("orc", params, n_override=n_override, seed=seed)
    o.keygen(with_cb)
    return o


@functools.lru_cache(maxsize=None)
def oracle_keys(params: str, seed: int, with_cb: bool, n_override: int = 0) -> dict:
    return oracle(params, seed, with_cb, n_override).export_keys()


def random_gate_batch(o: CpuTfhe, rng, G, kinds=None):
    kinds = kinds or GATE_KINDS
    ks = [kinds[int(rng.integers(0, len(kinds)))] for _ in range(G)]
    bits = rng.integers(0, 2, size=(G, 3))
    ins = np.zeros((G, 3, o.n + 1), np.uint32)
    for g in range(G):
        for i in range(3):
            ins[g, i] = o.encrypt(int(bits[g, i]))
    return ks, bits, ins


@functools.lru_cache(maxsize=None)
def keys_with_cb(n: int, seed: int) -> dict:
    """tfhe-80 keys with circuit-bootstrapping material at LWE dimension n (the engine's
    client keygen: the reference's CSPRNG stream and draw order, bit-identical keys)."""
    import paper_2010_09410_b200 as vsp
    return vsp.keygen(vsp.ParameterSet("tfhe-80", n_override=n), seed, True)


def phase_error(ph, bits, mu=1 << 29) -> np.ndarray:
    """phaseError (test_tfhe.cpp:80-86): |phase - (+-mu)| / 2^32 per ciphertext."""
    ph = np.asarray(ph, np.uint32)
    want = np.where(np.asarray(bits) != 0, np.uint32(mu), np.uint32((1 << 32) - mu))
    return np.abs((ph - want).astype(np.uint32).view(np.int32).astype(np.float64)) / 2.0 ** 32


def stddev_of_errors(err) -> float:
    """stddevOfErrors (test_tfhe.cpp:88-94): root mean square of the errors."""
    err = np.asarray(err, np.float64)
    return float(np.sqrt(np.mean(err * err)))
