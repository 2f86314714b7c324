"""Generate golden vectors from the REFERENCE itself (oracle/_ref/libhvpref.so, built
from /root/reference/proj/src by oracle/Makefile).  Run in the build container:

    python tests/golden/make_golden.py

Keys are not stored (they are reproducible from the seed and pinned by their SHA-256);
inputs and reference outputs of a few operations are stored verbatim.
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import CpuTfhe, GATE_KINDS  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gates(r, rng, count):
    kinds, ins, outs = [], [], []
    for g in range(count):
        kind = GATE_KINDS[g % len(GATE_KINDS)]
        x = np.zeros((3, r.n + 1), np.uint32)
        ar = 3 if kind == "MUX" else 1 if kind == "NOT" else 2
        for i in range(ar):
            x[i] = r.encrypt(int(rng.integers(0, 2)))
        kinds.append(GATE_KINDS.index(kind))
        ins.append(x)
        outs.append(r.hom_gate(kind, list(x[:ar])))
    return np.array(kinds, np.int32), np.stack(ins), np.stack(outs)


def main():
    rng = np.random.default_rng(1234)
    # test-det, fixture seed of test_mem.cpp:16 (with circuit-bootstrapping material)
    r = CpuTfhe("ref", "test-det", seed=515253)
    r.keygen(True)
    k = r.export_keys()
    kinds, ins, outs = gates(r, rng, 40)
    cb_in = np.stack([r.encrypt(1), r.encrypt(0)])
    cb_out = np.stack([r.circuit_bootstrap(c) for c in cb_in])
    np.savez_compressed(os.path.join(OUT, "testdet_seed515253.npz"),
                        key_sha=np.array([sha(k[x]) for x in
                                          ["lv0", "lv1", "lv2", "bk1", "ksk", "bk2", "pks_negs",
                                           "pks_id"]]),
                        kinds=kinds, ins=ins, outs=outs, cb_in=cb_in, cb_out=cb_out)
    # tfhe-80, fixture seed of test_tfhe.cpp:35 (no CB material, as the reference fixture)
    r = CpuTfhe("ref", "tfhe-80", seed=20200729)
    r.keygen(False)
    k = r.export_keys()
    kinds, ins, outs = gates(r, rng, 12)
    lvl0 = np.stack([r.encrypt(int(rng.integers(0, 2))) for _ in range(2)])
    trlwe = np.stack([r.bootstrap_to_trlwe(c) for c in lvl0])
    np.savez_compressed(os.path.join(OUT, "tfhe80_seed20200729.npz"),
                        key_sha=np.array([sha(k[x]) for x in ["lv0", "lv1", "lv2", "bk1", "ksk"]]),
                        kinds=kinds, ins=ins, outs=outs, br_in=lvl0, br_out=trlwe)
    # n = 630 variant of tfhe-80 (BASELINE config 1)
    r = CpuTfhe("ref", "tfhe-80", n_override=630, seed=630)
    r.keygen(False)
    k = r.export_keys()
    kinds, ins, outs = gates(r, rng, 4)
    np.savez_compressed(os.path.join(OUT, "tfhe80n630_seed630.npz"),
                        key_sha=np.array([sha(k[x]) for x in ["lv0", "lv1", "lv2", "bk1", "ksk"]]),
                        kinds=kinds, ins=ins, outs=outs)
    print("golden vectors written to", OUT)


if __name__ == "__main__":
    main()
