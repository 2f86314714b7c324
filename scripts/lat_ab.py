"""br_lat per-level time at T tasks (one level of NAND gates), for A/B of kernel knobs."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2010_09410_b200 as vsp
T = int(sys.argv[1]) if len(sys.argv) > 1 else 140
p = vsp.ParameterSet("tfhe-80", 630)
k = vsp.keygen(p, 5, False)
e = vsp.Engine(p); e.upload_keys(k)
bits = np.random.default_rng(1).integers(0, 2, 2 * T).astype(np.uint8)
ins = np.zeros((T, 3, p.n + 1), np.uint32)
ins[:, :2] = vsp.encrypt(p, k["lv0"], bits, 1).reshape(T, 2, p.n + 1)
kid = np.full(T, vsp.GATE_KINDS.index("NAND"), np.int32)
out = e.hom_gate_batch(kid, ins)
ok = np.array_equal(vsp.decrypt(k["lv0"], out), 1 - (bits[0::2] & bits[1::2]))
e.profile_reset(); e.profile_enable(True)
for _ in range(5):
    e.hom_gate_batch(kid, ins)
e.profile_enable(False)
ms, n = e.profile_read("br_lat")
import hashlib
print(f"T={T} br_lat {ms / max(n, 1):.3f} ms/level correct={ok} out={hashlib.sha1(out.tobytes()).hexdigest()[:12]}")
