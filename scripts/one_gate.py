"""A batch of T gates (default 1) bootstrapped a few times: narrow-level latency probe."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2010_09410_b200 as vsp
T = int(sys.argv[1]) if len(sys.argv) > 1 else 1
p = vsp.ParameterSet("tfhe-80", 630)
k = vsp.keygen(p, 5, False)
e = vsp.Engine(p); e.upload_keys(k)
ins = np.zeros((T, 3, p.n + 1), np.uint32)
ins[:, :2] = vsp.encrypt(p, k["lv0"], np.ones(2 * T, np.uint8), 1).reshape(T, 2, p.n + 1)
for _ in range(3):
    out = e.hom_gate_batch(["NAND"] * T, ins)
print("ok", vsp.decrypt(k["lv0"], out)[:4])
