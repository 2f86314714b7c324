"""One hom_gate_batch_dev of G NAND/XOR gates at n=630 after one warm-up call (for ncu
captures of a single blind-rotation launch: --launch-skip 1)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2010_09410_b200 as vsp
G = int(sys.argv[1]) if len(sys.argv) > 1 else 1184
p = vsp.ParameterSet("tfhe-80", 630)
k = vsp.keygen(p, 5, False)
e = vsp.Engine(p)
e.upload_keys(k)
rng = np.random.default_rng(1)
kid = rng.choice([3, 9], G).astype(np.int32)
ins = np.zeros((G, 3, p.n + 1), np.uint32)
ins[:, :2] = vsp.encrypt(p, k["lv0"], rng.integers(0, 2, 2 * G).astype(np.uint8), 2).reshape(G, 2, p.n + 1)
d_in = torch.from_numpy(ins.view(np.int32)).cuda()
d_out = torch.empty((G, p.n + 1), dtype=torch.int32, device="cuda")
for _ in range(2):
    e.hom_gate_batch_dev(kid, d_in.data_ptr(), d_out.data_ptr(), G)
torch.cuda.synchronize()
print("done", G)
