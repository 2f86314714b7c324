"""Level-2 blind rotation (circuit bootstrap core) per-launch time at T tasks, for A/B of
br2q variants; prints a hash of the outputs so variants are compared word for word."""
import hashlib
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2010_09410_b200 as vsp
T = int(sys.argv[1]) if len(sys.argv) > 1 else 30
p = vsp.ParameterSet("tfhe-80", 630)
k = vsp.keygen(p, 5, True, device=0)
e = vsp.Engine(p)
e.upload_keys(k)
rng = np.random.default_rng(3)
cts = rng.integers(0, 2**32, (T, p.n + 1), dtype=np.uint64).astype(np.uint32)
out = e.blind_rotate_lvl2(cts, 1 << 52)
e.profile_reset()
e.profile_enable(True)
for _ in range(5):
    e.blind_rotate_lvl2(cts, 1 << 52)
e.profile_enable(False)
ms, n = e.profile_read("br2")
print(f"T={T} br2 {ms / max(n, 1):.3f} ms/launch out={hashlib.sha1(out.tobytes()).hexdigest()[:12]}")
