"""Circuit bootstrapping latency probe (ROM read at tfhe-80 n=630)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2010_09410_b200 as vsp
p = vsp.ParameterSet("tfhe-80", 630)
k = vsp.keygen(p, 5, True)
e = vsp.Engine(p); e.upload_keys(k)
rng = np.random.default_rng(1)
luts = vsp.encrypt_rom(p, k, rng.integers(0, 256, 512).astype(np.uint8), 6)
addr = vsp.encrypt(p, k["lv0"], rng.integers(0, 2, 7), 10)
for _ in range(2):
    out = e.rom_read(luts, 512, addr)
print("ok", out.shape)
