"""Blind-rotation time per launch vs batch size T, for the latency kernel (br_lat, T <=
2 x SMs) and the throughput kernel (br1024, W tasks per CTA); calibrates br_warps_for()."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2010_09410_b200 as vsp
p = vsp.ParameterSet("tfhe-80", 630)
k = vsp.keygen(p, 5, False)
e = vsp.Engine(p); e.upload_keys(k)
res = {}
for T in [1, 8, 74, 148, 296, 444, 592, 740, 888, 1036, 1184]:
    ins = np.zeros((T, 3, p.n + 1), np.uint32)
    ins[:, :2] = vsp.encrypt(p, k["lv0"], np.ones(2 * T, np.uint8), 1).reshape(T, 2, p.n + 1)
    d_in = torch.from_numpy(ins.view(np.int32)).cuda(); d_out = torch.empty((T, p.n + 1), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    kinds = ["NAND"] * T
    row = {}
    for mode in ["auto", "w1"]:
        if mode == "w1":
            os.environ["VSP_BR_WARPS"] = str(max(1, min(8, (T + 147) // 148)))
        else:
            os.environ.pop("VSP_BR_WARPS", None)
        e.hom_gate_batch_dev(kinds, d_in.data_ptr(), d_out.data_ptr(), T, s.cuda_stream); torch.cuda.synchronize()
        e.profile_reset(); e.profile_enable(True)
        for _ in range(3):
            e.hom_gate_batch_dev(kinds, d_in.data_ptr(), d_out.data_ptr(), T, s.cuda_stream)
        torch.cuda.synchronize(); e.profile_enable(False)
        for name in ("br_lat", "br1024"):
            ms, n = e.profile_read(name)
            if n:
                row[f"{mode}:{name}"] = round(ms / n, 3)
    res[T] = row
    print(T, row, flush=True)
os.environ.pop("VSP_BR_WARPS", None)
json.dump(res, open("gpurun_out/br_occupancy.json", "w"))
