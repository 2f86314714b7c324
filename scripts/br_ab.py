"""A/B of blind-rotation kernel variants (env knobs read once per process): each variant
runs in its own subprocess on the same keys and 4,096-gate n=630 batch; prints step time,
br1024 / br_lat / iks event time per step and a hash of the outputs (must match the
baseline's: the variants are bit-exact by construction).

    python scripts/br_ab.py '{}' '{"VSP_BR_SLOTS": "4", "VSP_BR_OFS": "1"}' ...
    python scripts/br_ab.py --gates 140 ...        (a narrow level: br_lat)
"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(G, reps):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import paper_2010_09410_b200 as vsp
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
    s = torch.cuda.current_stream()
    for _ in range(2):
        e.hom_gate_batch_dev(kid, d_in.data_ptr(), d_out.data_ptr(), G, s.cuda_stream)
    torch.cuda.synchronize()
    e.profile_reset()
    e.profile_enable(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        e.hom_gate_batch_dev(kid, d_in.data_ptr(), d_out.data_ptr(), G, s.cuda_stream)
    b.record(s)
    torch.cuda.synchronize()
    e.profile_enable(False)
    res = {"step_ms": round(a.elapsed_time(b) / reps, 3)}
    for name in ("br1024", "br_lat", "iks"):
        ms, n = e.profile_read(name)
        if n:
            res[name + "_ms"] = round(ms / reps, 3)
    out = d_out.cpu().numpy()
    res["hash"] = hashlib.sha256(out.tobytes()).hexdigest()[:16]
    res["decrypt_ok"] = bool(np.array_equal(
        vsp.decrypt(k["lv0"], out.view(np.uint32)),
        np.where(kid == 3, 1 - (vsp.decrypt(k["lv0"], ins[:, 0]) & vsp.decrypt(k["lv0"], ins[:, 1])),
                 vsp.decrypt(k["lv0"], ins[:, 0]) ^ vsp.decrypt(k["lv0"], ins[:, 1]))))
    print("RESULT " + json.dumps(res), flush=True)


def main():
    args = sys.argv[1:]
    G, reps = 4096, 5
    if args and args[0] == "--child":
        child(int(args[1]), int(args[2]))
        return
    if args and args[0] == "--gates":
        G = int(args[1])
        args = args[2:]
    variants = [json.loads(a) for a in args] or [{}]
    rows = []
    for v in variants:
        env = dict(os.environ, **v)
        r = subprocess.run([sys.executable, __file__, "--child", str(G), str(reps)], env=env,
                           capture_output=True, text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
        res = json.loads(line[0][7:]) if line else {"error": r.stderr[-800:]}
        res["variant"] = v
        rows.append(res)
        print(json.dumps(res), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(rows, open(os.path.join(ROOT, "gpurun_out", f"br_ab_{G}.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
