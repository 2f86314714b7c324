"""Calibrates br_plan's cost model (vsp_capi.cu): blind-rotation launch time at n = 630 for
one wave of each kernel -- br1024 at W = 1..8 tasks per SM (forced), br1024p at W = 3, 4
(the plan's own pick), br_lat at 148 and 149 tasks, br_lat2 at 149 and 296 -- each in its
own process (the kernel-choice knobs are read once)."""
import json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(T, reps=3):
    sys.path.insert(0, ROOT)
    import numpy as np, torch
    import paper_2010_09410_b200 as vsp
    p = vsp.ParameterSet("tfhe-80", 630)
    k = vsp.keygen(p, 5, False)
    e = vsp.Engine(p)
    e.upload_keys(k)
    ins = np.zeros((T, 3, p.n + 1), np.uint32)
    ins[:, :2] = vsp.encrypt(p, k["lv0"], np.ones(2 * T, np.uint8), 1).reshape(T, 2, p.n + 1)
    d_in = torch.from_numpy(ins.view(np.int32)).cuda()
    d_out = torch.empty((T, p.n + 1), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    kid = np.full(T, 3, np.int32)
    e.hom_gate_batch_dev(kid, d_in.data_ptr(), d_out.data_ptr(), T, s.cuda_stream)
    torch.cuda.synchronize()
    e.profile_reset()
    e.profile_enable(True)
    for _ in range(reps):
        e.hom_gate_batch_dev(kid, d_in.data_ptr(), d_out.data_ptr(), T, s.cuda_stream)
    torch.cuda.synchronize()
    e.profile_enable(False)
    out = {}
    for name in ("br1024", "br_lat"):
        ms, n = e.profile_read(name)
        if n:
            out[name] = round(ms / reps, 3)
    print("RESULT " + json.dumps(out), flush=True)


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--child":
        child(int(sys.argv[2]))
        return
    runs = [(f"br1024 W={w}", 148 * w, {"VSP_BR_WARPS": str(w), "VSP_BR_PAIR": "0"}) for w in range(1, 9)]
    runs += [("br1024p W=3", 444, {}), ("br1024p W=4", 592, {})]
    runs += [("br_lat 148", 148, {}), ("br_lat 149", 149, {}),
             ("br_lat2 149", 149, {"VSP_LAT_TASKS": "2"}), ("br_lat2 296", 296, {"VSP_LAT_TASKS": "2"})]
    res = {}
    for name, T, env in runs:
        r = subprocess.run([sys.executable, __file__, "--child", str(T)], env=dict(os.environ, **env),
                           capture_output=True, text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
        res[name] = json.loads(line[0][7:]) if line else {"error": r.stderr[-300:]}
        print(name, T, res[name], flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(res, open(os.path.join(ROOT, "gpurun_out", "calib_waves.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
