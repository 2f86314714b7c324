"""BASELINE configs[4] at N=1: gates/s for single-level batches of 1k .. 1M gates
(bench.py --gates G), summarised into gpurun_out/sweep.json."""
import json, subprocess, sys
res = []
for G in [1024, 4096, 16384, 65536, 262144, 1048576]:
    steps = 2 if G >= 262144 else 5
    r = subprocess.run([sys.executable, "bench.py", "--gates", str(G), "--steps", str(steps),
                        "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--headline-only"],
                       capture_output=True, text=True, timeout=1800)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception:
        print(G, "failed", r.stderr[-500:], flush=True)
        continue
    row = {"gates": G, "gates_per_s": d["value"], "ms_per_step": d["ms_per_step"],
           "br_frac_fp64": d["roofline"]["frac"], "breakdown": d["breakdown"],
           "decrypt_correct": d["outputs_decrypt_correct"], "clocks": d["clocks"]}
    res.append(row)
    print(json.dumps(row), flush=True)
json.dump(res, open("gpurun_out/sweep.json", "w"), indent=1)
