# GPU parity suite + default bench (one JSON line with the memory and cycle sub-objects).
set -x
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -8 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python - <<'P'
import json; d=json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
print("gates/s", d["value"], "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"])
print("memory", d["memory"]["value"], d["memory"]["kernel_ms_per_access"])
print("cycle", d["cycle"]["value"], d["cycle"]["kernel_ms_per_cycle"])
P
