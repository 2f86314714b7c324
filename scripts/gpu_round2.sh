# Milestone evidence: parity tests, headline bench (with CPU baseline), reference arm,
# memory + cycle configs, launch list of the headline bench.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1
timeout 900 python bench.py --config memory --steps 3 --warmup 1 > gpurun_out/bench_memory.json 2> gpurun_out/bench_memory.err
timeout 900 python bench.py --config cycle --steps 3 --warmup 1 > gpurun_out/bench_cycle.json 2> gpurun_out/bench_cycle.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches.csv gpurun_out/launches.json > /dev/null
cat gpurun_out/bench.json gpurun_out/bench_ref.json gpurun_out/bench_memory.json gpurun_out/bench_cycle.json
