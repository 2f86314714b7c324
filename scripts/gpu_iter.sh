# Inner loop: parity, latency probe, headline bench, cycle bench (no CPU baselines).
O=gpurun_out/iter.log
: > $O
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log >> $O
VSP_LAT_PROBE=1 timeout 300 python scripts/one_gate.py 74 2>&1 | tail -5 >> $O
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json >> $O
timeout 600 python bench.py --config cycle --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_cycle.json 2> gpurun_out/bench_cycle.err; cat gpurun_out/bench_cycle.json >> $O; tail -2 gpurun_out/bench_cycle.err >> $O
cat $O
