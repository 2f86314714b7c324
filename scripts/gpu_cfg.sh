# Memory (configs[1]) and cycle (configs[2]) benches with their reference CPU baselines.
timeout 900 python bench.py --config memory --steps 3 --warmup 1 > gpurun_out/bench_memory.json 2> gpurun_out/bench_memory.err
timeout 1200 python bench.py --config cycle --steps 3 --warmup 1 > gpurun_out/bench_cycle.json 2> gpurun_out/bench_cycle.err
tail -2 gpurun_out/bench_memory.err gpurun_out/bench_cycle.err
cat gpurun_out/bench_memory.json gpurun_out/bench_cycle.json
