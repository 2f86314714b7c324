# Memory (configs[1]) and cycle (configs[2]) benches + narrow-level BR latency.
set -x
timeout 900 python bench.py --config memory --steps 3 --warmup 1 > gpurun_out/bench_memory.json 2> gpurun_out/bench_memory.err; tail -3 gpurun_out/bench_memory.err; cat gpurun_out/bench_memory.json
timeout 900 python bench.py --config cycle --steps 3 --warmup 1 > gpurun_out/bench_cycle.json 2> gpurun_out/bench_cycle.err; tail -3 gpurun_out/bench_cycle.err; cat gpurun_out/bench_cycle.json
