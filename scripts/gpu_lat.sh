# Latency kernel: parity (gate tests use narrow batches) + cycle/memory benches + BR latency sweep.
O=gpurun_out/lat.log
: > $O
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log >> $O
timeout 600 python bench.py --config cycle --steps 3 --warmup 1 > gpurun_out/bench_cycle.json 2> gpurun_out/bench_cycle.err; cat gpurun_out/bench_cycle.json >> $O; tail -2 gpurun_out/bench_cycle.err >> $O
timeout 600 python bench.py --config memory --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_memory.json 2> gpurun_out/bench_memory.err; cat gpurun_out/bench_memory.json >> $O
timeout 600 python scripts/br_occupancy.py >> $O 2>&1
cat $O
