set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | tee gpurun_out/bench2.json
timeout 600 ncu --set full --clock-control none -k regex:iks_kernel -s 1 -c 1 -o gpurun_out/prof_iks2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_iks2.log 2>&1
