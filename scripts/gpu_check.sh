set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench3.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:br1024 -s 1 -c 1 -o gpurun_out/prof_br3 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full3.log 2>&1
