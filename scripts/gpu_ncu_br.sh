# One ncu --set full capture of the blind-rotation and key-switch kernels (1 GPU).
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"br1024|iks_b2" -c 2 \
  -o gpurun_out/prof_br python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_br.log 2>&1
tail -3 gpurun_out/ncu_br.log
ls -la gpurun_out/
