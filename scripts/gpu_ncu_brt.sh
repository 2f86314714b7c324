# ncu of the TMEM blind rotation at W=12 (1 GPU).
VSP_BR_TMEM=1 VSP_BR_WARPS=12 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"br1024" -c 1 \
  -o gpurun_out/prof_brt python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_brt.log 2>&1
tail -3 gpurun_out/ncu_brt.log
