# ncu --set full of the cycle path's latency kernels (narrow-level blind rotation, level-2
# blind rotation of the circuit bootstrap, private key switch) in one cycle of the bench.
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"br_lat|br2q|pks_kernel" -c 4 \
  -o gpurun_out/prof_cycle_v2 python bench.py --config cycle --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_cycle.log 2>&1
tail -3 gpurun_out/ncu_cycle.log
