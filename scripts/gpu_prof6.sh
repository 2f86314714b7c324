# Evidence for the round: ncu launch list of the headline bench and one --set full capture
# of the blind-rotation (both launches of a step) and key-switch kernels.
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"br1024|iks_b2|br_lat" -s 3 -c 3 \
  -o gpurun_out/prof_v6 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_v6.log 2>&1
tail -2 gpurun_out/ncu_v6.log
