set -x
timeout 900 ncu --set full --clock-control none -k regex:"pks" -c 1 -o /tmp/pks python bench.py --config memory --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_pks.log 2>&1
ncu -i /tmp/pks.ncu-rep --page raw --csv > gpurun_out/pks_raw.csv 2>/dev/null
ncu -i /tmp/pks.ncu-rep --page details --csv > gpurun_out/pks_details.csv 2>/dev/null
tail -2 gpurun_out/ncu_pks.log
