# Session-3 evidence (1 GPU): headline launch list, a narrow level's split-K key switch
# under ncu --set full (raw CSV), and the 1k..1M sweep.
set -x
O=gpurun_out/ev3
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --headline-only > $O/b_ncu.log 2>&1
python scripts/ncu_summary.py launches $O/launches.csv $O/launches.json > /dev/null
timeout 600 ncu --set full --clock-control none -k regex:"iks_gemm|cutlass|gemm|br_lat" \
  --launch-skip 8 -c 8 -o /tmp/s3_lat python scripts/br_once.py 140 > $O/lat.log 2>&1
ncu -i /tmp/s3_lat.ncu-rep --page raw --csv > $O/lat_raw.csv 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/cycle_launches.csv \
  python bench.py --config cycle --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/c_ncu.log 2>&1
gzip -f $O/*.csv
timeout 2400 python scripts/sweep.py > $O/sweep.log 2>&1
cp gpurun_out/sweep.json $O/
ls -la $O
