# Session-3 ncu captures (--set full) of the current kernels, summarised on the box:
# headline batch (br1024<8>, br1024p<4>, split-K key switch), a 140-gate narrow level
# (br_lat + key switch), one memory access (br2q, pks_stream, chains).
set -x
O=gpurun_out/ncu_s3
mkdir -p $O
timeout 900 ncu --set full --clock-control none -k regex:"br1024|iks_gemm|cutlass" --launch-skip 5 -c 5 \
  -o /tmp/s3_gates python scripts/br_once.py 4096 > $O/gates.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"br_lat|iks_gemm|cutlass|gate_prep" --launch-skip 5 -c 5 \
  -o /tmp/s3_lat python scripts/br_once.py 140 > $O/lat.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:"br2q|pks|cmux_chain|br1024|br_lat|cutlass" -c 30 \
  -o /tmp/s3_mem python bench.py --config memory --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/mem.log 2>&1
for r in gates lat mem; do
  python scripts/ncu_summary.py rep /tmp/s3_$r.ncu-rep $O/${r}_summary.json > /dev/null 2>&1 || \
    ncu -i /tmp/s3_$r.ncu-rep --page raw --csv > $O/${r}_raw.csv
done
ls -la $O
