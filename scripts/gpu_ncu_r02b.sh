# ncu of the round-2 kernels on the headline batch: br1024p remainder wave and the INT8
# GEMM key switch (selectors, cuBLASLt GEMM, epilogue); CSV exported on the box.
set -x
O=gpurun_out/ncu_r02b
mkdir -p $O
timeout 900 ncu --set full --clock-control none -k regex:"br1024p|iks_gemm|gemm|Kernel|sm100" \
  --launch-skip 5 -c 5 -o /tmp/r02b python scripts/br_once.py 4096 > $O/ncu.log 2>&1
ncu -i /tmp/r02b.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_gates.csv python bench.py --steps 2 --warmup 1 --headline-only \
  --no-cpu-baseline --no-e2e > $O/bench_under_ncu.log 2>&1
gzip -f $O/*.csv
ls -la $O
