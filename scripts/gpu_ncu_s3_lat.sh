# ncu --set full of one 148-task narrow level (br_lat) and its key switch (session 3).
set -x
O=gpurun_out/ncu_s3
mkdir -p $O
timeout 900 ncu -f --set full --clock-control none -k regex:"br_lat|iks_gemm|gate_prep" --launch-skip 4 -c 4 \
  -o /tmp/s3_lat148 python scripts/br_once.py 148 > $O/lat148.log 2>&1
python scripts/ncu_summary.py rep /tmp/s3_lat148.ncu-rep $O/lat148_summary.json > /dev/null 2>&1
ls -la $O
