# ncu --set full with source counters of one whole-wave br1024<8> launch (1184 tasks) and one
# 140-task br_lat launch (1 GPU).
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"br1024_kernel" --launch-skip 1 -c 1 \
  -o gpurun_out/src_br1024 python scripts/br_once.py 1184 > gpurun_out/ncu_src1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"br_lat_kernel" --launch-skip 1 -c 1 \
  -o gpurun_out/src_brlat python scripts/br_once.py 140 > gpurun_out/ncu_src2.log 2>&1
tail -3 gpurun_out/ncu_src1.log gpurun_out/ncu_src2.log
ls -la gpurun_out/
