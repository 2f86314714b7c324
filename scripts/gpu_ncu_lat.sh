timeout 600 ncu --set full --clock-control none --import-source on -k regex:"br_lat" -s 1 -c 1 -o gpurun_out/prof_lat python scripts/one_gate.py 1 > gpurun_out/ncu_lat.log 2>&1
tail -2 gpurun_out/ncu_lat.log
