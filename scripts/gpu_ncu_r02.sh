# Round-2 ncu evidence (1 GPU): (1) the headline gate batch (br1024 W=8 whole waves, W=4
# remainder, forked + final iks_b2) and (2) one ROM read + RAM cycle (circuit bootstrap
# br2q + pks_kernel, CMUX chains, key switches, control-unit br_lat, write-bar br1024).
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"br1024|iks_b2" \
  --launch-skip 4 -c 4 -o gpurun_out/r02_gates python scripts/br_once.py 4096 \
  > gpurun_out/r02_gates_ncu.log 2>&1
timeout 1500 ncu --set full --clock-control none \
  -k regex:"br1024|iks_b2|pks_kernel|br2q|cmux_chain1024|br_lat" -c 40 \
  -o gpurun_out/r02_mem python bench.py --config memory --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
  > gpurun_out/r02_mem_ncu.log 2>&1
tail -2 gpurun_out/r02_gates_ncu.log gpurun_out/r02_mem_ncu.log
