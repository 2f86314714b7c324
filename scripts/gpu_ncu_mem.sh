# ncu --set full of the memory-access kernels (write-bar br1024, iks_b2, pks, br2q, CMUX
# chains, br_lat) on one ROM read + RAM cycle at 512 B (bench.py --config memory), 1 GPU.
set -x
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"br1024|iks_b2|pks_kernel|br2q|cmux_chain1024|br_lat" -c 14 \
  -o gpurun_out/r02_mem python bench.py --config memory --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
  > gpurun_out/r02_mem_ncu.log 2>&1
tail -3 gpurun_out/r02_mem_ncu.log
