# Round-2 ncu evidence (1 GPU), exported to CSV on the box (reports are too big to copy):
# (1) the headline gate batch (br1024 W=8 whole waves, W=4 remainder, forked + final iks_b2)
# (2) a 140-gate narrow level (br_lat, iks_b2)
# (3) one ROM read + RAM cycle (br2q, pks_kernel, CMUX chains, key switches, br_lat,
#     write-bar br1024)
set -x
O=gpurun_out/ncu_r02
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"br1024|iks_b2" \
  --launch-skip 4 -c 4 -o /tmp/r02_gates python scripts/br_once.py 4096 > $O/gates.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"br_lat|iks_b2|iks_init" \
  --launch-skip 3 -c 3 -o /tmp/r02_lat python scripts/br_once.py 140 > $O/lat.log 2>&1
timeout 1500 ncu --set full --clock-control none \
  -k regex:"br1024|iks_b2|pks_kernel|br2q|cmux_chain1024|br_lat" -c 40 \
  -o /tmp/r02_mem python bench.py --config memory --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
  > $O/mem.log 2>&1
for r in gates lat mem; do
  ncu -i /tmp/r02_$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null
done
ncu -i /tmp/r02_gates.ncu-rep --page source --csv --print-source cuda,sass -k regex:"br1024_kernel<8" > $O/gates_br8_source.csv 2>/dev/null
ncu -i /tmp/r02_lat.ncu-rep --page source --csv --print-source cuda,sass -k regex:"br_lat" > $O/lat_source.csv 2>/dev/null
gzip -f $O/*.csv
ls -la $O
