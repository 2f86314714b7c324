# A/B of br_lat variants: per-level time at 140 and 74 tasks, hash-compared outputs.
O=gpurun_out/latab.log
: > $O
for T in 140 74; do
  for E in 0 1 2; do
    echo "EXT=$E" >> $O
    VSP_LAT_EXT=$E timeout 300 python scripts/lat_ab.py $T >> $O 2>&1
  done
done
cat $O
