O=gpurun_out/latprobe.log
: > $O
VSP_LAT_PROBE=1 timeout 300 python scripts/lat_ab.py 140 2>&1 | grep -m4 probe >> $O
cat $O
