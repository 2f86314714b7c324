O=gpurun_out/latq.log
: > $O
timeout 300 python scripts/lat_ab.py 140 >> $O 2>&1
timeout 300 python scripts/lat_ab.py 74 >> $O 2>&1
cat $O
