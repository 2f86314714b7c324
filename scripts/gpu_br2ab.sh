O=gpurun_out/br2ab.log
: > $O
VSP_BR2_EXT=0 timeout 300 python scripts/br2_ab.py 30 >> $O 2>&1
timeout 300 python scripts/br2_ab.py 30 >> $O 2>&1
VSP_BR2_PROBE=1 timeout 300 python scripts/br2_ab.py 30 2>&1 | grep -m8 "probe" >> $O
cat $O
