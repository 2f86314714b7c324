O=gpurun_out/br2ab.log
: > $O
VSP_BR2_MODE=1 timeout 300 python scripts/br2_ab.py 30 >> $O 2>&1
for S in 0 4 8 12; do echo "STG=$S" >> $O; VSP_BR2_STG=$S timeout 300 python scripts/br2_ab.py 30 >> $O 2>&1; done
VSP_BR2_PROBE=1 timeout 300 python scripts/br2_ab.py 30 2>&1 | grep -m4 "probe" >> $O
cat $O
