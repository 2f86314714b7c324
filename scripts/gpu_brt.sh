# TMEM blind-rotation variant: parity under forced W, then bench per W.
O=gpurun_out/brt.log
: > $O
VSP_BR_TMEM=1 VSP_BR_WARPS=12 timeout 900 python -m pytest tests/test_gates_gpu.py -x -q > gpurun_out/brt_pytest.log 2>&1
tail -5 gpurun_out/brt_pytest.log >> $O
for W in 8 12; do
  VSP_BR_TMEM=1 VSP_BR_WARPS=$W timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/brt_$W.json 2> gpurun_out/brt_$W.err
  echo "tmem W=$W" >> $O; tail -2 gpurun_out/brt_$W.err >> $O; cat gpurun_out/brt_$W.json >> $O
done
VSP_BR_WARPS=8 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/brv2_8.json 2>&1
echo "v2 W=8" >> $O; cat gpurun_out/brv2_8.json >> $O
cat $O
