O=gpurun_out/prod.log; : > $O
VSP_BR_PROD=1 VSP_BR_WARPS=7 timeout 600 python -m pytest tests/test_gates_gpu.py -x -q -k "tfhe80 or n630" > gpurun_out/prod_pytest.log 2>&1; tail -2 gpurun_out/prod_pytest.log >> $O
for cfg in "VSP_BR_PROD=1 VSP_BR_WARPS=7" "VSP_BR_WARPS=7" "VSP_BR_WARPS=8"; do
  env $cfg timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/prod.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/prod.json')); print('$cfg', d['value'], d['breakdown'], d['outputs_decrypt_correct'])" >> $O
done
cat $O
