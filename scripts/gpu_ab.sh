# A/B of a tuning knob: parity under the knob, then bench with and without it.
# usage: bash scripts/gpu_ab.sh "VSP_KNOB=1"
O=gpurun_out/ab.log; : > $O
env $1 timeout 600 python -m pytest tests/test_gates_gpu.py -x -q > gpurun_out/ab_pytest.log 2>&1; tail -2 gpurun_out/ab_pytest.log >> $O
for cfg in "$1" "VSP_NONE=1" "$1"; do
  env $cfg timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$cfg', d['value'], d['breakdown'], d['outputs_decrypt_correct'])" >> $O
  env $cfg timeout 300 python bench.py --gates 16384 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('  16k $cfg', d['value'], d['breakdown'])" >> $O
done
cat $O
