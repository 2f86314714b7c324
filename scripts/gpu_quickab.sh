# Quick A/B: narrow level, headline bench line (no CPU baseline), headline parity test.
O=gpurun_out/quickab.log
: > $O
timeout 300 python scripts/lat_ab.py 140 >> $O 2>&1
timeout 600 python bench.py --headline-only --no-cpu-baseline > gpurun_out/bench_h.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/bench_h.json').read().strip().splitlines()[-1]);print('gates/s',d['value'],'e2e',d['e2e']['value'],'frac',d['roofline']['frac'],d['breakdown'])" >> $O
timeout 900 python -m pytest -q -x tests/test_parity_prod_gpu.py -k "headline or all_gate_kinds or cmux_chain or rom_read" 2>&1 | tail -2 >> $O
cat $O
