# Quick A/B of the current build: 4096-gate batch + 140-gate narrow level (hash + times),
# then the gate / production parity tests.
set -x
python scripts/br_ab.py '{}' 2>&1 | grep step_ms
python scripts/br_ab.py --gates 140 '{}' 2>&1 | grep step_ms
timeout 900 python -m pytest tests/test_gates_gpu.py tests/test_parity_prod_gpu.py -x -q 2>&1 | tail -3
