set -x
timeout 900 python scripts/br_occupancy.py 2>&1 | tail -15
