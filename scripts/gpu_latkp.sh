set -x
python scripts/br_ab.py --gates 140 '{}' '{"VSP_LAT_KP": "1"}' '{"VSP_LAT_KP": "2"}' '{}' 2>&1 | grep step_ms
