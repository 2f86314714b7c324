set -x
python scripts/br_ab.py --gates 140 '{"VSP_IKS_SPLIT": "1"}' '{"VSP_IKS_SPLIT": "2"}' '{"VSP_IKS_SPLIT": "4"}' '{"VSP_IKS_SPLIT": "8"}' '{"VSP_IKS_SPLIT": "16"}' '{"VSP_IKS_SPLIT": "24"}' 2>&1 | grep step_ms
python scripts/br_ab.py --gates 64 '{"VSP_IKS_SPLIT": "1"}' '{"VSP_IKS_SPLIT": "8"}' '{"VSP_IKS_SPLIT": "16"}' 2>&1 | grep step_ms
python scripts/br_ab.py '{"VSP_IKS_SPLIT": "1"}' '{"VSP_IKS_SPLIT": "2"}' '{"VSP_IKS_SPLIT": "4"}' 2>&1 | grep step_ms
