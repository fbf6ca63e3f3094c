set -x
OMCG_MOVE_VARIANT=4 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
bash scripts/ab.sh "OMCG_XS_DEEP=0" "OMCG_XS_DEEP=1" "OMCG_XS_DEEP=2" "OMCG_MOVE_VARIANT=4" "OMCG_MOVE_VARIANT=5" "OMCG_MOVE_VARIANT=0"
