OMCG_MOVE_POOL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
bash scripts/ab.sh "OMCG_MOVE_POOL=1" "OMCG_MOVE_POOL=0"
