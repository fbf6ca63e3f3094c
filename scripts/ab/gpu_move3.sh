set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
bash scripts/ab.sh "OMCG_MOVE_VARIANT=0" "OMCG_MOVE_VARIANT=1" "OMCG_MOVE_VARIANT=2" "OMCG_MOVE_VARIANT=3"
BENCH_ARGS="--event-fusion 0" bash scripts/ab.sh "CLASSIC=1"
