set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
OMCG_MOVE_CAP=16 timeout 900 python -m pytest tests -m gpu -x -q -k "not queue_trace" 2>&1 | tail -3
bash scripts/ab.sh "OMCG_MOVE_CAP=0" "OMCG_MOVE_CAP=8" "OMCG_MOVE_CAP=16" "OMCG_MOVE_CAP=32" "OMCG_MOVE_CAP=64" "OMCG_MOVE_CAP=0" "OMCG_MOVE_CAP=12" "OMCG_MOVE_CAP=24"
