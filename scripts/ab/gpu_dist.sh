nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
export BENCH_ARGS="--steps 10 --warmup 3"
bash scripts/ab.sh "OMCG_MOVE_CAP_AB=20" "OMCG_MOVE_CAP_AB=0" "OMCG_MOVE_CAP_AB=20" "OMCG_MOVE_CAP_AB=16"
