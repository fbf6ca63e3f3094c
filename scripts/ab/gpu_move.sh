set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -6
bash scripts/ab.sh "OMCG_XS_FUSED=1" "OMCG_MOVE_OCC=1" "OMCG_TRACE_INIT=1"
python bench.py --steps 5 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['kernel_share'], d['queue_iterations'], d['gpu_launches'])"
