set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -4
bash scripts/ab.sh "OMCG_XS_FUSED=1" "OMCG_XS_FUSED=0" "OMCG_XS_FUSED=1 OMCG_TRACE_INIT=1"
OMCG_TRACE_INIT=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | grep "omcg init"
