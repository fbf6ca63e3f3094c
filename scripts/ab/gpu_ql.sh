timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
BENCH_ARGS="--mode openmc-queueless" bash scripts/ab.sh "QL_FUSED=1"
BENCH_ARGS="--mode openmc-queueless --event-fusion 0" bash scripts/ab.sh "QL_FUSED=0"
BENCH_ARGS="--mode openmc-queueless --in-flight 250000" bash scripts/ab.sh "QL_FUSED=1_P1=250k"
bash scripts/ab.sh "QUEUED=1"
