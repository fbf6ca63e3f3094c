timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -1
bash scripts/ab.sh "OMCG_MOVE_VARIANT=0" "OMCG_MOVE_VARIANT=6"
for t in 0 4096 65536; do BENCH_ARGS="--tail $t" bash scripts/ab.sh "TAIL=$t"; done
