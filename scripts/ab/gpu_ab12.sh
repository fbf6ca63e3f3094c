timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -1
bash scripts/ab.sh "OMCG_TAIL_REGS=0" "OMCG_TAIL_REGS=64"
