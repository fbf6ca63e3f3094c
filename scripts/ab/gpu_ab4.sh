set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
OMCG_XSF_WARPS=4 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "assembly or macro" 2>&1 | tail -2
bash scripts/ab.sh "OMCG_XSF_WARPS=8" "OMCG_XSF_WARPS=4" "OMCG_XSF_WARPS=8" "OMCG_XSF_WARPS=4"
