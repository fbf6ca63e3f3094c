for sh in 2 3 4; do OMCG_XSF_SHAPE=$sh timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "assembly or macro" 2>&1 | tail -1; done
bash scripts/ab.sh "OMCG_XSF_SHAPE=0" "OMCG_XSF_SHAPE=1" "OMCG_XSF_SHAPE=2" "OMCG_XSF_SHAPE=3" "OMCG_XSF_SHAPE=4"
