timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -1
bash scripts/ab.sh OMCG_PIN_LIBRARY=1 OMCG_PIN_LIBRARY=0 OMCG_PIN_LIBRARY=1 OMCG_PIN_LIBRARY=0
for v in 1 0 1 0; do OMCG_PIN_LIBRARY=$v OMCG_PARTICLES=1000000 OMCG_BATCHES=3 OMCG_INACTIVE=1 bin/openmc --event -i 1000000 -b 4000 -m 20000 2>&1 | grep -oE "init [0-9.]+s|wall [0-9.]+s" | tr '\n' ' '; echo " pin=$v"; done
