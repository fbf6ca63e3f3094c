timeout 1200 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -2
bash scripts/ab.sh "FMA=1" "FMA=1"
