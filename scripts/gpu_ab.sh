# A/B on one box: parity subset (-k filter $1), then interleaved C2 FoM of the in-tree
# build ("head") against ab_libs/<variant> builds: bash scripts/gpu_ab.sh <pytest -k expr> <rounds> variant...
K=$1; shift
if [ "$K" != "-" ]; then timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "$K" 2>&1 | tail -3; fi
bash scripts/ab_run.sh "$@"
