timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
export BENCH_ARGS="--steps 10 --warmup 3"
bash scripts/ab.sh "OMCG_LIB_AB=$PWD/ab_libs/libomcg_base.so" "OMCG_X=0" "OMCG_LIB_AB=$PWD/ab_libs/libomcg_base.so" "OMCG_X=0"
python scripts/phase.py 2>&1 | grep "tail:"
