BENCH_ARGS="--tasks 2" bash scripts/ab.sh "P5=2"
BENCH_ARGS="--tasks 4" bash scripts/ab.sh "P5=4"
bash scripts/ab.sh "P5=1"
