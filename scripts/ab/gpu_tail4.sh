for t in 16384 10000 24000 16384; do BENCH_ARGS="--steps 10 --warmup 3 --tail $t" bash scripts/ab.sh "T=$t"; done
BENCH_ARGS="--steps 10 --warmup 3 --tasks 2" bash scripts/ab.sh "P5=2"
