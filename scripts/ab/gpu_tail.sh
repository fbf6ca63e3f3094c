for t in 8192 16384 32768; do BENCH_ARGS="--tail $t" bash scripts/ab.sh "TAIL=$t"; done
