export BENCH_ARGS="--steps 10 --warmup 3"
bash scripts/ab.sh "OMCG_TAIL_BLOCK=128" "OMCG_TAIL_BLOCK=32" "OMCG_TAIL_BLOCK=64" "OMCG_TAIL_BLOCK=128"
for t in 4096 8192 32768; do BENCH_ARGS="--steps 10 --warmup 3 --tail $t" bash scripts/ab.sh "OMCG_TAIL_BLOCK=32"; done
