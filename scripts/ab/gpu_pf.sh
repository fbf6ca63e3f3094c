export BENCH_ARGS="--steps 10 --warmup 3"
bash scripts/ab.sh "OMCG_X=0" "OMCG_LIB_AB=$PWD/ab_libs/libomcg_pf.so" "OMCG_X=0" "OMCG_LIB_AB=$PWD/ab_libs/libomcg_pf.so"
