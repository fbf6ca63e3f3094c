export BENCH_ARGS="--steps 10 --warmup 3"
L=$PWD/ab_libs
bash scripts/ab.sh "OMCG_X=0" "OMCG_LIB_AB=$L/libomcg_B32.so" "OMCG_LIB_AB=$L/libomcg_B128.so" "OMCG_LIB_AB=$L/libomcg_B256.so" "OMCG_X=0" "OMCG_LIB_AB=$L/libomcg_B32.so" "OMCG_LIB_AB=$L/libomcg_B128.so" "OMCG_LIB_AB=$L/libomcg_B256.so"
