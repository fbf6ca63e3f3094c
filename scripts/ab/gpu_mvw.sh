export BENCH_ARGS="--steps 10 --warmup 3"
L=$PWD/ab_libs
bash scripts/ab.sh "OMCG_X=0" "OMCG_LIB_AB=$L/libomcg_W2.so" "OMCG_LIB_AB=$L/libomcg_W8.so" "OMCG_LIB_AB=$L/libomcg_C16.so" "OMCG_X=0" "OMCG_LIB_AB=$L/libomcg_W2.so" "OMCG_LIB_AB=$L/libomcg_W8.so" "OMCG_LIB_AB=$L/libomcg_C16.so"
