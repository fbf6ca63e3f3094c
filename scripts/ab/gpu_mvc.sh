export BENCH_ARGS="--steps 10 --warmup 3"
L=$PWD/ab_libs
bash scripts/ab.sh "OMCG_LIB_AB=$L/libomcg_C16.so" "OMCG_LIB_AB=$L/libomcg_C8.so" "OMCG_LIB_AB=$L/libomcg_C12.so" "OMCG_LIB_AB=$L/libomcg_C24.so" "OMCG_LIB_AB=$L/libomcg_C16.so OMCG_MOVE_CAP_AB=28" "OMCG_LIB_AB=$L/libomcg_C16.so OMCG_MOVE_CAP_AB=14" "OMCG_LIB_AB=$L/libomcg_C16.so" "OMCG_LIB_AB=$L/libomcg_C8.so" "OMCG_LIB_AB=$L/libomcg_C12.so"
