export BENCH_ARGS="--steps 10 --warmup 3"
bash scripts/ab.sh "OMCG_XSF_WARPS=4" "OMCG_XSF_WARPS=9" "OMCG_XSF_WARPS=10" "OMCG_XSF_WARPS=4" "OMCG_XSF_WARPS=9"
