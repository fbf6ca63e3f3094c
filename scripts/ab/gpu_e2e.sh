for i in 1 2 3; do OMCG_TRACE_INIT=1 python bench.py --steps 5 --warmup 2 --no-cpu-baseline 2>&1 | grep -E "omcg|value" | cut -c1-200; done
