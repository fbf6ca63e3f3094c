# A/B of env switches on the C2 bench (short: 2 inactive + 5 active batches).
# usage: bash scripts/ab.sh "ENV=.. ENV2=.." "ENV=.." ...   (BENCH_ARGS: extra bench.py flags)
for v in "$@"; do
  r=$(env $v timeout 600 python bench.py ${BENCH_ARGS:---steps 5 --warmup 2} --no-cpu-baseline 2>/dev/null | tail -1)
  python - "$v" "$r" <<'PY'
import json,sys
try:
    d=json.loads(sys.argv[2]); print(f"{sys.argv[1]:40s} FoM {d['value']/1e6:7.3f}M  e2e {d['e2e']['value']/1e6:6.3f}M  init {d['t_init_s']:.3f}s  xs-frac {d['roofline']['frac']}  iters {d['queue_iterations']}")
except Exception as e: print(sys.argv[1], "FAILED", sys.argv[2][:300])
PY
done
