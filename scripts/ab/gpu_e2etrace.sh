for i in 1 2 3 4 5 6; do OMCG_TRACE_INIT=1 python bench.py --no-cpu-baseline --steps 10 --warmup 3 2> /tmp/tr.err | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(f\"FoM {d['value']/1e6:.3f}M e2e {d['e2e']['value']/1e6:.3f}M\")"; python - <<'PY'
import re
L=open('/tmp/tr.err').read().split('[omcg run] energy meter started')
# second call = timed one
if len(L) > 2:
    seg = '[omcg run] energy meter started' + L[2]
    print('   ', ' | '.join(l.replace('[omcg run] ','').strip() for l in seg.splitlines() if l.startswith('[omcg run]')))
PY
done
