for i in 1 2 3 4 5 6; do python bench.py --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(f\"FoM {d['value']/1e6:.3f}M e2e {d['e2e']['value']/1e6:.3f}M clocks {d['clocks']}\")"; done
