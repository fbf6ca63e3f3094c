# EDP methodology probe: a 12-evaluation EDP campaign (1 worker) with the tuner's CPU
# use sampled, then the first 6 evaluations re-run standalone (FoM + energy lines kept).
rm -rf /tmp/c5p; mkdir -p gpurun_out/r02
export OMCG_TRACE_INIT=1
( timeout 900 bash scripts/run_campaign.sh /tmp/c5p 12 1 edp > gpurun_out/r02/edp_probe_report.txt 2>&1 ) &
CP=$!
for i in $(seq 1 60); do sleep 1; ps -eo pid,pcpu,nlwp,comm --sort=-pcpu | head -5 | tr '\n' '|'; echo; done > gpurun_out/r02/edp_probe_ps.txt
wait $CP
nproc >> gpurun_out/r02/edp_probe_ps.txt
python scripts/c5_elapsed_check.py /tmp/c5p --standalone 6 > gpurun_out/r02/edp_probe_elapsed.json
for e in 0 1 2 3 4; do echo "== eval $e"; cat /tmp/c5p/evals/$e/launcher; cat /tmp/c5p/evals/$e/stderr.log; tail -2 /tmp/c5p/evals/$e/stdout.log; done > gpurun_out/r02/edp_probe_evals.txt
python - <<'PY'
import json; d=json.load(open('gpurun_out/r02/edp_probe_elapsed.json'))
print(json.dumps(d['summary'], indent=1))
for s in d['standalone']: print(s)
PY
