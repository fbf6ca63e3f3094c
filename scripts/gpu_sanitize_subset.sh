# Re-run of chosen compute-sanitizer cases: bash scripts/gpu_sanitize_subset.sh "tool:case ..."
mkdir -p gpurun_out/sanitize
S=/usr/local/cuda/bin/compute-sanitizer
for tc in $1; do
  tool=${tc%%:*}; c=${tc#*:}
  extra=""; [ "$tool" = racecheck ] && extra="--racecheck-report analysis"
  timeout 900 $S --tool $tool $extra --error-exitcode 9 --target-processes all python scripts/sanitize_case.py $c > gpurun_out/sanitize/${tool}_${c}.txt 2>&1
  rc=$?
  echo "$tool $c rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize/${tool}_${c}.txt | tr '\n' ' ') $(grep -E 'parity' gpurun_out/sanitize/${tool}_${c}.txt)" | tee -a gpurun_out/sanitize/summary_rerun.txt
done
