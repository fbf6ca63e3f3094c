# compute-sanitizer memcheck / racecheck / synccheck / initcheck over the sanitize cases.
# Logs: gpurun_out/sanitize/<tool>_<case>.txt; summary: gpurun_out/sanitize/summary.txt
mkdir -p gpurun_out/sanitize
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for c in pincell_queued pincell_queueless pincell_unfused pincell_cap1_p5 pincell_2rank pincell_nccl1 assembly_queued assembly_queueless assembly_unfused pincell_dsq assembly_dsq; do
    extra=""
    [ "$tool" = racecheck ] && extra="--racecheck-report analysis"
    timeout 420 $S --tool $tool $extra --error-exitcode 9 --target-processes all python scripts/sanitize_case.py $c > gpurun_out/sanitize/${tool}_${c}.txt 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize/${tool}_${c}.txt | tr '\n' ' ') $(grep -E 'parity' gpurun_out/sanitize/${tool}_${c}.txt)" >> gpurun_out/sanitize/summary.txt
  done
done
cat gpurun_out/sanitize/summary.txt
