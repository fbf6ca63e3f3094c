# C5 EDP campaign at the reference's budget (256 evaluations) with workers <= leasable GPUs
# (1 worker on a 1-GPU box: no evaluation waits for another's GPU lease, so the harness's
# elapsed is the evaluation's own run time), metrics.txt energy over the whole evaluation.
rm -rf /tmp/c5_edp
W=${C5_WORKERS:-1}
timeout 2400 bash scripts/run_campaign.sh /tmp/c5_edp 256 "$W" edp > gpurun_out/c5_edp_report.txt 2>&1
cp /tmp/c5_edp/results.csv gpurun_out/c5_edp_results.csv
python scripts/c5_elapsed_check.py /tmp/c5_edp > gpurun_out/c5_edp_elapsed.json
head -30 gpurun_out/c5_edp_report.txt; tail -12 gpurun_out/c5_edp_elapsed.json
