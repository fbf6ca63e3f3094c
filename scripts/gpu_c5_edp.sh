# C5 EDP variant (96 evaluations, 4 workers) on a fresh box (no profiler run before it).
rm -rf /tmp/c5_full_edp
timeout 1200 bash scripts/run_campaign.sh /tmp/c5_full_edp 96 4 edp > gpurun_out/c5_full_edp_report.txt 2>&1; cp /tmp/c5_full_edp/results.csv gpurun_out/c5_full_edp_results.csv; head -30 gpurun_out/c5_full_edp_report.txt
