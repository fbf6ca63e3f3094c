# C5 at the reference's own budget: the unchanged campaigns/openmc campaign (256 evaluations,
# 4 workers) against bin/openmc on the GPU, then an EDP variant (96 evaluations).
rm -rf /tmp/c5_full_fom /tmp/c5_full_edp
timeout 2400 bash scripts/run_campaign.sh /tmp/c5_full_fom 256 4 fom > gpurun_out/c5_full_fom_report.txt 2>&1; cp /tmp/c5_full_fom/results.csv gpurun_out/c5_full_fom_results.csv; head -30 gpurun_out/c5_full_fom_report.txt
timeout 1200 bash scripts/run_campaign.sh /tmp/c5_full_edp 96 4 edp > gpurun_out/c5_full_edp_report.txt 2>&1; cp /tmp/c5_full_edp/results.csv gpurun_out/c5_full_edp_results.csv; head -30 gpurun_out/c5_full_edp_report.txt
