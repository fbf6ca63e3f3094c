set -x
# C4: full core on 1 GPU (vacuum boundaries, 37 assemblies + water reflector)
OMCG_PROBLEM=core OMCG_PARTICLES=2000000 OMCG_BATCHES=6 OMCG_INACTIVE=2 timeout 600 bin/openmc --event -i 2000000 -b 4000 -m 20000 > gpurun_out/c4_core.out 2> gpurun_out/c4_core.err; tail -3 gpurun_out/c4_core.err; cat gpurun_out/c4_core.out
# C3 sweep
timeout 1500 python scripts/sweep_c3.py gpurun_out/c3_sweep.json > gpurun_out/c3.log 2>&1; tail -2 gpurun_out/c3.log
# C5: unchanged campaign, 4 workers sharing the GPU via the flock lease, FoM then EDP
rm -rf /tmp/camp_fom /tmp/camp_edp
timeout 1800 bash scripts/run_campaign.sh /tmp/camp_fom 48 4 fom > gpurun_out/c5_fom_report.txt 2>&1; cp /tmp/camp_fom/results.csv gpurun_out/c5_fom_results.csv; cat gpurun_out/c5_fom_report.txt | head -20
timeout 1200 bash scripts/run_campaign.sh /tmp/camp_edp 24 4 edp > gpurun_out/c5_edp_report.txt 2>&1; cp /tmp/camp_edp/results.csv gpurun_out/c5_edp_results.csv; head -20 gpurun_out/c5_edp_report.txt
