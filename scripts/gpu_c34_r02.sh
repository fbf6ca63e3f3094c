# C4 (full core, 1 GPU, bin/openmc) and the C3 sweep at the current build.
mkdir -p gpurun_out/r02
OMCG_PROBLEM=core OMCG_PARTICLES=2000000 OMCG_BATCHES=6 OMCG_INACTIVE=2 timeout 600 bin/openmc --event -i 2000000 -b 4000 -m 20000 > gpurun_out/r02/c4_core.out 2> gpurun_out/r02/c4_core.err; tail -3 gpurun_out/r02/c4_core.err; cat gpurun_out/r02/c4_core.out
timeout 1500 python scripts/sweep_c3.py gpurun_out/r02/c3_sweep.json > gpurun_out/r02/c3.log 2>&1; tail -2 gpurun_out/r02/c3.log
