# Final round-2 evidence (publish read-back build): -m gpu suite + smoke, 3 bench lines,
# the reference arm, ncu launch list + --set full captures, and a compute-sanitizer subset
# over the queued paths the read-back change touches.
bash scripts/gpu_tests.sh
for i in 1 2 3; do timeout 600 python bench.py > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err; tail -1 gpurun_out/bench_$i.json | cut -c1-160; done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.json | cut -c1-200
bash scripts/gpu_profile.sh ${1:-r02g}
bash scripts/gpu_sanitize_subset.sh "memcheck:pincell_queued memcheck:assembly_queued memcheck:pincell_cap1_p5 memcheck:pincell_2rank racecheck:assembly_queued racecheck:pincell_cap1_p5 synccheck:assembly_queued synccheck:pincell_2rank initcheck:assembly_queued initcheck:pincell_queued"
