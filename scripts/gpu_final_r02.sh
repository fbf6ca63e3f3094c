# Round-2 evidence for the current build: -m gpu suite + smoke, ncu launch list and
# --set full captures (scripts/gpu_profile.sh), then 3 bench lines.
bash scripts/gpu_tests.sh
bash scripts/gpu_profile.sh ${1:-r02c}
for i in 1 2 3; do timeout 600 python bench.py > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err; tail -1 gpurun_out/bench_$i.json | cut -c1-160; done
