# Round-2 evidence after the branch-free divisions: -m gpu suite + smoke, ncu launch
# list and --set full captures (scripts/gpu_profile.sh), 3 bench lines, the reference arm.
bash scripts/gpu_tests.sh
bash scripts/gpu_profile.sh ${1:-r02f}
for i in 1 2 3; do timeout 600 python bench.py > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err; tail -1 gpurun_out/bench_$i.json | cut -c1-160; done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.json | cut -c1-200
