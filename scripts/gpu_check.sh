# Quick state check on one B200: -m gpu suite + smoke + one bench line.
bash scripts/gpu_tests.sh
timeout 600 python bench.py > gpurun_out/bench_1.json 2> gpurun_out/bench_1.err; tail -1 gpurun_out/bench_1.json
