# Round pass on one B200: -m gpu suite + smoke, the bench line (3 runs), the
# C5 EDP campaign (256 evaluations, 1 worker) and its elapsed-vs-run-time check.
bash scripts/gpu_tests.sh
for i in 1 2 3; do timeout 600 python bench.py > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err; tail -1 gpurun_out/bench_$i.json | cut -c1-200; done
bash scripts/gpu_c5_edp.sh
