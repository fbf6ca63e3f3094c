# Three default bench runs on one box (the committed bench line is the median-e2e run).
for i in 1 2 3; do timeout 900 python bench.py > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err; tail -c 300 gpurun_out/bench_$i.json; echo; done
