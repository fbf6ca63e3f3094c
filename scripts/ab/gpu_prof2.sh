set -x
python bench.py --steps 5 --warmup 2 --no-cpu-baseline 2>/dev/null > gpurun_out/bench_short.json; python -c "import json; d=json.load(open('gpurun_out/bench_short.json')); print(d['value'], d['kernel_share'], d['queue_iterations'], d['gpu_launches'])"
cat > /tmp/run2.py <<'PY'
import sys; sys.path.insert(0,'.')
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
r = P.run(p, n_particles=1000000, n_batches=2, n_inactive=1).result
print("FoM", r.fom)
PY
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/launches.csv python /tmp/run2.py > /dev/null 2>&1
for k in k_move:8 k_xs_fuel_fused:10 k_collide:8; do
  name=${k%%:*}; skip=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${name}\$" -s $skip -c 1 -o gpurun_out/r01_${name} python /tmp/run2.py > gpurun_out/ncu_${name}.log 2>&1; tail -1 gpurun_out/ncu_${name}.log
done
