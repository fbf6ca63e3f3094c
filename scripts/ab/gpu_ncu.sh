# ncu evidence for profiles/: launch list (2 batches of C2) + full sets of the hot kernels
set -x
cat > /tmp/run2.py <<'PY'
import sys; sys.path.insert(0,'.')
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
r = P.run(p, n_particles=1000000, n_batches=2, n_inactive=1).result
print("FoM", r.fom)
PY
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/launches.csv python /tmp/run2.py > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log
for k in k_xs_fuel:30 k_advance:60 k_collide:40 k_xs_nonfuel:40 k_cross:40; do
  name=${k%%:*}; skip=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${name}\$" -s $skip -c 1 -o gpurun_out/r01_${name} python /tmp/run2.py > gpurun_out/ncu_${name}.log 2>&1; tail -1 gpurun_out/ncu_${name}.log
done
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
