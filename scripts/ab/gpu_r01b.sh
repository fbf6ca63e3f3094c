# Round-1 re-entry evidence pass: GPU parity, smoke, bench, launch list, ncu full of the hot kernels.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/ -q -m gpu 2>&1 | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
cat > /tmp/run2.py <<'PY'
import sys; sys.path.insert(0,'.')
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
r = P.run(p, n_particles=1000000, n_batches=2, n_inactive=1).result
print("FoM", r.fom)
PY
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/launches.csv python /tmp/run2.py > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log
for k in k_xs_fuel_seg:30 k_advance:60 k_collide:40 k_xs_nonfuel:40 k_cross:40 k_tail_warp:0; do
  name=${k%%:*}; skip=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${name}\$" -s $skip -c 1 -o gpurun_out/r01_${name} python /tmp/run2.py > gpurun_out/ncu_${name}.log 2>&1; tail -1 gpurun_out/ncu_${name}.log
done
