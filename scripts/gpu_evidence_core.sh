# Evidence pass without the C5 campaigns: GPU tests, smoke, bench, ncu launch list + full captures, C4, C3.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests/ -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json | cut -c1-400
cat > /tmp/run2.py <<'PY'
import sys; sys.path.insert(0,'.')
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
r = P.run(p, n_particles=1000000, n_batches=2, n_inactive=1).result
print("FoM", r.fom)
PY
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/launches.csv python /tmp/run2.py > /dev/null 2>&1
for k in k_move:8 k_xs_fuel_fused:10 k_collide:8 k_tail_warp:0 k_sort_scatter:6 k_sort_hist:6; do
  name=${k%%:*}; skip=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${name}\$" -s $skip -c 1 -o gpurun_out/r01_${name} python /tmp/run2.py > gpurun_out/ncu_${name}.log 2>&1; tail -1 gpurun_out/ncu_${name}.log
done
OMCG_PROBLEM=core OMCG_PARTICLES=2000000 OMCG_BATCHES=6 OMCG_INACTIVE=2 timeout 600 bin/openmc --event -i 2000000 -b 4000 -m 20000 > gpurun_out/c4_core.out 2> gpurun_out/c4_core.err; tail -3 gpurun_out/c4_core.err; cat gpurun_out/c4_core.out
timeout 1500 python scripts/sweep_c3.py gpurun_out/c3_sweep.json > gpurun_out/c3.log 2>&1; tail -1 gpurun_out/c3.log
