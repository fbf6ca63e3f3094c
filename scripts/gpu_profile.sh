# Profiling pass (round tag $1, default r02): ncu launch list over 2 C2 batches, then
# ncu --set full captures (source-correlated) of the hot kernels at large and mid-batch
# launches. Summarise here with: python scripts/ncu_summary.py <tag> gpurun_out
TAG=${1:-r02}
set -x
cat > /tmp/run2.py <<'PY'
import sys; sys.path.insert(0,'.')
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
r = P.run(p, n_particles=1000000, n_batches=2, n_inactive=1).result
print("FoM", r.fom)
PY
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/launches.csv python /tmp/run2.py > /dev/null 2>&1
for k in k_move:0:big k_move:30:mid k_xs_fuel_fused:0:big k_xs_fuel_fused:12:mid k_collide:3:big k_tail_warp:0:all; do
  name=${k%%:*}; rest=${k#*:}; skip=${rest%%:*}; lab=${rest##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${name}\$" -s $skip -c 1 -o gpurun_out/${TAG}_${name}@${lab} python /tmp/run2.py > gpurun_out/ncu_${name}_${lab}.log 2>&1; tail -1 gpurun_out/ncu_${name}_${lab}.log
done
ls -la gpurun_out/*.ncu-rep
timeout 300 python scripts/phase.py > gpurun_out/phase.txt 2>&1; cat gpurun_out/phase.txt
