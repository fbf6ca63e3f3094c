# Source-correlated ncu --set full captures of the fuel lookup and the move kernel
# (one big launch each from a C2 batch) for per-instruction L1 analysis.
# usage: bash scripts/gpu_ncu_src.sh <tag>
TAG=${1:-r02b}
cat > /tmp/run2.py <<'PY'
import sys; sys.path.insert(0,'.')
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
r = P.run(p, n_particles=1000000, n_batches=2, n_inactive=1).result
print("FoM", r.fom)
PY
for k in k_xs_fuel_fused:0:big k_move:0:big; do
  name=${k%%:*}; rest=${k#*:}; skip=${rest%%:*}; lab=${rest##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${name}\$" -s $skip -c 1 -o gpurun_out/${TAG}_${name}@${lab} python /tmp/run2.py > gpurun_out/ncu_${name}_${lab}.log 2>&1; tail -1 gpurun_out/ncu_${name}_${lab}.log
done
ls -la gpurun_out/*.ncu-rep
