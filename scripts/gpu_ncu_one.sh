# One source-correlated ncu --set full capture: bash scripts/gpu_ncu_one.sh <tag> <kernel> [skip]
TAG=$1; K=$2; SKIP=${3:-0}
cat > /tmp/run2.py <<'PY'
import sys; sys.path.insert(0,'.')
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
r = P.run(p, n_particles=1000000, n_batches=2, n_inactive=1).result
print("FoM", r.fom)
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${K}\$" -s $SKIP -c 1 -o gpurun_out/${TAG}_${K} python /tmp/run2.py > gpurun_out/ncu_${TAG}_${K}.log 2>&1; tail -1 gpurun_out/ncu_${TAG}_${K}.log
