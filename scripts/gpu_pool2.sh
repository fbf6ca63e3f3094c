cat > /tmp/run2.py <<'PY'
import sys; sys.path.insert(0,'.')
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
r = P.run(p, n_particles=1000000, n_batches=2, n_inactive=1).result
print("FoM", r.fom)
PY
OMCG_MOVE_POOL=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_move_pool" -s 8 -c 1 -o gpurun_out/pool_k_move_pool python /tmp/run2.py > gpurun_out/ncu_pool.log 2>&1; tail -1 gpurun_out/ncu_pool.log
