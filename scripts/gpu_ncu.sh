set -x
export OMCG_NCU=1
cat > /tmp/run2.py <<'PY'
import sys; sys.path.insert(0,'.')
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
r = P.run(p, n_particles=1000000, n_batches=2, n_inactive=1).result
print("FoM", r.fom)
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_xs_fuel -s 40 -c 1 -o gpurun_out/prof_xs_fuel2 python /tmp/run2.py > gpurun_out/ncu_xs.log 2>&1; tail -2 gpurun_out/ncu_xs.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_collide -s 40 -c 1 -o gpurun_out/prof_collide2 python /tmp/run2.py > gpurun_out/ncu_coll.log 2>&1; tail -2 gpurun_out/ncu_coll.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tail -s 1 -c 1 -o gpurun_out/prof_tail python /tmp/run2.py > gpurun_out/ncu_adv.log 2>&1; tail -2 gpurun_out/ncu_adv.log
ls -la gpurun_out/
