cat > /tmp/run2.py <<'PY'
import sys; sys.path.insert(0,'.')
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
r = P.run(p, n_particles=1000000, n_batches=2, n_inactive=1).result
print("FoM", r.fom)
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_move\$" -s 8 -c 1 -o gpurun_out/r01_k_move python /tmp/run2.py > gpurun_out/ncu_mv.log 2>&1; tail -1 gpurun_out/ncu_mv.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_xs_fuel_fused\$" -s 10 -c 1 -o gpurun_out/r01_k_xs_fuel_fused python /tmp/run2.py > gpurun_out/ncu_xs.log 2>&1; tail -1 gpurun_out/ncu_xs.log
