timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -1
bash scripts/ab.sh "SEL=binary" "SEL=binary"
cat > /tmp/run2.py <<'PY'
import sys; sys.path.insert(0,'.')
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
r = P.run(p, n_particles=1000000, n_batches=2, n_inactive=1).result
print("FoM", r.fom)
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_xs_fuel_fused4\$" -s 10 -c 1 -o gpurun_out/r01_k_xs_fuel_fused4 python /tmp/run2.py > gpurun_out/ncu_xsf4.log 2>&1; tail -1 gpurun_out/ncu_xsf4.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_move\$" -s 8 -c 1 -o gpurun_out/r01_k_move python /tmp/run2.py > gpurun_out/ncu_mv.log 2>&1; tail -1 gpurun_out/ncu_mv.log
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/launches.csv python /tmp/run2.py > /dev/null 2>&1
