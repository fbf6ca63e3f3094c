set -x
bash scripts/ab.sh "OMCG_MOVE_VOTE=1" "OMCG_MOVE_VOTE=0"
cat > /tmp/run2.py <<'PY'
import sys; sys.path.insert(0,'.')
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
r = P.run(p, n_particles=1000000, n_batches=2, n_inactive=1).result
print("FoM", r.fom)
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_move$" -s 8 -c 1 -o gpurun_out/mv_k_move python /tmp/run2.py > gpurun_out/ncu_k_move.log 2>&1; tail -1 gpurun_out/ncu_k_move.log
OMCG_MOVE_VOTE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_move_vote$" -s 8 -c 1 -o gpurun_out/mv_k_move_vote python /tmp/run2.py > gpurun_out/ncu_k_move_vote.log 2>&1; tail -1 gpurun_out/ncu_k_move_vote.log
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/launches_mv.csv python /tmp/run2.py > /dev/null 2>&1
