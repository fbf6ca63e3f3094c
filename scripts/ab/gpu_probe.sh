set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5
python - <<PY
import sys; sys.path.insert(0,'.')
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
for prof in (False, True):
    r = P.run(p, n_particles=1000000, n_batches=7, n_inactive=2, profile=prof).result
    names=["xs_fuel","xs_nonfuel","adv","cross","coll","sort","refill","tail"]
    print(f"prof={prof} FoM={r.fom:.4e} t_active={r.t_active:.3f} iters={r.queue_iterations} launches={r.kernel_launches} tails={r.tail_launches} k={r.k_mean:.5f}",
          " ".join(f"{n}={r.prof_ms[i]/5:.1f}ms" for i,n in enumerate(names)) if prof else "")
PY
