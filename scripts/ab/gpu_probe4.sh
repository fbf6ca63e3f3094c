python - <<PY
import sys; sys.path.insert(0,'.')
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
for kw in [dict(tail_threshold=16384), dict(tail_threshold=65536), dict(tail_threshold=131072), dict(tail_threshold=262144), dict(tasks_per_gpu=2), dict(tasks_per_gpu=2, tail_threshold=65536)]:
    args = dict(n_particles=1000000, n_batches=7, n_inactive=2); args.update(kw)
    r = P.run(p, **args).result
    print(f"{kw} FoM={r.fom:.4e} t_active={r.t_active:.3f} iters={r.queue_iterations} launches={r.kernel_launches} k={r.k_mean:.6f}")
PY
