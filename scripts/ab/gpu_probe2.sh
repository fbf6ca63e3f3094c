python - <<PY
import sys; sys.path.insert(0,'.')
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
for kw in [dict(), dict(tasks_per_gpu=2), dict(tasks_per_gpu=2, particles_in_flight=500000), dict(particles_in_flight=250000), dict(particles_in_flight=2000000, n_particles=2000000), dict(n_bins=100000), dict(n_bins=100), dict(sort_threshold=-1), dict(mode="openmc-queueless")]:
    args = dict(n_particles=1000000, n_batches=7, n_inactive=2); args.update(kw)
    r = P.run(p, **args).result
    print(f"{kw} FoM={r.fom:.4e} t_active={r.t_active:.3f} iters={r.queue_iterations} launches={r.kernel_launches} k={r.k_mean:.5f}")
PY
