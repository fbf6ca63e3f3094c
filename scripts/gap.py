"""Kernel time vs batch time: sum of per-launch CUDA-event times (profile=1) against the active time."""
import sys; sys.path.insert(0, '.')
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
for prof in (0, 1):
    r = P.run(p, n_particles=1000000, n_batches=5, n_inactive=1, profile=prof).result
    k = sum(r.prof_ms[i] for i in range(8))
    print(f"profile={prof} t_active/batch {1e3 * r.t_active / 4:.2f} ms  kernels/batch {k / 4:.2f} ms  "
          f"iterations/batch {r.queue_iterations / 5:.0f}  FoM {r.fom / 1e6:.3f}M")
