import sys; sys.path.insert(0, '.')
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
r = P.run(p, n_particles=1000000, n_batches=2, n_inactive=1, profile=1).result
print("t_active", r.t_active)
