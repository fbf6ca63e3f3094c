import sys
sys.path.insert(0, ".")
import paper_2402_09222_b200 as P
p = P.Problem("pincell")
out = P.run(p, n_particles=6000, n_batches=1, n_inactive=0, seed=1, particles_in_flight=1500,
            tail_threshold=300, sort_threshold=0, trace_queues=True, device_schedule=1)
print("ok", out.result.k_coll[0])
