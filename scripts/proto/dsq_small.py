import sys
sys.path.insert(0, ".")
import paper_2402_09222_b200 as P
p = P.Problem("pincell")
for ds in (0, 1):
    out = P.run(p, n_particles=600, n_batches=1, n_inactive=0, seed=1, particles_in_flight=600,
                tail_threshold=20, sort_threshold=-1, trace_queues=True, device_schedule=ds)
    import numpy as np
    t = np.asarray(out.queue_trace).reshape(-1, 3)
    print("ds", ds, "trace", [(int(a), int(b)) for a, b, _ in t[:12]], flush=True)
