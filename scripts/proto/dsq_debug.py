import sys, traceback
sys.path.insert(0, ".")
import numpy as np
import paper_2402_09222_b200 as P
for kind, n, inf, tail, sort in (("pincell", 6000, 1500, 300, 0), ("pincell", 4000, 4000, 0, -1)):
    p = P.Problem(kind)
    for ds in (0, 1):
        try:
            out = P.run(p, n_particles=n, n_batches=1, n_inactive=0, seed=1, particles_in_flight=inf,
                        tail_threshold=tail, sort_threshold=sort, trace_queues=True, device_schedule=ds)
            t = np.asarray(out.queue_trace).reshape(-1, 3)
            print(kind, n, "ds", ds, "iters", len(t), "k", out.result.k_coll[0], "seq", "".join("FXMCCT"[int(x)] if x < 6 else "?" for x in t[:60, 0]), flush=True)
        except Exception as e:
            print(kind, n, "ds", ds, "ERROR", e, flush=True)
