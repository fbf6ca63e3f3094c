import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np
import oracle as O
import paper_2402_09222_b200 as P
kind, n, inflight, tail, sort = P.PINCELL, 6000, 1500, 300, 0
o = O.Problem(kind, 1234, 4000)
want = o.queue_trace(n, inflight, tail, seed=1, event_fusion=True, move_cap=20)
p = P.Problem(kind, 1234)
got = P.run(p, n_particles=n, n_batches=1, n_inactive=0, seed=1, particles_in_flight=inflight,
            tail_threshold=tail, sort_threshold=sort, trace_queues=True, event_fusion=1).queue_trace
print(got.shape, want.shape)
for i in range(min(len(got), len(want))):
    if not np.array_equal(got[i], want[i]):
        for j in range(max(0, i - 3), min(i + 6, len(got), len(want))):
            print(j, got[j].tolist(), want[j].tolist())
        break
