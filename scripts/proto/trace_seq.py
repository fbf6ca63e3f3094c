import sys, json
sys.path.insert(0, ".")
import numpy as np
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
out = P.run(p, n_particles=1000000, n_batches=1, n_inactive=0, trace_queues=True)
t = np.asarray(out.queue_trace).reshape(-1, 3)
json.dump({"queue": t[:, 0].tolist(), "n": t[:, 1].tolist()}, open("gpurun_out/trace_seq.json", "w"))
print(len(t))
