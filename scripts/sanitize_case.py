"""One small transport run for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): python scripts/sanitize_case.py <case>. The run is also
checked bit-for-bit against the oracle so a sanitizer pass is a correct pass.
Cases cover the queued loop (event fusion, move cap, one kernel per event),
queueless mode, the fuel-queue sort, the tail, P5 sub-banks, the 2-rank
loopback exchange, the one-rank NCCL path and the device-driven loop."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402  (checker only)
import paper_2402_09222_b200 as P  # noqa: E402

CASES = {
    "pincell_queued": ("pincell", 2000, dict(particles_in_flight=1000, tail_threshold=200, sort_threshold=0)),
    "pincell_queueless": ("pincell", 2000, dict(mode="openmc-queueless", particles_in_flight=1000, tail_threshold=100)),
    "pincell_unfused": ("pincell", 2000, dict(particles_in_flight=1000, event_fusion=0, tail_threshold=100)),
    "pincell_cap1_p5": ("pincell", 600, dict(particles_in_flight=300, move_event_cap=1, tasks_per_gpu=2)),
    "pincell_2rank": ("pincell", 2000, dict(particles_in_flight=1000, n_gpus=2, devices=[0, 0])),
    "pincell_nccl1": ("pincell", 2000, dict(particles_in_flight=1000, force_nccl=True)),
    "assembly_queued": ("assembly", 600, dict(particles_in_flight=600, sort_threshold=100, tail_threshold=50)),
    "assembly_queueless": ("assembly", 600, dict(mode="openmc-queueless", particles_in_flight=300, tail_threshold=50)),
    "assembly_unfused": ("assembly", 400, dict(particles_in_flight=400, event_fusion=0, tail_threshold=50)),
    # the device-driven queued loop: guarded candidates, persistent fuel lookup and collisions
    "pincell_dsq": ("pincell", 2000, dict(particles_in_flight=2000, tail_threshold=100, sort_threshold=0,
                                          device_schedule=1)),
    "assembly_dsq": ("assembly", 600, dict(particles_in_flight=600, sort_threshold=100, tail_threshold=50,
                                           device_schedule=1)),
}

name = sys.argv[1]
kind, n, kw = CASES[name]
out = P.run(P.Problem(kind), n_particles=n, n_batches=2, n_inactive=1, seed=1, record_batch=2, record_n=min(n, 200),
            **kw)
o = O.Problem(P.KINDS[kind], 1234, 4000)
ores, otally, orecs = o.run(n, 2, 1, seed=1, record_batch=2, record_n=min(n, 200))
rec = O.records_array(orecs, min(n, 200))
ok = all(np.array_equal(out.records[f], rec[f]) for f in ("n_xs", "n_adv", "n_cross", "n_coll", "n_sites", "term"))
ok = ok and all(out.result.k_coll[b] == ores.k_coll[b] for b in range(2)) and np.array_equal(out.tally, otally)
print(f"{name}: launches {out.result.kernel_launches_total} parity {'ok' if ok else 'FAILED'}")
sys.exit(0 if ok else 1)
