"""C4 sharded-path evidence on one B200: the full-core problem run as 1, 2 and 4
ranks (ranks sharing GPU 0 through the in-process loopback BatchComm: the same
partition, int64 reductions and fission-bank exchange plan as the NCCL path).
k-eff per batch and the int64 tallies must be bit-identical for every rank count.

python scripts/c4_sharded.py [out.json]
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2402_09222_b200 as P  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c4_sharded.json"
prob = P.Problem("core")
N, B, I = 2_000_000, 5, 2
rows, ref = [], None
for ranks in (1, 2, 4):
    t0 = time.time()
    o = P.run(prob, n_particles=N, n_batches=B, n_inactive=I, particles_in_flight=N // ranks,
              n_gpus=ranks, devices=[0] * ranks)
    r = o.result
    k = [r.k_coll[b] for b in range(B)]
    if ref is None:
        ref = (k, o.tally.copy())
    same = k == ref[0] and np.array_equal(o.tally, ref[1])
    rows.append(dict(ranks=ranks, histories_per_batch=N, fom_shared_gpu=r.fom, k_coll=k, k_mean=r.k_mean,
                     bit_identical_to_1_rank=bool(same), wall_s=time.time() - t0))
    print(json.dumps(rows[-1]), flush=True)
    assert same, f"{ranks} ranks differ from 1 rank"
json.dump({"note": "C4 full core, 2e6 histories/batch, ranks sharing one B200 via the loopback BatchComm "
                   "(FoM is not a scaling number: the ranks share one GPU)", "runs": rows}, open(out, "w"), indent=1)
