"""Internal (non-tuned) knobs of the queued loop at C2: tail threshold and move-kernel event
cap, interleaved repeats on one box. python scripts/sweep_internal.py (GPU)"""
import sys
sys.path.insert(0, ".")
import paper_2402_09222_b200 as P

p = P.Problem("assembly")
pts = [dict(tail_threshold=t, move_event_cap=c) for t in (8192, 16384, 32768) for c in (12, 20, 32)]
res = {}
for rep in range(2):
    for kw in pts:
        r = P.run(p, n_particles=1000000, n_batches=7, n_inactive=2, **kw).result
        res.setdefault(str(kw), []).append(r.fom)
for k, v in sorted(res.items(), key=lambda x: -max(x[1])):
    print(f"{k:50s} " + " ".join(f"{x / 1e6:.3f}" for x in v))
