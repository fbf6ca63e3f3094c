"""Interleaved A/B of runtime options of omcg_run at C2 (GPU):
python scripts/ab_runtime.py R 'k=v,k=v' 'k=v' ...  ('' = defaults). 7 batches, 2 inactive."""
import sys
sys.path.insert(0, ".")
import paper_2402_09222_b200 as P

R = int(sys.argv[1])
variants = sys.argv[2:] or [""]
parse = lambda s: {k: int(v) for k, v in (x.split("=") for x in s.split(",") if x)}
p = P.Problem("assembly")
res = {v: [] for v in variants}
for _ in range(R):
    for v in variants:
        res[v].append(P.run(p, n_particles=1000000, n_batches=7, n_inactive=2, **parse(v)).result.fom)
for v, f in res.items():
    print(f"{v or 'default':40s} mean {sum(f) / len(f) / 1e6:.3f}  " + " ".join(f"{x / 1e6:.3f}" for x in f))
