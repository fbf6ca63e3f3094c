"""Quick C2 timing: python scripts/run_c2.py [batches] [inactive] [key=value ...] (GPU)."""
import sys
sys.path.insert(0, ".")
import paper_2402_09222_b200 as P

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 7
ni = int(sys.argv[2]) if len(sys.argv) > 2 else 2
kw = {}
for a in sys.argv[3:]:
    k, v = a.split("=")
    kw[k] = int(v) if v.lstrip("-").isdigit() else v
p = P.Problem("assembly")
names = ["xs_fuel", "xs_nonfuel", "adv", "cross", "coll", "sort", "refill", "tail"]
for prof in (0, 1):
    r = P.run(p, n_particles=1000000, n_batches=nb, n_inactive=ni, profile=prof, **kw).result
    na = nb - ni
    extra = " ".join(f"{n}={r.prof_ms[i] / na:.1f}ms" for i, n in enumerate(names)) if prof else ""
    print(f"{kw} prof={prof} FoM={r.fom:.4e} t_active={r.t_active:.3f} iters={r.queue_iterations} k={r.k_mean:.6f} {extra}")
