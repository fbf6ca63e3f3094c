"""Wall-clock spread of repeated e2e calls (prints the per-call particles/s)."""
import sys, time
sys.path.insert(0, ".")
import paper_2402_09222_b200 as P
p = P.Problem("assembly", host_threads=8)
ws = []
for _ in range(8):
    P.run(p, n_particles=1000000, n_batches=1, n_inactive=0, seed=7, devices=[0])
    t0 = time.perf_counter()
    r = P.run(p, n_particles=1000000, n_batches=13, n_inactive=3, seed=1, devices=[0], profile=2).result
    ws.append(time.perf_counter() - t0)
print(sys.argv[1:], " ".join(f"{13e6 / w / 1e6:.2f}M" for w in ws))
