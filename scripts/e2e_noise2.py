"""Wall-clock spread of the e2e call with and without profile=2 (fuel-lookup CUDA events)."""
import sys, time
sys.path.insert(0, ".")
import paper_2402_09222_b200 as P
p = P.Problem("assembly", host_threads=8)
ws = {0: [], 2: []}
for _ in range(6):
    for prof in (0, 2):
        P.run(p, n_particles=1000000, n_batches=1, n_inactive=0, seed=7, devices=[0])
        t0 = time.perf_counter()
        r = P.run(p, n_particles=1000000, n_batches=13, n_inactive=3, seed=1, devices=[0], profile=prof).result
        ws[prof].append(time.perf_counter() - t0)
for k, v in ws.items():
    print("profile", k, " ".join(f"{13e6 / w / 1e6:.2f}M" for w in v))
