"""Wall-clock spread of the e2e call with and without nvidia-smi sampling in the background."""
import subprocess, sys, time
sys.path.insert(0, ".")
import paper_2402_09222_b200 as P
p = P.Problem("assembly", host_threads=8)
kw = dict(n_particles=1000000, n_batches=15, n_inactive=5, seed=1, devices=[0])
P.run(p, n_particles=1000000, n_batches=1, n_inactive=0, seed=7, devices=[0])
for mode in ("none", "smi200", "none", "smi200"):
    proc = None
    if mode != "none":
        proc = subprocess.Popen(["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.DEVNULL)
        time.sleep(2.0)
    ws = []
    for _ in range(4):
        t0 = time.perf_counter(); r = P.run(p, **kw).result; ws.append(time.perf_counter() - t0)
    if proc: proc.terminate(); proc.wait()
    print(mode, " ".join(f"{15e6 / w / 1e6:.2f}M" for w in ws), f"fom {r.fom / 1e6:.2f}M")
