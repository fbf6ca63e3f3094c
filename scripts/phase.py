"""Per-batch launch timeline (profile=1, OMCG_PROF_LOG): kernel time before and
after the source is exhausted (last refill of the batch), and in small launches."""
import os, re, subprocess, sys
if os.environ.get("PHASE_CHILD") != "1":
    env = dict(os.environ, PHASE_CHILD="1", OMCG_PROF_LOG="1")
    r = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True)
    sys.stdout.write(r.stdout)
    names = ["xs_fuel", "xs_nonfuel", "move", "cross", "collide", "sort", "refill", "tail"]
    L = [tuple(map(float, m.groups())) for m in re.finditer(r"\[launch\] class (\d+) items (\d+) ms ([\d.]+)", r.stderr)]
    batches, cur = [], []
    for c, it, ms in L:
        cur.append((int(c), int(it), ms))
        if c == 7:
            batches.append(cur); cur = []
    import json
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump({"classes": names, "batches": batches[-2:]}, open("gpurun_out/phase_launches.json", "w"))
    for b in batches[-2:]:
        tot = sum(x[2] for x in b)
        last_refill = max(i for i, x in enumerate(b) if x[0] == 6)
        after = b[last_refill + 1:]
        print(f"batch: {len(b)} launches, {tot:.2f} ms kernels; after source exhausted: {len(after)} launches "
              f"{sum(x[2] for x in after):.2f} ms ({100 * sum(x[2] for x in after) / tot:.1f} %)")
        for thr in (10000, 50000, 200000):
            sm = [x for x in b if x[1] < thr and x[0] != 7]
            print(f"  launches with < {thr} items (excl. tail): {len(sm)}  {sum(x[2] for x in sm):.2f} ms")
        tl = [x for x in b if x[0] == 7]
        print(f"  tail: {tl}")
        per = {}
        for x in after:
            per.setdefault(names[x[0]], [0, 0.0]); per[names[x[0]]][0] += 1; per[names[x[0]]][1] += x[2]
        print("  after exhaustion by class:", {k: (v[0], round(v[1], 2)) for k, v in per.items()})
    sys.exit(0)
sys.path.insert(0, ".")
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
r = P.run(p, n_particles=1000000, n_batches=3, n_inactive=1, profile=1).result
print(f"t_active/batch {1e3 * r.t_active / 2:.2f} ms  FoM {r.fom / 1e6:.3f}M")
