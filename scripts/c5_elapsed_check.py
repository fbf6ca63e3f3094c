"""EDP methodology check of a C5 campaign directory: per evaluation, the
harness's elapsed (results.csv, proj/src/harness.cpp:311-323: EDP = energy x
elapsed) against the binary's own wall time over its whole process (main()
entry to exit) and the energy it wrote to metrics.txt over that same span
(bin/openmc stderr line "energy <J> J over <s> s (GPU, whole process)"; the
NVML marks are taken before CUDA is initialised). With workers <= leasable
GPUs no evaluation waits for another's lease, so the two times agree to
within process creation (exec, dynamic loading) and the harness's polling.

It then re-runs the first --standalone K evaluations (default 6) standalone
the way the harness spawns them (/bin/sh script <launcher args> in the
evaluation's directory, AUTOTUNE_LAUNCHER_ARGS set), timed from outside on
the wall clock, and compares the harness's elapsed with that standalone time
(the "elapsed equals the standalone run time" criterion).

usage: python scripts/c5_elapsed_check.py <campaign out dir> [--standalone K]
"""
import csv
import json
import os
import re
import statistics
import subprocess
import sys
import time

out = sys.argv[1]
rows = list(csv.DictReader(open(os.path.join(out, "results.csv"))))
pts = []
for r in rows:
    if r["status"] != "ok":
        continue
    err = open(os.path.join(out, "evals", r["eval_id"], "stderr.log")).read()
    m = re.search(r"energy ([0-9.]+) J over ([0-9.]+) s", err)
    if not m:
        continue
    pts.append({"eval_id": int(r["eval_id"]), "harness_elapsed_s": float(r["elapsed_sec"]),
                "binary_wall_s": float(m.group(2)), "energy_j": float(m.group(1)),
                "objective_edp": float(r["objective"])})
ratios = [p["harness_elapsed_s"] / p["binary_wall_s"] for p in pts if p["binary_wall_s"] > 0]
summary = {
    "evaluations_ok": len(pts), "evaluations": len(rows),
    "elapsed_over_binary_wall": {"median": statistics.median(ratios) if ratios else None,
                                 "min": min(ratios) if ratios else None, "max": max(ratios) if ratios else None},
    "median_gap_s": statistics.median(p["harness_elapsed_s"] - p["binary_wall_s"] for p in pts) if pts else None,
    "edp_equals_energy_times_elapsed": all(
        abs(p["objective_edp"] - p["energy_j"] * p["harness_elapsed_s"]) <= 1e-3 * max(1.0, p["objective_edp"])
        for p in pts),
}
K = int(sys.argv[sys.argv.index("--standalone") + 1]) if "--standalone" in sys.argv else 6
standalone = []
for p in pts[:K]:
    d = os.path.join(out, "evals", str(p["eval_id"]))
    la = open(os.path.join(d, "launcher")).read().strip() if os.path.exists(os.path.join(d, "launcher")) else ""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, AUTOTUNE_LAUNCHER_ARGS=la, PATH=os.path.join(root, "bin") + ":" + os.environ["PATH"])
    for k, v in (("OMCG_PROBLEM", "assembly"), ("OMCG_PARTICLES", "1000000"), ("OMCG_BATCHES", "6"),
                 ("OMCG_INACTIVE", "2")):  # scripts/run_campaign.sh's defaults
        env.setdefault(k, v)
    t0 = time.perf_counter()
    r = subprocess.run(["/bin/sh", "script"] + la.split(), cwd=d, env=env, stdin=subprocess.DEVNULL,
                       capture_output=True, text=True)
    wall = time.perf_counter() - t0

    def fom(txt):
        m = re.findall(r"FOM:\s*([0-9.eE+-]+)", txt)
        return float(m[-1]) if m else None

    def line(txt, key):
        return next((x.strip() for x in txt.splitlines() if key in x), None)

    camp_out = open(os.path.join(d, "stdout.log")).read() if os.path.exists(os.path.join(d, "stdout.log")) else ""
    camp_err = open(os.path.join(d, "stderr.log")).read() if os.path.exists(os.path.join(d, "stderr.log")) else ""
    standalone.append({"eval_id": p["eval_id"], "rc": r.returncode, "standalone_wall_s": wall,
                       "harness_elapsed_s": p["harness_elapsed_s"],
                       "elapsed_over_standalone": p["harness_elapsed_s"] / wall,
                       "launcher": la, "fom_campaign": fom(camp_out), "fom_standalone": fom(r.stdout),
                       "energy_line_campaign": line(camp_err, "energy "), "energy_line_standalone": line(r.stderr, "energy "),
                       "stderr_standalone": r.stderr[-3000:] if os.environ.get("OMCG_TRACE_INIT") else None})
if standalone:
    rs = [x["elapsed_over_standalone"] for x in standalone]
    summary["elapsed_over_standalone_wall"] = {"median": statistics.median(rs), "min": min(rs), "max": max(rs),
                                               "n": len(rs)}
print(json.dumps({"summary": summary, "standalone": standalone, "points": pts[:10]}, indent=1))
