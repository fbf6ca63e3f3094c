"""EDP methodology check of a C5 campaign directory: per evaluation, the
harness's elapsed (results.csv, proj/src/harness.cpp:311-323: EDP = energy x
elapsed) against the binary's own wall time from its GPU lease to exit and the
energy it wrote to metrics.txt over that same span (bin/openmc stderr line
"energy <J> J over <s> s"). With workers <= leasable GPUs the two times agree
to within process start-up (CUDA initialisation before the lease).

usage: python scripts/c5_elapsed_check.py <campaign out dir>
"""
import csv
import json
import os
import re
import statistics
import sys

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
print(json.dumps({"summary": summary, "points": pts[:10]}, indent=1))
