"""Aggregate ncu source-page warp-stall samples per CUDA source line.
usage: python scripts/ncu_hot.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = None; agg = {}; src = {}; fname = ""
for r in rows:
    if r and r[0] == "File Path": fname = r[1].split("/")[-1]
    if r and r[0] == "Line No": h = r; continue
    if h is None or len(r) < 5: continue
    try: w = int(r[4]); ln = int(r[0])
    except ValueError: continue
    key = (fname, ln); agg[key] = agg.get(key, 0) + w; src[key] = r[1]
tot = sum(agg.values()) or 1
for k, w in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{100*w/tot:5.1f}% {k[0]}:{k[1]:<5d} {src[k][:100]}")
