"""Summarise ncu captures into profiles/ (committed evidence).

usage: python scripts/ncu_summary.py <round-tag> <gpurun_out dir>
reads  <dir>/<tag>_k_*.ncu-rep (ncu --set full, one launch each) and <dir>/launches.csv
writes profiles/<tag>_ncu_summary.json, profiles/<tag>_launches_summary.json,
       profiles/xs_fuel_ncu.json (dram bytes per fuel-XS queue entry, read by bench.py)
"""
import csv
import glob
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.per_cycle_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed_op_shfl.sum",
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "us": 1e-6, "usecond": 1e-6,
              "ms": 1e-3, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9, "s": 1, "second": 1,
              "byte/s": 1, "Kbyte/s": 1e3, "Mbyte/s": 1e6, "Gbyte/s": 1e9, "Tbyte/s": 1e12}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for m in METRICS:
        if m in h:
            i = h.index(m)
            v = vals[i].replace(",", "")
            try:
                x = float(v) * UNIT_SCALE.get(units[i], 1)
            except ValueError:
                x = v
            d[m] = x
    return d


def main():
    tag, src = sys.argv[1], sys.argv[2]
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    summary = {}
    for rep in sorted(glob.glob(os.path.join(src, f"{tag}_k_*.ncu-rep"))):
        name = os.path.basename(rep)[len(tag) + 1:-len(".ncu-rep")]
        d = raw(rep)
        threads = d.get("launch__grid_size", 0) * d.get("launch__block_size", 0)
        d["items_upper_bound"] = threads
        summary[name] = d
    note = ("ncu --set full --clock-control none, one launch per kernel from a 1e6-history C2 batch "
            "(1 inactive + 1 active); ncu flushes caches before each replay, so DRAM bytes are cold-cache "
            "upper bounds and times are serialised single launches")
    json.dump({"note": note, "kernels": summary}, open(os.path.join(prof, f"{tag}_ncu_summary.json"), "w"),
              indent=1)
    # dram bytes per fuel lookup (queue entry) of the fuel calculate_xs launch(es) captured
    # (captures may carry an @label: the largest launch of each kernel is used)
    def largest(base):
        c = [k for k in summary if k.split("@")[0] == base]
        return max(c, key=lambda k: summary[k].get("launch__grid_size", 0)) if c else None
    xs_kernels = [largest(k) for k in ("k_xs_fuel", "k_xs_fuel_fused", "k_xs_fuel_seg", "k_xs_fuel_combine")
                  if largest(k)]
    if xs_kernels:
        nseg = int(os.environ.get("OMCG_FUEL_SEGMENTS", "17"))  # 261 fuel nuclides in 16-nuclide segments
        # fuel lookups (queue entries) per block of each kernel
        per_block = {"k_xs_fuel": None, "k_xs_fuel_combine": None, "k_xs_fuel_fused": 32,
                     "k_xs_fuel_seg": 256 / nseg}
        per_block = {k: per_block[k.split("@")[0]] for k in xs_kernels}
        per, parts = 0.0, {}
        for k in xs_kernels:
            x = summary[k]
            items = x["launch__grid_size"] * (per_block[k] or x["launch__block_size"])
            b = (x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"]) / items
            parts[k] = {"lookups_in_capture": items, "dram_bytes_per_lookup": b}
            per += b
        json.dump({"dram_bytes_per_item": per, "kernels": parts,
                   "source": f"profiles/{tag}_ncu_summary.json ({'+'.join(xs_kernels)}, cold cache)"},
                  open(os.path.join(prof, "xs_fuel_ncu.json"), "w"), indent=1)
    # roofs per kernel for bench.py (profiles/roofline_ncu.json)
    roofs = {}
    for k, x in summary.items():
        base = k.split("@")[0]
        if base not in ("k_xs_fuel_fused", "k_move", "k_collide", "k_tail_warp"):
            continue
        dram = x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0)
        t = x.get("gpu__time_duration.sum")
        l1 = x.get("l1tex__throughput.avg.pct_of_peak_sustained_active")
        issue = x.get("smsp__issue_active.avg.pct_of_peak_sustained_active")
        d = {"binding": "L1/TEX throughput" if (l1 or 0) >= (issue or 0) else "issue (latency-bound warps)",
             "l1tex_pct": l1, "issue_active_pct": issue,
             "l1_data_pipe_wavefronts_pct": x.get("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
             "lanes_per_inst": x.get("smsp__thread_inst_executed_per_inst_executed.ratio"),
             "warps_per_sm": x.get("sm__warps_active.avg.per_cycle_active"),
             "l2_hit_pct": x.get("lts__t_sector_hit_rate.pct"),
             "dram_gbs": dram / t / 1e9 if t else None, "ms": 1e3 * t if t else None,
             "source": f"profiles/{tag}_ncu_summary.json ({k}, ncu --set full, cold cache)"}
        if base == "k_xs_fuel_fused":
            d["items"] = x["launch__grid_size"] * 32  # 32 fuel lookups per block
            d["dram_bytes_per_item"] = dram / d["items"]
        if base not in roofs or (d.get("items", 0) > roofs[base].get("items", 0)) or base != "k_xs_fuel_fused":
            roofs[base] = d
    if roofs:
        json.dump(roofs, open(os.path.join(prof, "roofline_ncu.json"), "w"), indent=1)
    lc = os.path.join(src, "launches.csv")
    if os.path.exists(lc):
        rows = list(csv.reader(open(lc)))
        hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        H = rows[hi]
        ki, mi, vi, ui = H.index("Kernel Name"), H.index("Metric Name"), H.index("Metric Value"), H.index("Metric Unit")
        tot, cnt = defaultdict(float), defaultdict(int)
        for r in rows[hi + 1:]:
            if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
                continue
            name = r[ki].split("(")[0].replace("void ", "").replace("omcg::", "").strip()
            tot[name] += float(r[vi].replace(",", "")) * UNIT_SCALE.get(r[ui], 1)
            cnt[name] += 1
        T = sum(tot.values())
        out = {k: {"ms": 1e3 * v, "share": v / T, "launches": cnt[k], "avg_us": 1e6 * v / cnt[k]}
               for k, v in sorted(tot.items(), key=lambda x: -x[1])}
        json.dump({"note": "ncu --metrics gpu__time_duration.sum --clock-control none over 2 batches of C2 "
                           "(cold-cache, serialised launches: compare shares, not absolutes)",
                   "total_ms": 1e3 * T, "launches": sum(cnt.values()), "kernels": out},
                  open(os.path.join(prof, f"{tag}_launches_summary.json"), "w"), indent=1)
    print(json.dumps({k: {m: summary[k].get(m) for m in ("gpu__time_duration.sum", "dram__bytes_read.sum",
                                                          "l1tex__t_sector_hit_rate.pct",
                                                          "lts__t_sector_hit_rate.pct",
                                                          "sm__throughput.avg.pct_of_peak_sustained_elapsed")}
                      for k in summary}, indent=1))


if __name__ == "__main__":
    main()
