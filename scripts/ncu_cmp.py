"""Key counters of one kernel capture: python scripts/ncu_cmp.py rep.ncu-rep [rep2 ...]"""
import csv, io, subprocess, sys
KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts.sum",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "dram__bytes_read.sum", "launch__registers_per_thread",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "smsp__inst_executed_op_shfl.sum", "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, v = rows[0], rows[2]
    d = dict(zip(h, v))
    print(rep)
    for k in KEYS:
        for name in d:
            if name == k or name.endswith("." + k):
                print(f"  {k:70s} {d[name]}")
