"""Text summary of one kernel in an .ncu-rep (ncu --set full): key raw
metrics + warp-stall breakdown, for profiles/.  Usage:
    python tools/ncu_summary.py report.ncu-rep "title line" > profiles/x.txt"""
import csv, io, subprocess, sys

rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
get = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
keys = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"]
print(f"# {title}")
print(f"# source: {rep} (ncu --set full --clock-control none)\n")
for k in keys:
    if k in get:
        v, u = get[k]
        print(f"{k:60s} {v} {u}")
stalls = {h[len("smsp__pcsamp_warps_issue_stalled_"):]: float(v.replace(",", "") or 0)
          for h, v in zip(hdr, vals)
          if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")}
tot = sum(stalls.values()) or 1.0
print("\nwarp stall samples (share):")
for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {k:28s} {100 * v / tot:5.1f}%")
