"""Summarise an ncu --set full report: duration, DRAM bytes, stall mix and
pipe utilisation per kernel (read here, no GPU needed)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
keys = ["dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "smsp__inst_executed_pipe_fp64.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "launch__grid_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
for r in rows[2:]:
    name = r[h.index("Kernel Name")][:40]
    print(f"=== {name}  {r[h.index('gpu__time_duration.sum')]} {units[h.index('gpu__time_duration.sum')]}")
    items = []
    for i, n in enumerate(h):
        if "smsp__pcsamp_warps_issue_stalled" in n and not n.endswith("not_issued"):
            try:
                items.append((float(r[i].replace(",", "")), n.split("stalled_")[1]))
            except ValueError:
                pass
    items.sort(reverse=True)
    tot = sum(v for v, _ in items) or 1
    print("    stalls:", ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in items[:6]))
    for k in keys:
        if k in h:
            print(f"    {k} = {r[h.index(k)]} {units[h.index(k)]}")
