"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel
count / total / share over the last N correction steps (a step starts at a
k_reset_ops launch).  Usage: launch_summary.py launches.csv [N]"""
import collections
import csv
import json
import sys

path = sys.argv[1]
n_steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
mi = h.index("Metric Name") if "Metric Name" in h else None
seq = []
for r in rows[hi + 1:]:
    if mi is not None and r[mi] != "gpu__time_duration.sum":
        continue  # launch lists captured with extra metrics
    v = float(r[vi].replace(",", ""))
    unit = r[ui]
    us = v / 1e3 if unit in ("ns", "nsecond") else v * 1e3 if unit in ("ms", "msecond") else v
    name = r[ki].split("(")[0].replace("void ", "")
    seq.append((name, us))
starts = [i for i, (n, _) in enumerate(seq) if n.endswith("k_reset_ops")]
first = starts[-n_steps] if len(starts) >= n_steps else 0
tail = seq[first:]
agg = collections.OrderedDict()
for n, us in tail:
    c, t = agg.get(n, (0, 0.0))
    agg[n] = (c + 1, t + us)
total = sum(t for _, t in agg.values())
out = {"source": path, "steps": n_steps, "launches": len(tail), "total_us": total,
       "kernels": {n: {"count": c, "total_us": round(t, 1), "avg_us": round(t / c, 2),
                       "share": round(t / total, 4)} for n, (c, t) in
                   sorted(agg.items(), key=lambda kv: -kv[1][1])}}
print(json.dumps(out, indent=1))
