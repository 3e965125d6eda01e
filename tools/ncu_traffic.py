"""DRAM traffic of the integrate launches (k_fuse<kIntegrate>, the roofline
kernel) of an ncu --set full capture of
tools/prof_workload.py, set beside the same launches' algorithmic bytes
(prof_workload --json).  Writes profiles/fuse_traffic.json, which bench.py
reports as roofline.traffic.
Usage: ncu_traffic.py REPORT WORKLOAD_JSON OUT_JSON"""
import csv
import json
import subprocess
import sys

rep, wl, dst = sys.argv[1:4]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
launches = []
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    if "k_fuse<0>" not in name:  # the roofline kernel: integrate
        continue
    b = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(m)
        b += float(r[i].replace(",", "")) * scale[units[i]]
    launches.append({"kernel": name.split("(")[0], "dram_bytes": b,
                     "duration_us": float(r[h.index("gpu__time_duration.sum")].replace(",", ""))
                     / (1e3 if units[h.index("gpu__time_duration.sum")] in ("nsecond", "ns") else 1)})
w = json.load(open(wl))
avg = sum(x["dram_bytes"] for x in launches) / max(len(launches), 1)
alg = w.get("alg_bytes_per_integrate_launch") or w["alg_bytes_per_fuse_launch"]
res = {"source": rep, "workload": w, "launches": launches, "bytes_per_launch": avg,
       "alg_bytes_per_launch": alg, "traffic_over_alg": avg / alg}
json.dump(res, open(dst, "w"), indent=1)
print(json.dumps({k: res[k] for k in ("bytes_per_launch", "alg_bytes_per_launch", "traffic_over_alg")}))
