"""Aggregate an ncu --set full report's SASS source page for one kernel
launch: stall samples and executed warp-instructions per opcode class, plus
the hottest instructions.
Usage: ncu_sass_profile.py REPORT KERNEL_SUBSTR [TOP] [NTH_LAUNCH]"""
import collections
import csv
import io
import subprocess
import sys

rep, ksub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
nth = int(sys.argv[4]) if len(sys.argv) > 4 else 0  # which launch of the matching kernel
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for line in out.splitlines():
    if line.startswith('"Kernel Name"'):
        cur = [line.split(",")[1].strip('"'), []]
        blocks.append(cur)
    elif cur is not None:
        cur[1].append(line)
matches = [(n, l) for n, l in blocks if ksub in n]
for name, lines in matches[nth:nth + 1]:
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]
    si, ii, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
    by_op = collections.defaultdict(lambda: [0, 0])
    hot = []
    for r in rows[1:]:
        try:
            s, n = int(r[si]), int(r[ii])
        except (ValueError, IndexError):
            continue
        op = r[src].split()[0] if r[src].split() else "?"
        if op.startswith("@"):
            op = r[src].split()[1]
        op = op.split(".")[0]
        by_op[op][0] += s
        by_op[op][1] += n
        hot.append((s, n, r[0], r[src].strip()))
    ts = sum(v[0] for v in by_op.values()) or 1
    ti = sum(v[1] for v in by_op.values()) or 1
    print(f"=== {name}: samples {ts}, warp-instructions {ti}")
    for op, (s, n) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:30]:
        print(f"  {op:10s} stall {100 * s / ts:5.1f}%   inst {100 * n / ti:5.1f}%")
    print("  hottest:")
    for s, n, addr, txt in sorted(hot, reverse=True)[:top]:
        print(f"    {100 * s / ts:5.2f}% n={n:9d} {txt[:90]}")
