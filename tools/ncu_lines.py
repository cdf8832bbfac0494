"""Aggregate an ncu source page (--print-source cuda,sass CSV) to per-source-line
warp-stall samples: python tools/ncu_lines.py report.ncu-rep [kernel-regex] [top]."""
import csv
import re
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 2 and sys.argv[2] != "-":
    cmd += ["-k", "regex:" + sys.argv[2]]
out = subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()
agg = defaultdict(lambda: [0, ""])
total = 0
fname = "?"
for row in csv.reader(out):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] in ("Function Name", "Line No", "Kernel Name"):
        continue
    try:
        line = int(row[0])
        s = int(row[4])
    except (ValueError, IndexError):
        continue
    agg[(fname, line)][0] += s
    agg[(fname, line)][1] = row[1][:90]
    total += s
print(f"total samples {total}")
for (f, l), (s, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100.0 * s / max(1, total):5.1f}%  {f}:{l:<5d} {src}")
