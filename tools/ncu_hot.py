"""Summarise an ncu source page (SASS) by stall samples: top instructions with
their neighbourhood.  Usage: python tools/ncu_hot.py rep.ncu-rep kernel_regex [n]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
si = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((float(r[si]), r[0], r[1].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
order = sorted(range(len(data)), key=lambda i: -data[i][0])
for i in order[:n]:
    v, addr, s = data[i]
    ctx = " | ".join(d[2][:40] for d in data[max(0, i - 2):i])
    print(f"{v / tot * 100:5.1f}%  {s[:60]:60s}  <- {ctx}")
