"""Per-kernel achieved HBM bandwidth from an ncu launch list with
gpu__time_duration.sum, dram__bytes_read.sum and dram__bytes_write.sum
(tooling, not part of the product): launches, mean ms and DRAM GB per launch,
achieved GB/s = DRAM bytes / duration, and its fraction of the measured copy
peak.  The synthetic-data generators are left out (not part of a join).
Usage: python tools/hbm_table.py launches.csv [peak_gbs]"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6549.0
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, ii = h.index("Kernel Name"), h.index("ID")
mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
launch = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("unnamed>::", "")
    name = name.replace("unsigned int", "u32").replace("unsigned long", "u64")
    d = launch.setdefault(r[ii], {"name": name})
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    if r[mi] == "gpu__time_duration.sum":
        d["ms"] = v / 1e6 if u == "ns" else (v / 1e3 if u in ("us", "usecond") else v)
    else:
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
        d[r[mi]] = v * scale
agg = {}
for d in launch.values():
    if re.match(r"k_(payload|skeys|rkeys|gen)", d["name"]):
        continue
    a = agg.setdefault(d["name"], [0, 0.0, 0.0])
    a[0] += 1
    a[1] += d.get("ms", 0.0)
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
print(f"| kernel | launches | ms / launch | DRAM GB / launch | achieved GB/s | of {peak:.0f} GB/s |")
print("|---|---|---|---|---|---|")
for n, (c, ms, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    gbs = b / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
    print(f"| `{n}` | {c} | {ms / c:.3f} | {b / c / 1e9:.3f} | {gbs:.0f} | {100 * gbs / peak:.1f}% |")
