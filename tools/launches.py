"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv): per
kernel launches, total ms and share; only launches after the first `skip`
(tooling, not part of the product).  Usage: python tools/launches.py f.csv [skip]"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr_i]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
agg, order = {}, []
launches = [r for r in rows[hdr_i + 1:] if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
for r in launches[skip:]:
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("(anonymous namespace)::", "")
    name = name.replace("unsigned int", "u32").replace("unsigned long", "u64").replace("unnamed>::", "")
    v = float(r[vi].replace(",", ""))
    v = v / 1e6 if r[ui] == "ns" else (v / 1e3 if r[ui] in ("us", "usecond") else v)
    if name not in agg:
        agg[name] = [0, 0.0]
        order.append(name)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(t for _, t in agg.values())
print(f"{'kernel':40s} {'launches':>8s} {'ms':>9s} {'share':>6s}")
for n in sorted(order, key=lambda n: -agg[n][1]):
    c, t = agg[n]
    print(f"{n:40s} {c:8d} {t:9.3f} {100 * t / tot:5.1f}%")
print(f"{'total':40s} {sum(c for c, _ in agg.values()):8d} {tot:9.3f}")
