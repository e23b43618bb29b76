"""Per-SASS-instruction executed counts / stall samples / smem wavefronts of one
launch in an ncu report (tooling).  Usage: python tools/sass_hot.py rep kernel_regex [min_exec]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
mn = float(sys.argv[3]) if len(sys.argv) > 3 else 1e5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", f"regex:{kern}", "--launch-skip", sys.argv[4] if len(sys.argv) > 4 else "0", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = [r for r in csv.reader(out.splitlines()) if len(r) > 20 or r[:1] == ["Kernel Name"]]
h = rows[1]
rows = [rows[0], rows[1]] + [r for r in rows[2:] if r[0].startswith("0x")]
ie, ss, wf = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("L1 Wavefronts Shared")
tot_i = sum(float(r[ie] or 0) for r in rows[2:])
tot_s = sum(float(r[ss] or 0) for r in rows[2:])
print(f"total inst {tot_i:.3e}  samples {tot_s:.0f}")
for k, r in enumerate(rows[2:]):
    x = float(r[ie] or 0)
    if x >= mn:
        print(f"{k:5d} {x:10.3e} {100*float(r[ss] or 0)/tot_s:5.1f}% wf={r[wf]:>9s}  {r[1].strip()[:90]}")
