"""Key ncu metrics + stall breakdown per launch of a report (tooling).
Usage: python tools/ncu_sum.py rep.ncu-rep [launch_index]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
        "lts__t_sectors_srcunit_tex_op_write.sum", "lts__t_requests_srcunit_tex_op_write.sum",
        "smsp__average_warp_latency_per_inst_issued.ratio"]
rows = r[2:]
sel = [int(sys.argv[2])] if len(sys.argv) > 2 else range(len(rows))
for li in sel:
    v = rows[li]
    print("==", v[h.index("Kernel Name")][:90], "grid", v[h.index("launch__grid_size")])
    for w in want:
        if w in h:
            print(f"   {w:60s} {v[h.index(w)]} {r[1][h.index(w)]}")
    st = []
    for i, n in enumerate(h):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
            try:
                st.append((float(v[i].replace(",", "")), n[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1
    print("   stalls:", ", ".join(f"{n} {100 * x / tot:.0f}%" for x, n in sorted(st, reverse=True)[:8]))
