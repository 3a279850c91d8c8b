"""One-screen summary of an ncu report: duration, DRAM bytes, issue/pipe use, stall reasons.

usage: python tools/ncu_brief.py REPORT.ncu-rep [kernel-substring]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
sub = sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__grid_size"]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if sub not in name:
        continue
    print("==", name[:100])
    for k in keys:
        if k in hdr:
            print(f"  {k:60s} {r[hdr.index(k)]:>14s} {units[hdr.index(k)]}")
    for h, u, v in zip(hdr, units, r):
        if h.startswith("sm__inst_executed_pipe_") and h.endswith("avg.pct_of_peak_sustained_active"):
            try:
                if float(v) >= 5:
                    print(f"  {h:60s} {v:>14s}")
            except ValueError:
                pass
    st = []
    for h, v in zip(hdr, r):
        if h.startswith("smsp__average_warp_latency_issue_stalled_") or h.startswith("smsp__average_warps_issue_stalled_"):
            if h.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(v), h))
                except ValueError:
                    pass
    for v, h in sorted(st, reverse=True)[:8]:
        print(f"  stall {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):40s} {v:8.3f}")
