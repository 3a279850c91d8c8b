"""Summarise a gpurun_out/ capture into profiles/ (tracked): the ncu launch
list (per-kernel mean duration, share of the step), the ncu --set full
metrics of the sweep kernel, and the bench lines.

usage: python tools/profile_summary.py <tag>      (e.g. r01_v8)
"""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1]

rows = list(csv.reader(open(os.path.join(OUT, "launches.csv"))))
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[hdr], rows[hdr + 1:]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = defaultdict(list)
for r in data:
    if len(r) > vi:
        agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
launch = {k: {"launches": len(v), "mean_us": sum(v) / len(v) / 1e3} for k, v in agg.items()}
step = {k: sum(v) for k, v in agg.items() if "sweep" in k or "propose" in k}
tot = sum(step.values())
launch["_share_of_step"] = {k: v / tot for k, v in step.items()}

raw = subprocess.run(["ncu", "-i", os.path.join(OUT, "sweep_full.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
H, U, V = r[0], r[1], r[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "smsp__warp_issue_stalled_barrier_per_warp_active.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"]
m = {k: (V[H.index(k)], U[H.index(k)]) for k in want if k in H}


def mb(k):
    v, u = m[k]
    v = float(v)
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


bench = json.load(open(os.path.join(OUT, "bench.json")))
n, mm = bench["config"]["n"], bench["config"]["ntree"]
dram = mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")
summary = {
    "kernel": "bart::sweep_kernel<4> (one MCMC iteration: in-kernel proposals + sequential tree sweep + sigma)",
    "command": "ncu --set full --clock-control none --import-source on -k regex:sweep -s 2003 -c 1 "
               "python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu  (launch 2003: after the 2000-iteration "
               "burn-in and 3 warm-up steps, i.e. at steady state)",
    "trees_at_capture": bench.get("trees"),
    "workload": bench["config"]["workload"],
    "duration_us_ncu": float(m["gpu__time_duration.sum"][0]) * (1e3 if m["gpu__time_duration.sum"][1] == "ms" else 1),
    "dram_bytes_per_launch": dram,
    "algorithmic_bytes_per_launch": 10.0 * n * mm,
    "metrics": {k: f"{v} {u}".strip() for k, (v, u) in m.items()},
    "bench_value_iters_per_s": bench["value"],
    "bench_sweep_ms_events": bench["roofline"]["kernel_ms"],
}
json.dump(summary, open(os.path.join(PROF, "sweep_ncu_summary.json"), "w"), indent=1)
json.dump(launch, open(os.path.join(PROF, f"{tag}_launch_summary.json"), "w"), indent=1)
shutil.copy(os.path.join(OUT, "launches.csv"), os.path.join(PROF, f"{tag}_launches.csv"))
for f in os.listdir(OUT):
    if f.startswith("bench") and f.endswith(".json") or f.startswith("timeline_") or f.startswith("fit_"):
        shutil.copy(os.path.join(OUT, f), os.path.join(PROF, f"{tag}_{f}"))
src = subprocess.run(["ncu", "-i", os.path.join(OUT, "sweep_full.ncu-rep"), "--page", "source", "--csv",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
open("/tmp/_src.csv", "w").write(src)
hot = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), "/tmp/_src.csv", "30"],
                     capture_output=True, text=True).stdout
open(os.path.join(PROF, f"{tag}_sweep_source_hotspots.txt"), "w").write(hot)
print(json.dumps(summary, indent=1))
print(json.dumps(launch, indent=1))
