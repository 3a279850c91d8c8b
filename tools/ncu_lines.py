"""Aggregate ncu source-page stall samples per CUDA source line.

usage: ncu -i rep --page source --csv --print-source cuda,sass > mix.csv
       python tools/ncu_lines.py mix.csv [top]
"""
import csv, sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr = None, None
agg = defaultdict(lambda: [0, 0, 0, ""])
stall_tot = defaultdict(int)
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("Function Name",) or len(r) < 8 or r[2] != "-":
        continue
    try:
        samp = int(r[4]); inst = int(r[7])
    except ValueError:
        continue
    k = (fname, int(r[0]))
    a = agg[k]
    a[0] += samp; a[1] += inst; a[3] = r[1][:90]
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                v = int(r[i])
            except ValueError:
                continue
            stall_tot[h] += v
            a[2] = a[2]
tot = sum(a[0] for a in agg.values())
print("total samples", tot)
print("stalls:", sorted(((v, k) for k, v in stall_tot.items()), reverse=True)[:10])
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{a[0]:7d} {100*a[0]/tot:5.1f}% inst {a[1]:10d}  {k[0]}:{k[1]}  {a[3]}")
