"""Per-CUDA-source-line instruction and stall-sample totals from
`ncu --page source --csv --print-source cuda,sass` output."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
per = defaultdict(lambda: [0.0, 0.0, ""])
fname = ""
hdr = None
cur = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:  # a cuda source line row
        cur = (fname, r[0], r[1].strip()[:80])
        continue
    if cur is None:
        continue
    try:
        ex = float(r[7].replace(",", "")) if r[7] else 0.0
        sm = float(r[6].replace(",", "")) if r[6] else 0.0
    except ValueError:
        continue
    e = per[cur]
    e[0] += ex
    e[1] += sm
tot_e = sum(v[0] for v in per.values()) or 1
tot_s = sum(v[1] for v in per.values()) or 1
print(f"total instructions {tot_e:.0f}, samples {tot_s:.0f}")
for k, v in sorted(per.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / tot_e * 100:5.1f}% inst {v[1] / tot_s * 100:5.1f}% smp  {k[0]}:{k[1]}  {k[2]}")
