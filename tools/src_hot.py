"""Per-CUDA-source-line totals from `ncu -i REP --page source --csv --print-source cuda,sass -k K`.
usage: python tools/src_hot.py BOTH.csv [top]"""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = defaultdict(lambda: [0, 0, ""])
fname, line, src, hdr = "?", "?", "", None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; iex = r.index("Instructions Executed"); ism = r.index("Warp Stall Sampling (All Samples)"); continue
    if hdr is None or len(r) <= iex:
        continue
    if r[0]:
        line, src = r[0], r[1]
        continue
    ex = r[iex].replace(",", "")
    if ex.isdigit():
        a = agg[(fname, line)]
        a[0] += int(ex); a[1] += int(r[ism] or 0); a[2] = src
tot = sum(v[0] for v in agg.values()); ts = sum(v[1] for v in agg.values())
print(f"total instr {tot:.4g} samples {ts}")
for (f, l), (ex, sm, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ex/tot*100:5.1f}% smp {sm/ts*100:5.1f}%  {f}:{l}  {s.strip()[:110]}")
