"""Hot SASS of one kernel from an ncu report: `ncu -i REP --page source --csv --print-source sass`.
usage: python tools/sass_hot.py SASS.csv [min_frac] [--range A B]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia, isrc, iex, ithr, isamp = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), \
    h.index("Thread Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = [(r[ia], r[isrc].strip(), int(r[iex] or 0), int(r[ithr] or 0), int(r[isamp] or 0)) for r in rows[2:] if len(r) > iex and r[iex].replace(",", "").isdigit()]
tot = sum(d[2] for d in data)
ts = sum(d[4] for d in data)
mf = float(sys.argv[2]) if len(sys.argv) > 2 else 0.001
print(f"total warp instr {tot:.4g}, samples {ts}")
from collections import Counter
op = Counter()
for d in data:
    op[d[1].split()[0] if not d[1].startswith('@') else d[1].split()[1]] += d[2]
print("by opcode:", ", ".join(f"{k}:{v/tot*100:.1f}%" for k, v in op.most_common(25)))
for i, d in enumerate(data):
    if d[2] >= mf * tot:
        print(f"{i:5d} {d[2]/tot*100:6.2f}% thr/w={d[3]/max(d[2],1):5.1f} smp={d[4]:6d}  {d[1]}")
