"""K2w per-region instruction / stall shares from an ncu report (source page).
usage: python tools/k2_regions.py REP [kernel-regex]"""
import csv, io, re, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]; k = sys.argv[2] if len(sys.argv) > 2 else "k2_warp"
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{k}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
src = open("paper_2308_16619_b200/csrc/csv_replay_warp.cuh").read().splitlines()
# regions: by marker comments / function starts in the current source
marks = []
for n, l in enumerate(src, 1):
    m = re.search(r"// ---- (\w[\w -]*)|^(?:template|__device__)[^(]*\b(\w+)\(", l)
    if m:
        marks.append((n, (m.group(1) or m.group(2)).strip()))
def region(f, line):
    if f != "csv_replay_warp.cuh":
        return "other:" + f
    name = "top"
    for n, nm in marks:
        if n <= line: name = nm
        else: break
    return name
agg = defaultdict(lambda: [0, 0]); fname = "?"; line = 0; iex = ism = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": iex = r.index("Instructions Executed"); ism = r.index("Warp Stall Sampling (All Samples)"); continue
    if iex is None or len(r) <= iex: continue
    if r[0]: line = int(r[0]); continue
    ex = r[iex].replace(",", "")
    if ex.isdigit():
        a = agg[region(fname, line)]; a[0] += int(ex); a[1] += int(r[ism] or 0)
tot = sum(v[0] for v in agg.values()); ts = sum(v[1] for v in agg.values())
for n, (e, s) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{n:40s} instr {100 * e / tot:5.1f}%  stall-samples {100 * s / ts:5.1f}%")
