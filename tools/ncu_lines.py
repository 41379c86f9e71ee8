"""Per-source-line hot spots of one kernel in an ncu report (built with -lineinfo).

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [TOP]
Prints the source lines with the most warp-stall samples and executed instructions.
"""

import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    fname, rows, head = "", [], None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            head = r
            continue
        if head is None or not r[0] or r[0] == "Function Name":
            continue
        d = dict(zip(head[4:], r[4:]))
        try:
            samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            inst = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        rows.append((samp, inst, f"{fname}:{r[0]}", r[1].strip()[:90]))
    ts = sum(x[0] for x in rows) or 1
    ti = sum(x[1] for x in rows) or 1
    print(f"total samples {ts}, warp instructions {ti:.3e}")
    for samp, inst, loc, src in sorted(rows, reverse=True)[:top]:
        print(f"{100 * samp / ts:5.1f}% smp {100 * inst / ti:5.1f}% ins  {loc:<28} {src}")


if __name__ == "__main__":
    main()
