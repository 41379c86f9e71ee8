"""Summarise `ncu --set full` reports into profiles/ (text summary + per-kernel DRAM traffic).

usage: python tools/ncu_summary.py OUT.txt TITLE report1.ncu-rep [report2.ncu-rep ...]
Also rewrites profiles/ncu_traffic.json (dram read+write bytes per launch, read by bench.py).
"""

import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "launch__grid_size",
    "launch__block_size",
]
STALL = "smsp__average_warps_issue_stalled_"
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    head, units, data = r[0], r[1], r[2:]
    for d in data:
        yield {h: (v, u) for h, u, v in zip(head, units, d)}


def main():
    out_txt, title, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    lines = [title, ""]
    traffic = {}
    for rep in reps:
        for row in rows(rep):
            name = row["Kernel Name"][0]
            lines.append(name)
            for m in METRICS:
                if m in row:
                    v, u = row[m]
                    lines.append(f"  {m:<60} {v} {u}")
            st = []
            for k, (v, u) in row.items():
                if k.startswith(STALL) and k.endswith("_per_issue_active.ratio"):
                    try:
                        st.append((float(v), k[len(STALL):-len("_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            st.sort(reverse=True)
            lines.append("  top stalls (warps per issue): " + ", ".join(f"{n}={v:.2f}" for v, n in st[:6]))
            lines.append("")
            byt = 0.0
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                v, u = row[m]
                byt += float(v.replace(",", "")) * SCALE.get(u, 1.0)
            key = "k2_warp" if "k2_" in name else ("k1_streams" if "k1_" in name else name)
            traffic.setdefault(key, byt)
    with open(out_txt, "w") as f:
        f.write("\n".join(lines))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if os.path.dirname(os.path.abspath(out_txt)) == os.path.join(root, "profiles"):
        # only a summary committed under profiles/ feeds bench.py's roofline.traffic (config 3 captures)
        tj = os.path.join(root, "profiles", "ncu_traffic.json")
        with open(tj, "w") as f:
            json.dump({"source": f"{os.path.relpath(out_txt, root)} (ncu --set full, one launch per kernel)",
                       "workload": "config3", **traffic}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
