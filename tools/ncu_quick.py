"""Key metrics of one kernel in an ncu report: python tools/ncu_quick.py REP [kernel-regex]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; k = sys.argv[2] if len(sys.argv) > 2 else "k2_warp"
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{k}", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, u, v = r[0], r[1], r[2]
want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for w in want:
    if w in h:
        i = h.index(w); print(f"  {w:70s} {v[i]} {u[i]}")
st = [(float(v[i].replace(',', '')), n) for i, n in enumerate(h)
      if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio") and v[i]]
print("  stalls:", ", ".join(f"{n[34:-23]}={x:.2f}" for x, n in sorted(st, reverse=True)[:8]))
