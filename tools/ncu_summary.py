"""Key counters of an ncu report: tools/ncu_summary.py REP [kernel-substring]"""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "smsp__inst_executed.sum"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
sub = sys.argv[2] if len(sys.argv) > 2 else ""
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    if sub not in name:
        continue
    print("==", name[:100])
    for k in KEYS:
        if k in h:
            print(f"  {k:80s} {r[h.index(k)]}")
    st = [(float(r[i]), w) for i, w in enumerate(h)
          if w.startswith("smsp__average_warps_issue_stalled_") and w.endswith("_per_issue_active.ratio")
          and r[i] not in ("", "n/a")]
    for v, w in sorted(st, reverse=True)[:9]:
        print(f"  stall {w[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:30s} {v:.3f}")
