"""Summarise an ncu --set full report: per kernel time, throughput, smem
wavefronts / conflicts, DRAM bytes and the stall breakdown (pc sampling)."""
import csv
import subprocess
import sys


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
    for r in rows[2:]:
        print("###", r[hdr.index("Kernel Name")][:90])
        for k in keys:
            if k in hdr:
                print(f"  {k} = {r[hdr.index(k)]} {units[hdr.index(k)]}")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    st.append((h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i].replace(",", ""))))
                except ValueError:
                    pass
        tot = sum(v for _, v in st) or 1.0
        st.sort(key=lambda x: -x[1])
        print("  stalls (pc samples %):", ", ".join(f"{k} {100 * v / tot:.1f}" for k, v in st[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
