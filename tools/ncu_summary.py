"""Summarise ncu outputs into profiles/ (tracked evidence).

    python tools/ncu_summary.py launches gpurun_out/launches_c2.csv > profiles/r01_c2_launches.md
    python tools/ncu_summary.py report gpurun_out/prof_c2.ncu-rep > profiles/r01_c2_kernels.md
"""
import csv
import io
import subprocess
import sys


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg, cnt, tot = {}, {}, 0.0
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        name = r[ki].split("(")[0].replace("void ", "").replace("pqrr_b200::", "").replace(
            "<unnamed>::", "")[:70]
        agg[name] = agg.get(name, 0.0) + v
        cnt[name] = cnt.get(name, 0) + 1
        tot += v
    print(f"# kernel launch list ({path})\n")
    print("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: "
          "compare shares, not absolutes)\n")
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"| `{k}` | {cnt[k]} | {v / 1e6:.3f} | {100 * v / tot:.1f}% |")
    print(f"\ntotal: {tot / 1e6:.3f} ms over {sum(cnt.values())} launches")


WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "smem LSU wavefronts % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem ld wavefronts"),
    ("smsp__sass_inst_executed_op_shared_ld.sum", "smem ld instructions"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, units = r[0], r[1]
    ki = h.index("Kernel Name")
    stalls = [n for n in h if n.startswith("smsp__average_warps_issue_stalled")
              and n.endswith("per_issue_active.ratio")]
    print(f"# ncu --set full summary ({path})\n")
    for row in r[2:]:
        name = row[ki].split("(")[0].replace("void ", "").replace("pqrr_b200::", "").replace(
            "<unnamed>::", "")
        print(f"## `{name}`\n\n| metric | value |\n|---|---|")
        for m, label in WANT:
            if m in h:
                i = h.index(m)
                print(f"| {label} (`{m}`) | {row[i]} {units[i]} |")
        ld, inst = "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", \
            "smsp__sass_inst_executed_op_shared_ld.sum"
        if ld in h and inst in h:
            try:
                w = float(row[h.index(ld)].replace(",", ""))
                n = float(row[h.index(inst)].replace(",", ""))
                print(f"| smem wavefronts per ld instruction | {w / max(n, 1):.2f} |")
            except ValueError:
                pass
        st = []
        for n in stalls:
            try:
                st.append((float(row[h.index(n)] or 0), n))
            except ValueError:
                pass
        st.sort(reverse=True)
        print("| top stalls (warps per issue) | " + ", ".join(
            f"{n[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]}="
            f"{v:.2f}" for v, n in st[:5]) + " |\n")


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])
