"""Top source lines by warp-stall samples of one kernel in an ncu report:
tools/ncu_lines.py REP KERNEL_REGEX [N]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        inst = int(r[hdr.index("Instructions Executed")])
    except (ValueError, IndexError):
        continue
    rows.append((samp, inst, fname, r[0], r[1].strip()[:90]))
tot = sum(s for s, *_ in rows) or 1
print(f"total samples {tot}")
for s, i, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% {i:>12d}  {f}:{ln}  {src}")
