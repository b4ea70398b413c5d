"""Top stalled SASS instructions of one kernel in an ncu report, with the
stall reasons of each (ncu --page source --print-source sass)."""
import csv
import subprocess
import sys


def main(path, kregex, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kregex}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
    hdr = rows[hi]
    i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    data = []
    for r in rows[hi + 1:]:
        try:
            data.append((int(r[i_s]), r))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    data.sort(key=lambda x: -x[0])
    for n, r in data[:top]:
        rs = sorted(((int(r[i]) if r[i].isdigit() else 0, h[6:]) for i, h in reasons), reverse=True)[:3]
        print(f"{100 * n / tot:5.1f}% {r[0][-5:]} {r[i_src][:70]:70s} {rs}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
