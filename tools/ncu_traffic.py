"""Record ncu per-launch DRAM traffic of the hot kernels into
profiles/ncu_traffic.json: {config: {kernel: {dram_bytes, ncu_ms, report, commit}}}.
Usage: python tools/ncu_traffic.py <report.ncu-rep> <config> <commit>"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KERNELS = ["rerank_pair_kernel", "ivf_filter_kernel", "recheck_smem_kernel", "recheck_lut_kernel", "lut_pass_kernel",
           "select_large_kernel", "assign_tc_kernel"]


def main(rep, config, commit):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]

    def val(r, k):
        v = float(r[hdr.index(k)].replace(",", ""))
        u = units[hdr.index(k)]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "msecond": 1, "usecond": 1e-3,
                    "nsecond": 1e-6}.get(u, 1)

    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    tj = json.load(open(path)) if os.path.exists(path) else {}
    ent = tj.setdefault(config, {})
    seen = set()
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        for k in KERNELS:
            if k in name:
                e = {"dram_bytes": val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"),
                     "ncu_ms": val(r, "gpu__time_duration.sum"), "report": os.path.basename(rep),
                     "commit": commit}
                # several launches of one kernel in a search: keep the longest
                if k not in seen or e["ncu_ms"] > ent[k]["ncu_ms"]:
                    ent[k] = e
                    seen.add(k)
    json.dump(tj, open(path, "w"), indent=1, sort_keys=True)
    print(json.dumps(ent, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:4])
