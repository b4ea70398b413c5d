"""Summarise ncu launch lists: per-kernel total ms.  usage: sum_lists.py CSV..."""
import csv
import sys
from collections import defaultdict

for p in sys.argv[1:]:
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(p) as f:
        rows = [r for r in csv.reader(l for l in f if l.startswith('"'))]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        v = v / 1e6 if r[ui] in ("ns", "nsecond") else v / 1e3 if r[ui] in ("us", "usecond") else v
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name] += v
        cnt[name] += 1
    print(f"== {p}: total {sum(tot.values()):.3f} ms")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:12]:
        print(f"  {v:8.3f} ms  x{cnt[k]:<4d} {k[:90]}")
