"""Markdown tables of the bench lines under profiles/ (README):
tools/numbers_table.py r24"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r24"


def load(name):
    try:
        with open(os.path.join(ROOT, "profiles", f"{tag}_bench_{name}.json")) as f:
            return json.load(f)
    except Exception:
        return None


def fmt_q(v):
    return f"{v / 1e6:.3f}M" if v >= 1e6 else f"{v / 1e3:.1f}k"


print("| config | value (q/s, device) | e2e (q/s, host API) | parity in the same run | recall@1/10/100 | reference CPU path | stages (ms) |")
print("|---|---|---|---|---|---|---|")
for c in ("c1", "c2", "c3", "c4"):
    d = load(c)
    if not d:
        continue
    cb = d.get("cpu_baseline", {})
    par = f"{cb.get('parity_mode')}: ids {cb.get('id_match')}, dist bits {cb.get('dist_bits_match')}, {cb.get('queries_compared')} queries"
    if cb.get("add_check"):
        a = cb["add_check"]
        par += f"; add path {a['ids']} ids: lists {a['list_match']}, codes {a['codes_match']}, rcodes {a['rcodes_match']}"
    if "codes_match" in cb:
        par += f"; index bytes: codes {cb['codes_match']}, rcodes {cb.get('rcodes_match')}"
    st = d.get("stages_ms", {})
    stages = ", ".join(f"{k[3:]} {v:.2f}" for k, v in st.items() if k != "ms_total")
    print(f"| {c.upper()} | {fmt_q(d['value'])} | {fmt_q(d['e2e']['value'])} | {par} | "
          f"{d.get('recall@1')} / {d.get('recall@10')} / {d.get('recall@100')} | "
          f"{cb.get('value', 0):.1f} q/s on {cb.get('cores')} cores | {stages}; total {st.get('ms_total', 0):.2f} |")
    if d.get("add"):
        print(f"|  | add: {d['add']['vectors_per_s'] / 1e6:.1f}M vectors/s ({d['add']['seconds']} s) | | | | 1-thread {cb.get('time_per_query_1thread_s')} s/query | roofline frac {d['roofline']['frac']:.3f} ({d['roofline']['kernel'][:30]}) |")
for c in ("ref_c2", "ref_c4"):
    d = load(c)
    if d:
        print(f"\n`--impl reference` {c[4:].upper()}: {d.get('value')} {d.get('unit')} ({d.get('cpu_baseline', {}).get('cores')} cores); "
              f"product library mapped: {d.get('native_so_loaded')}")
d = load("c5")
if d:
    print("\n| batch | device latency | q/s | e2e latency (host API) | e2e q/s |")
    print("|---|---|---|---|---|")
    for r in d["sweep"]:
        print(f"| {r['batch']} | {r['latency_ms']:.3f} ms | {fmt_q(r['qps'])} | {r['e2e_latency_ms']:.3f} ms | {fmt_q(r['e2e_qps'])} |")
