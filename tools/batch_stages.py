"""Per-stage times of small batches on a bench config (C5 latency analysis)."""
import argparse, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
import paper_1102_3828_b200 as pq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--batches", default="1,16,256")
args = ap.parse_args()
cfg = dict(bench.CONFIGS[args.config])
coarse, P, rq = bench.train_codebooks(pq, cfg, 0)
ix, _, _, _ = bench.build_index(pq, cfg, coarse, P, rq, 0, 0, 1)
allq = pq.synth(3, 0, 4096, cfg["clusters"], seed=bench.SEED)
def wall(q):
    for _ in range(5):
        ix.search(q, cfg["w"], cfg["kprime"], cfg["k"])
    ts = []
    for _ in range(30):
        t0 = time.perf_counter()
        ix.search(q, cfg["w"], cfg["kprime"], cfg["k"])
        ts.append((time.perf_counter() - t0) * 1e3)
    return round(float(np.median(ts)), 3)


for B in [int(b) for b in args.batches.split(",")]:
    q = allq[:B]
    ix.set_graph(True)
    wg = wall(q)
    sg = ix.last_stats()
    ix.set_graph(False)
    ws = wall(q)
    st = ix.last_stats()
    ix.set_graph(True)
    print(B, "graph: wall ms", wg, "device ms", round(sg["ms_total"], 3), "kernels", sg["kernels"],
          "| sync path: wall ms", ws, {k: round(v, 3) for k, v in st.items() if k.startswith("ms_")},
          "kernels", st["kernels"], "items", st["work_items"], flush=True)
