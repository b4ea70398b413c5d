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
ix, _, _ = bench.build_index(pq, cfg, coarse, P, rq, 0, 0, 1)
allq = pq.synth(3, 0, 4096, cfg["clusters"], seed=bench.SEED)
for B in [int(b) for b in args.batches.split(",")]:
    q = allq[:B]
    for _ in range(5):
        ix.search(q, cfg["w"], cfg["kprime"], cfg["k"])
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        ix.search(q, cfg["w"], cfg["kprime"], cfg["k"])
        ts.append((time.perf_counter() - t0) * 1e3)
    st = ix.last_stats()
    print(B, "wall ms", round(float(np.median(ts)), 3), {k: round(v, 3) for k, v in st.items() if k.startswith("ms_")},
          "kernels", st["kernels"], "items", st["work_items"], flush=True)
