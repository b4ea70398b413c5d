"""Search time / retries vs the threshold target alpha and sample density
(PQRR_ALPHA, PQRR_SAMPLES) on one bench config; median of 5 searches."""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import bench  # noqa: E402
import paper_1102_3828_b200 as pq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--grid", default="2.0:64,1.7:64,1.5:64,1.5:128,1.3:128,1.3:256")
args = ap.parse_args()
cfg = dict(bench.CONFIGS[args.config])
coarse, P, rq = bench.train_codebooks(pq, cfg, 0)
ix, _, _, _ = bench.build_index(pq, cfg, coarse, P, rq, 0, 0, 1)
q = pq.synth(3, 0, cfg["nq"], cfg["clusters"], seed=bench.SEED)
ref = None
for g in args.grid.split(","):
    a, sp = g.split(":")
    os.environ["PQRR_ALPHA"], os.environ["PQRR_SAMPLES"] = a, sp
    ix.search(q, cfg["w"], cfg["kprime"], cfg["k"])
    tot, rows = [], []
    for rep in range(5):
        ids, d, c = ix.search(q, cfg["w"], cfg["kprime"], cfg["k"])
        st = ix.last_stats()
        tot.append(st["ms_total"])
        rows.append(st)
    if ref is None:
        ref = ids.copy()
    st = rows[int(np.argsort(tot)[2])]
    print(args.config, "alpha", a, "samples", sp, "total", round(float(np.median(tot)), 3),
          {k: round(v, 3) for k, v in st.items() if k.startswith("ms_")},
          "cand/q", round(st["candidates"] / cfg["nq"]), "retries", st["retries"],
          "same_ids", bool((ids == ref).all()), flush=True)
