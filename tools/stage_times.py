"""Per-search stage times for N consecutive searches of a bench config."""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1102_3828_b200 as pq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--searches", type=int, default=4)
args = ap.parse_args()
cfg = dict(bench.CONFIGS[args.config])
coarse, P, rq = bench.train_codebooks(pq, cfg, 0)
ix, _, _ = bench.build_index(pq, cfg, coarse, P, rq, 0, 0, 1)
q = pq.synth(3, 0, cfg["nq"], cfg["clusters"], seed=bench.SEED)
for i in range(args.searches):
    ix.search(q, cfg["w"], cfg["kprime"], cfg["k"])
    st = ix.last_stats()
    print(i, {k: round(v, 2) for k, v in st.items() if k.startswith("ms_")}, st["work_items"], "retries", st["retries"], flush=True)
