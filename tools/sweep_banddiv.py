"""Filter tightness / time vs the K4f band divisor on one bench config."""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1102_3828_b200 as pq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--values", default="40,60,80,100,120,160")
args = ap.parse_args()
cfg = dict(bench.CONFIGS[args.config])
coarse, P, rq = bench.train_codebooks(pq, cfg, 0)
ix, _, _ = bench.build_index(pq, cfg, coarse, P, rq, 0, 0, 1)
q = pq.synth(3, 0, cfg["nq"], cfg["clusters"], seed=bench.SEED)
for v in args.values.split(","):
    os.environ["PQRR_BANDDIV"] = v
    for rep in range(2):
        ix.search(q, cfg["w"], cfg["kprime"], cfg["k"])
    st = ix.last_stats()
    print(args.config, "band_div", v, "cand/q", round(st["candidates"] / cfg["nq"]),
          "exact/q", round(st["exact_candidates"] / cfg["nq"]), "filter ms", round(st["ms_filter"], 3),
          "scan ms", round(st["ms_scan"], 3), "total", round(st["ms_total"], 3), "retries", st["retries"],
          flush=True)
