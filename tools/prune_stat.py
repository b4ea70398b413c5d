"""How many probed (query, list) pairs could be skipped by the list lower bound
sum_j min_c LUT_j[c] > tau?  Uses the exact k'-th shortlist distance as tau
(the sampled tau is ~ the 2k'-th, so this under-counts a little)."""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import bench  # noqa: E402
import paper_1102_3828_b200 as pq  # noqa: E402
from oracle.oracle_py import Oracle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--nq", type=int, default=32)
args = ap.parse_args()
cfg = dict(bench.CONFIGS[args.config])
coarse, P, rq = bench.train_codebooks(pq, cfg, 0)
ix, _, _ = bench.build_index(pq, cfg, coarse, P, rq, 0, 0, 1)
q = pq.synth(3, 0, args.nq, cfg["clusters"], seed=bench.SEED)
ids, d, c = ix.search(q, cfg["w"], cfg["kprime"], 0)
probes, pdist = Oracle().coarse_probe(coarse.centroids, q.astype(np.float32), cfg["w"])
feat = []  # (live, rank, gap, ratio, sum_m - d_coarse)
offs, _, _, _ = ix.export_lists_subset(np.arange(cfg["kc"], dtype=np.uint32))
lens = np.diff(offs).astype(np.int64)
tot_pairs = tot_entries = skip_pairs = skip_entries = 0
by_rank = np.zeros(cfg["w"])
for i in range(args.nq):
    tau = d[i, c[i] - 1]
    xr = q[i].astype(np.float32)[None, :] - coarse.centroids[probes[i]]
    luts = pq.build_lut(P, xr)
    for r, (l, lut) in enumerate(zip(probes[i], luts)):
        sm = np.float32(0)
        for j in range(cfg["m"]):
            sm = np.float32(sm + lut.values[j].min())
        feat.append((sm <= tau, r, pdist[i, r] - pdist[i, 0], pdist[i, r] / max(pdist[i, 0], 1e-9),
                     pdist[i, r] / tau))
        tot_pairs += 1
        tot_entries += lens[l]
        if sm > tau:
            skip_pairs += 1
            skip_entries += lens[l]
            by_rank[r] += 1
print(args.config, f"pairs skippable {skip_pairs / tot_pairs:.3f}, entries {skip_entries / tot_entries:.3f}")
print("skippable share by probe rank (per 8):", np.round(by_rank.reshape(-1, 8).mean(1) / args.nq, 2).tolist())

f = np.array(feat, dtype=np.float64)
live = f[:, 0] > 0


def auc(score):  # P(score(live) < score(dead)): lower score should mean live
    o = np.argsort(score, kind="stable")
    rk = np.empty(len(score))
    rk[o] = np.arange(len(score))
    nl, nd = live.sum(), (~live).sum()
    return 1 - (rk[live].sum() - nl * (nl - 1) / 2) / (nl * nd)


for k, name in [(1, "rank"), (2, "gap d(q,l)-d(q,l0)"), (3, "ratio d(q,l)/d(q,l0)"), (4, "d(q,l)/tau")]:
    print(f"AUC {name}: {auc(f[:, k]):.3f}")
