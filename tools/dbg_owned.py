"""Owned re-rank per shard vs the oracle re-rank of the owned subset."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1102_3828_b200 as pq  # noqa: E402
from oracle.oracle_py import Oracle  # noqa: E402
from paper_1102_3828_b200.sharded import shard_range, _rerank_owned  # noqa: E402

o = Oracle()
seed, K = 0, 256
centers = o.synth_centers(seed, K, 128)
base = o.synth_rows(seed, 2, 0, 120_000, centers)
train = o.synth_rows(seed, 1, 0, 20_000, centers).astype(np.float32)
queries = o.synth_rows(seed, 3, 0, 64, centers)
qf = queries.astype(np.float32)
coarse, books = o.ivf_train(train, 128, 8, iterations=4, seed=0)
rbooks = o.ivf_refine_train(coarse, books, 8, train, 16, iterations=4, seed=0)
oix = o.ivf_build(coarse, books, 8, base.astype(np.float32))
oix.refine_encode(rbooks, 16, base.astype(np.float32))
P = pq.ProductQuantizer(128, 8, 256, books.reshape(8, 256, 16))
R = pq.RefineQuantizer(pq.ProductQuantizer(128, 16, 256, rbooks.reshape(16, 256, 8)))
stream = torch.cuda.current_stream()
for ns, v, kp, k in [(2, 16, 300, 100), (3, 8, 1000, 50)]:
    si, sd, sc = oix.search(qf, v, kp)
    dq = torch.from_numpy(queries).cuda()
    dsi = torch.from_numpy(si.view(np.int32)).cuda()
    dsc = torch.from_numpy(sc.view(np.int32)).cuda()
    for r in range(ns):
        lo, hi = shard_range(len(base), r, ns)
        ix = pq.IvfIndex(pq.Codebook(coarse), P, R)
        ix.add(base[lo:hi], id_base=lo)
        ix.finalize()
        gi, gd, gc = [t.cpu().numpy() for t in _rerank_owned(ix, dq, dsi, dsc, k, stream)]
        gi = gi.view(np.uint32)
        bad = 0
        for q in range(len(queries)):
            row = si[q, :sc[q]]
            own = row[(row >= lo) & (row < hi)]
            kk = min(k, len(own))
            ri, rd = oix.rerank(qf[q:q + 1], own[None, :], np.array([len(own)], np.uint32), kk) if kk else (np.zeros((1, 0)), None)
            if gc[q] != kk or not np.array_equal(gi[q, :kk], ri[0]):
                bad += 1
                if bad == 1:
                    print("  q", q, "cnt", gc[q], kk, "dev", gi[q, :6], gd[q, :6], "orc", ri[0, :6], rd[0, :6] if kk else None)
        print(f"shards={ns} r={r} lo={lo}: bad rows {bad}", flush=True)
