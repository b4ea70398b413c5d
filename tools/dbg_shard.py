"""Per-shard k=0 search vs the oracle shard (ids offset by the shard base)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1102_3828_b200 as pq  # noqa: E402
from oracle.oracle_py import Oracle  # noqa: E402

o = Oracle()
seed, K = 0, 256
centers = o.synth_centers(seed, K, 128)
base = o.synth_rows(seed, 2, 0, 120_000, centers)
train = o.synth_rows(seed, 1, 0, 20_000, centers).astype(np.float32)
queries = o.synth_rows(seed, 3, 0, 64, centers)
coarse, books = o.ivf_train(train, 128, 8, iterations=4, seed=0)
P = pq.ProductQuantizer(128, 8, 256, books.reshape(8, 256, 16))
for lo, hi, v, kp in [(80000, 120000, 8, 1000), (0, 40000, 8, 1000), (60000, 120000, 16, 300),
                      (40000, 80000, 8, 1000)]:
    ix = pq.IvfIndex(pq.Codebook(coarse), P)
    ix.add(base[lo:hi], id_base=lo)
    ix.finalize()
    di, dd, dc = ix.search(queries, v, kp, 0)
    oix = o.ivf_build(coarse, books, 8, base[lo:hi].astype(np.float32))
    oi, od, oc = oix.search(queries.astype(np.float32), v, kp)
    bad = 0
    for q in range(len(queries)):
        n = oc[q]
        if dc[q] != n or not np.array_equal(di[q, :n], oi[q, :n] + lo):
            bad += 1
    print(f"lo={lo} v={v} kp={kp}: bad rows {bad}; stats {ix.last_stats()}")
    if bad:
        print(" dev", di[0, :8], "orc+lo", oi[0, :8] + lo)
