"""Run one v=24 k'=1000 search with PQRR_DEBUG_DUMP set; save the index and
queries next to the device dump for CPU analysis (tools/dbg_analyze.py)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1102_3828_b200 as pq  # noqa: E402
from oracle.oracle_py import Oracle  # noqa: E402

out = os.environ["PQRR_DEBUG_DUMP"]
o = Oracle()
centers = o.synth_centers(0, 256, 128)
base = o.synth_rows(0, 2, 0, 120000, centers)
train = o.synth_rows(0, 1, 0, 20000, centers).astype(np.float32)
q = o.synth_rows(0, 3, 0, 64, centers)
coarse, books = o.ivf_train(train, 128, 8, iterations=4, seed=0)
P = pq.ProductQuantizer(128, 8, 256, books.reshape(8, 256, 16))
dix = pq.ivf_build(pq.Codebook(coarse), P, base)
di, dd, dc = dix.search(q, 24, 1000, 0)
lists = dix.export_lists()
np.savez(out + "/index.npz", coarse=coarse, books=books, q=q, di=di, dd=dd,
         **{f"l{i}": np.asarray(a) for i, a in enumerate(lists)})
print("stats", dix.last_stats())
print("lists", [np.asarray(a).shape for a in lists])
