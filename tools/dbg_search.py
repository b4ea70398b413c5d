import sys, os, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1102_3828_b200 as pq
from oracle.oracle_py import Oracle
o = Oracle()
centers = o.synth_centers(0, 256, 128)
base = o.synth_rows(0, 2, 0, 120000, centers)
train = o.synth_rows(0, 1, 0, 20000, centers).astype(np.float32)
q = o.synth_rows(0, 3, 0, 64, centers)
coarse, books = o.ivf_train(train, 128, 8, iterations=4, seed=0)
oix = o.ivf_build(coarse, books, 8, base.astype(np.float32))
P = pq.ProductQuantizer(128, 8, 256, books.reshape(8, 256, 16))
dix = pq.ivf_build(pq.Codebook(coarse), P, base)
oi, od, oc = oix.search(q.astype(np.float32), 24, 1000)
di, dd, dc = dix.search(q, 24, 1000, 0)
print(os.environ.get("PQRR_STRAT"), os.environ.get("PQRR_TOPW"), "match", np.array_equal(di, oi), dix.last_stats()['retries'])
# coarse probes check via shortlist of v=24 with k'=huge? compare first rows
print(di[0,:12]); print(oi[0,:12]); print(dd[0,:12]); print(od[0,:12])
