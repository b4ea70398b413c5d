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
v, kp = 8, 100
oi, od, oc = oix.search(q.astype(np.float32), v, kp)
di, dd, dc = dix.search(q, v, kp, 0)
st = dix.last_stats()
print("retries", st["retries"], "counts equal", np.array_equal(dc, oc))
for i in range(len(q)):
    n = oc[i]
    if not np.array_equal(di[i, :n], oi[i, :n]):
        print("q", i, "oc", oc[i], "dc", dc[i], "common", len(set(di[i,:n]) & set(oi[i,:n])),
              "dev", di[i, :5], dd[i, :5], "orc", oi[i, :5], od[i, :5], "dev last", dd[i, n-1], "orc last", od[i, n-1])
