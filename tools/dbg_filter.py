"""Filter-path debugging: one mid-size search, compare to the oracle, print stats."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1102_3828_b200 as pq  # noqa: E402
from oracle.oracle_py import Oracle  # noqa: E402

o = Oracle()
centers = o.synth_centers(0, 256, 128)
base = o.synth_rows(0, 2, 0, 120000, centers)
train = o.synth_rows(0, 1, 0, 20000, centers).astype(np.float32)
q = o.synth_rows(0, 3, 0, 64, centers)
coarse, books = o.ivf_train(train, 128, 8, iterations=4, seed=0)
oix = o.ivf_build(coarse, books, 8, base.astype(np.float32))
P = pq.ProductQuantizer(128, 8, 256, books.reshape(8, 256, 16))
dix = pq.ivf_build(pq.Codebook(coarse), P, base)
for v, kp in [(24, 1000), (8, 100), (64, 5000)]:
    oi, od, oc = oix.search(q.astype(np.float32), v, kp)
    di, dd, dc = dix.search(q, v, kp, 0)
    st = dix.last_stats()
    bad = [i for i in range(len(q)) if not np.array_equal(di[i, :oc[i]], oi[i, :oc[i]])]
    print(f"v={v} k'={kp} env={os.environ.get('PQRR_SCAN')},{os.environ.get('PQRR_FILTER_ALL')} "
          f"bad={len(bad)} retries={st['retries']} cand={st['candidates']} scanned={st['scanned_entries']}")
    if bad:
        i = bad[0]
        common = len(set(di[i, :oc[i]]) & set(oi[i, :oc[i]]))
        print("  q", i, "common", common, "of", oc[i], "dev d0..3", dd[i, :4], "orc", od[i, :4])
