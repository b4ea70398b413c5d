"""Small end-to-end case for compute-sanitizer (memcheck / racecheck /
synccheck): one index build (tensor-core assign + encode + layout), fused
searches on the sampled two-phase and single-phase paths (LUT pass, K4f, K4r,
selections, CTA-pair re-ranker), the packed merge and a 2-shard group search.
Checked against the CPU oracle so a sanitizer run also proves the results."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1102_3828_b200 as pq  # noqa: E402
from oracle.oracle_py import Oracle  # noqa: E402
from paper_1102_3828_b200.sharded import IndexGroup, shard_range  # noqa: E402


def main():
    o = Oracle()
    centers = o.synth_centers(0, 64, 128)
    base = o.synth_rows(0, 2, 0, 30_000, centers)
    train = o.synth_rows(0, 1, 0, 6000, centers).astype(np.float32)
    q = o.synth_rows(0, 3, 0, 24, centers)
    coarse, books = o.ivf_train(train, 128, 8, iterations=3, seed=0)
    rbooks = o.ivf_refine_train(coarse, books, 8, train, 16, iterations=3, seed=0)
    P = pq.ProductQuantizer(128, 8, 256, books.reshape(8, 256, 16))
    R = pq.RefineQuantizer(pq.ProductQuantizer(128, 16, 256, rbooks.reshape(16, 256, 8)))
    ix = pq.ivf_build(pq.Codebook(coarse), P, base, rq=R)
    oix = o.ivf_build(coarse, books, 8, base.astype(np.float32))
    oix.refine_encode(rbooks, 16, base.astype(np.float32))
    qf = q.astype(np.float32)
    for v, kp, k in [(8, 300, 50), (40, 2000, 100)]:
        si, _, sc = oix.search(qf, v, kp)
        ri, rd = oix.rerank(qf, si, sc, k)
        gi, gd, _ = ix.search(q, v, kp, k)
        assert np.array_equal(gi, ri) and np.array_equal(gd.view(np.uint32), rd.view(np.uint32)), (v, kp, k)
    shards = []
    for r in range(2):
        lo, hi = shard_range(len(base), r, 2)
        s = pq.IvfIndex(pq.Codebook(coarse), P, R)
        s.add(base[lo:hi], id_base=lo)
        s.finalize()
        shards.append(s)
    g = IndexGroup(shards)
    gi, gd, _ = g.search(q, 8, 300, 50)
    si, _, sc = oix.search(qf, 8, 300)
    ri, rd = oix.rerank(qf, si, sc, 50)
    assert np.array_equal(gi, ri) and np.array_equal(gd.view(np.uint32), rd.view(np.uint32))
    g.close()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
