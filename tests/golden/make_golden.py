"""Generate tests/golden/*.npz — golden vectors for the IVFADC+R path.

Run in the build container (needs /root/reference for oracle/_ref):
    python tests/golden/make_golden.py

Every expected OUTPUT below is produced by oracle/_ref/libpqrr_ref.so, i.e. by
the reference's own code compiled in place: kernels.cpp (assign_batch,
encode_batch, decode_batch, scan_topk incl. its OpenMP partitioned merge),
distance.hpp l2_sq, product_quantizer.hpp adc_distance, topk.hpp TopK, and
rng.hpp SplitMix64 / bounded_u32 / uniform01.  Inputs that the reference
cannot produce (it declares but never defines a generator or a trainer) come
from the oracle restatement with fixed seeds; the restatement's RNG pieces are
pinned against the reference's rng.hpp in the same file.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle_py import Oracle, RefLib, build  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    build(ref=True)
    o = Oracle()
    r = RefLib()
    o.set_threads(0)
    r.set_threads(0)

    # ---------------- primitives
    rng = np.random.default_rng(1102_3828)
    l2_a, l2_b, l2_out = [], [], []
    for d in list(range(1, 20)) + [32, 64, 127, 128, 129]:
        for _ in range(4):
            a = (rng.standard_normal(d) * rng.uniform(0.1, 100)).astype(np.float32)
            b = (rng.standard_normal(d) * rng.uniform(0.1, 100)).astype(np.float32)
            l2_a.append(np.pad(a, (0, 129 - d)))
            l2_b.append(np.pad(b, (0, 129 - d)))
            l2_out.append((d, r.l2_sq(a, b)))
    lut = (rng.random((8, 256)) * 1000).astype(np.float32)
    codes = rng.integers(0, 256, size=(10000, 8), dtype=np.uint8)
    codes[5000:5100] = codes[0]  # exact ADC ties broken by id
    r.set_threads(4)
    sc_ids, sc_d = r.scan_topk(lut, codes, 100, id_base=7)  # n >= 8192: partitioned merge path
    sc_ids1, sc_d1 = r.scan_topk(lut, codes[:3000], 50, id_base=0)  # serial path
    r.set_threads(0)
    tk_ids = rng.permutation(5000).astype(np.uint32)
    tk_d = rng.integers(0, 50, 5000).astype(np.float32)  # many equal distances
    tk_oi, tk_od = r.topk(tk_ids, tk_d, 64)
    sm = r.splitmix(12345, 16)
    bu = r.bounded_u32(7, 1000, 64)
    un = r.uniform01(7, 64)
    np.savez_compressed(
        os.path.join(OUT, "primitives.npz"),
        l2_a=np.array(l2_a), l2_b=np.array(l2_b),
        l2_d=np.array([d for d, _ in l2_out], np.int32),
        l2_out=np.array([v for _, v in l2_out], np.float32),
        lut=lut, codes=codes, scan_ids=sc_ids, scan_dists=sc_d, scan_ids_serial=sc_ids1,
        scan_dists_serial=sc_d1, topk_in_ids=tk_ids, topk_in_d=tk_d, topk_ids=tk_oi,
        topk_d=tk_od, splitmix=sm, bounded=bu, uniform01=un)

    # ---------------- small IVFADC+R instance (SIFT-like generator, seed 0)
    seed, K, d = 0, 64, 128
    centers = o.synth_centers(seed, K, d)
    base = o.synth_rows(seed, 2, 0, 4000, centers)
    train = o.synth_rows(seed, 1, 0, 3000, centers)
    queries = o.synth_rows(seed, 3, 0, 24, centers)
    trf = train.astype(np.float32)
    c, m, mprime = 32, 8, 16
    coarse, books = o.ivf_train(trf, c, m, iterations=6, seed=3)
    rbooks = o.ivf_refine_train(coarse, books, m, trf, mprime, iterations=6, seed=5)
    bf = base.astype(np.float32)
    qf = queries.astype(np.float32)
    # reference kernels on the shared codebooks
    assign, adist = r.assign(bf, coarse)
    res = bf - coarse[assign]
    codes = r.encode(books, res, m)
    dec = r.decode(books, codes, d)
    rec1 = coarse[assign] + dec
    rcodes = r.encode(rbooks, bf - rec1, mprime)
    # lists in id order per list (ivf_index.hpp:15-16)
    order = np.argsort(assign, kind="stable")
    offsets = np.zeros(c + 1, np.uint64)
    offsets[1:] = np.cumsum(np.bincount(assign, minlength=c))
    ids_l = order.astype(np.uint32)
    codes_l = codes[order]
    v, kprime, k = 6, 60, 10
    sl_ids, sl_d, sl_cnt = r.ivf_search(coarse, books, m, offsets, ids_l, codes_l, qf, v, kprime)
    rr_ids, rr_d = r.ivf_rerank(coarse, books, rbooks, m, mprime, assign, codes, rcodes, qf,
                                sl_ids, sl_cnt, k)
    # v = c equals the exhaustive scan over coarse-residual estimates
    ex_ids, ex_d, ex_cnt = r.ivf_search(coarse, books, m, offsets, ids_l, codes_l, qf[:4], c, 200)
    gt_ids, _ = o.exact_nearest(bf, qf)
    np.savez_compressed(
        os.path.join(OUT, "ivf_small.npz"),
        seed=seed, clusters=K, base=base, train=train, queries=queries,
        base_sha256=np.frombuffer(hashlib.sha256(base.tobytes()).digest(), np.uint8),
        coarse=coarse, books=books, rbooks=rbooks, c=c, m=m, mprime=mprime,
        assign=assign, assign_dist=adist, codes=codes, rcodes=rcodes, offsets=offsets, ids_l=ids_l,
        v=v, kprime=kprime, k=k, sl_ids=sl_ids, sl_dists=sl_d, sl_cnt=sl_cnt, rr_ids=rr_ids,
        rr_dists=rr_d, ex_ids=ex_ids, ex_dists=ex_d, ex_cnt=ex_cnt, gt_ids=gt_ids)
    print("golden fixtures written to", OUT)


def main_adc():
    """adc_small.npz: exhaustive ADC / ADC+R (adc_index.hpp, refine.hpp:30-53).
    Expected outputs from the reference's code: codes = kernels::encode_batch(y),
    shortlist = kernels::scan_topk(build_lut(x), all codes) (what adc_search
    computes), residual codes = encode_batch(y - decode(code)),
    re-rank = l2_sq(x, decode + decode_r) through the reference l2_sq and TopK."""
    build(ref=True)
    o = Oracle()
    r = RefLib()
    seed, K, d = 0, 64, 128
    centers = o.synth_centers(seed, K, d)
    base = o.synth_rows(seed, 2, 0, 12000, centers)
    train = o.synth_rows(seed, 1, 0, 3000, centers).astype(np.float32)
    queries = o.synth_rows(seed, 3, 0, 16, centers)
    m, mprime = 8, 8
    books = o.pq_train(train, m, iterations=6, seed=11)
    rbooks = o.refine_train(books, m, train, mprime, iterations=6, seed=12)
    bf, qf = base.astype(np.float32), queries.astype(np.float32)
    codes = r.encode(books, bf, m)
    dec = r.decode(books, codes, d)
    rcodes = r.encode(rbooks, bf - dec, mprime)
    rdec = r.decode(rbooks, rcodes, d)
    kprime, k = 200, 20
    r.set_threads(4)  # n >= 8192: scan_topk's partitioned merge path
    sl = [r.scan_topk(r.build_lut(books, x, m), codes, kprime) for x in qf]
    sl_ids = np.stack([a for a, _ in sl])
    sl_d = np.stack([b for _, b in sl])
    yhat = dec + rdec
    rr = []
    for q in range(len(qf)):
        dd = np.array([r.l2_sq(qf[q], yhat[i]) for i in sl_ids[q]], np.float32)
        rr.append(r.topk(sl_ids[q], dd, k))
    np.savez_compressed(
        os.path.join(OUT, "adc_small.npz"), base=base, queries=queries, books=books,
        rbooks=rbooks, m=m, mprime=mprime, codes=codes, rcodes=rcodes, kprime=kprime, k=k,
        sl_ids=sl_ids, sl_dists=sl_d, rr_ids=np.stack([a for a, _ in rr]),
        rr_dists=np.stack([b for _, b in rr]))
    print("adc fixture written to", OUT)


if __name__ == "__main__":
    if sys.argv[1:] == ["adc"]:
        main_adc()
    else:
        main()
        main_adc()
