"""Parity at BASELINE scale (configs[0] = C1 in full): the device path against
the reference's own CPU implementation (oracle/_ref, via oracle/ref_harness.py)
on the same seeded synthetic data.

* codebooks: device ivf_train / ivf_refine_train vs the host trainer, bit for bit;
* add path: every list, id, code and refinement code of the 1M-vector index
  (device add from device-generated rows vs the reference's assign_batch /
  encode_batch on host-generated rows), byte for byte;
* search: all 1000 queries, fused device search (w = 8, k' = 100, k = 100) vs
  the reference search + re-rank, ids and distance bits;
* the add-path lookup seam (pqrr_dev_lookup_ids) on a random id sample.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

C1 = dict(n=1_000_000, train=100_000, nq=1000, clusters=1024, kc=1024, m=8, mprime=8, w=8,
          kprime=100, k=100)


def test_c1_full_parity_against_reference(pq, reflib):
    from oracle import ref_harness as H
    from oracle.oracle_py import Oracle

    cfg = C1
    reflib.set_threads(0)
    c_coarse, c_books, c_rbooks, centers = H.cpu_train(cfg, 0)
    train = pq.synth(1, 0, cfg["train"], cfg["clusters"], seed=0).astype(np.float32)
    prm = pq.TrainParams(iterations=25, seed=0)
    coarse, P = pq.ivf_train(train, cfg["kc"], cfg["m"], params=prm)
    rq = pq.ivf_refine_train(coarse, P, train, cfg["mprime"], prm)
    assert np.array_equal(coarse.centroids.view(np.uint32), c_coarse.view(np.uint32))
    assert np.array_equal(P.flat().view(np.uint32), c_books.view(np.uint32))
    assert np.array_equal(rq.pq.flat().view(np.uint32), c_rbooks.view(np.uint32))

    hx = H.cpu_build(cfg, 0, codebooks=(c_coarse, c_books, c_rbooks))
    ix = pq.IvfIndex(coarse, P, rq)
    ix.add_synthetic(0, cfg["clusters"], 0, cfg["n"], id_base=0)
    ix.finalize()
    offs, ids, codes, rcodes = ix.export_lists()
    np.testing.assert_array_equal(offs, hx.offs)
    np.testing.assert_array_equal(ids, hx.ids)
    np.testing.assert_array_equal(codes, hx.codes)
    np.testing.assert_array_equal(rcodes, hx.rcodes_list_order())

    queries = Oracle().synth_rows(0, 3, 0, cfg["nq"], centers)
    gi, gd, gc = ix.search(queries, cfg["w"], cfg["kprime"], cfg["k"])
    ri, rd, _ = H.ref_search(reflib, hx, queries, cfg["w"], cfg["kprime"], cfg["k"])
    np.testing.assert_array_equal(gi, ri)
    np.testing.assert_array_equal(gd.view(np.uint32), rd.view(np.uint32))
    assert (gc == cfg["k"]).all()
    # shortlists too (k = 0: the IVFADC top-k' in (dist, id) order)
    si, sd, sc = ix.search(queries[:200], cfg["w"], cfg["kprime"], 0)
    ri0, rd0, rc0 = H.ref_search(reflib, hx, queries[:200], cfg["w"], cfg["kprime"], 0)
    np.testing.assert_array_equal(sc, rc0)
    np.testing.assert_array_equal(si, ri0)
    np.testing.assert_array_equal(sd.view(np.uint32), rd0.view(np.uint32))

    sid = np.random.default_rng(3).choice(cfg["n"], 5000, replace=False).astype(np.uint32)
    lst, lc, lrc = ix.lookup_ids(sid)
    np.testing.assert_array_equal(lst, hx.list_of_id[sid])
    np.testing.assert_array_equal(lc, hx.codes_by_id[sid])
    np.testing.assert_array_equal(lrc, hx.rcodes_by_id[sid])
    missing, _, _ = ix.lookup_ids(np.array([cfg["n"] + 5], np.uint32))
    assert missing[0] == 0xFFFFFFFF
    ix.close()
