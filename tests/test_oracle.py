"""CPU suite: the oracle restatement pinned against the reference's own code
(oracle/_ref, live) and the golden vectors that code produced (tests/golden),
plus the SPEC.md known-answer examples.  No GPU needed."""
import numpy as np
import pytest


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


# ------------------------------------------------------------------ primitives
def test_l2_sq_matches_reference_golden(oracle, golden_prims):
    g = golden_prims
    for a, b, d, v in zip(g["l2_a"], g["l2_b"], g["l2_d"], g["l2_out"]):
        got = np.float32(oracle.l2_sq(a[:d], b[:d]))
        assert got.view(np.uint32) == np.float32(v).view(np.uint32), d


def test_scan_topk_matches_reference_golden(oracle, golden_prims):
    g = golden_prims
    ids, d = oracle.scan_topk(g["lut"], g["codes"], 100, id_base=7)
    np.testing.assert_array_equal(ids, g["scan_ids"])
    np.testing.assert_array_equal(bits(d), bits(g["scan_dists"]))
    ids, d = oracle.scan_topk(g["lut"], g["codes"][:3000], 50)
    np.testing.assert_array_equal(ids, g["scan_ids_serial"])
    np.testing.assert_array_equal(bits(d), bits(g["scan_dists_serial"]))


def test_topk_ties_by_id(oracle, golden_prims):
    g = golden_prims
    ids, d = oracle.topk(g["topk_in_ids"], g["topk_in_d"], 64)
    np.testing.assert_array_equal(ids, g["topk_ids"])
    np.testing.assert_array_equal(d, g["topk_d"])


def test_rng_matches_reference(oracle, golden_prims):
    g = golden_prims
    np.testing.assert_array_equal(oracle.splitmix_raw(12345, 16), g["splitmix"])
    np.testing.assert_array_equal(oracle.bounded_u32(7, 1000, 64), g["bounded"])
    np.testing.assert_array_equal(oracle.uniform01(7, 64), g["uniform01"])


def test_live_reference_kernels(oracle, reflib):
    rng = np.random.default_rng(5)
    pts = rng.standard_normal((3000, 24)).astype(np.float32) * 10
    cen = rng.standard_normal((37, 24)).astype(np.float32) * 10
    cen[5] = cen[3]  # duplicate centroid: lowest index must win
    a1, d1 = oracle.assign(pts, cen)
    a2, d2 = reflib.assign(pts, cen)
    np.testing.assert_array_equal(a1, a2)
    np.testing.assert_array_equal(bits(d1), bits(d2))
    assert not np.any(a1 == 5)
    books = rng.standard_normal((4, 256, 6)).astype(np.float32)
    np.testing.assert_array_equal(oracle.encode(books, pts, 4), reflib.encode(books, pts, 4))
    codes = rng.integers(0, 256, (50, 4), dtype=np.uint8)
    np.testing.assert_array_equal(bits(oracle.decode(books, codes, 24)),
                                  bits(reflib.decode(books, codes, 24)))
    np.testing.assert_array_equal(bits(oracle.build_lut(books, pts[0], 4)),
                                  bits(reflib.build_lut(books, pts[0], 4)))


# ------------------------------------------------------------------ generator
def test_generator_deterministic_and_shaped(oracle, golden_ivf):
    g = golden_ivf
    centers = oracle.synth_centers(int(g["seed"]), int(g["clusters"]), 128)
    base = oracle.synth_rows(int(g["seed"]), 2, 0, 4000, centers)
    np.testing.assert_array_equal(base, g["base"])
    # row ranges are independent (counter streams)
    part = oracle.synth_rows(int(g["seed"]), 2, 1000, 10, centers)
    np.testing.assert_array_equal(part, g["base"][1000:1010])
    assert base.min() == 0 and base.max() <= 255
    assert not np.any((base > 0) & (base < 4))  # values < 4 zeroed
    # sets are independent streams
    assert not np.array_equal(oracle.synth_rows(0, 3, 0, 5, centers), base[:5])


def test_ln_sincos_accuracy(oracle):
    for u in [1.0, 0.5, 0.123456789, 1e-9, 2.0 ** -53, 0.999999]:
        assert abs(oracle.ln(u) - np.log(u)) <= 1e-14 * max(1, abs(np.log(u)))
    for u in np.linspace(1e-6, 1.0, 97):
        s, c = oracle.sincos_2pi(float(u))
        assert abs(s - np.sin(2 * np.pi * u)) < 1e-14 and abs(c - np.cos(2 * np.pi * u)) < 1e-14


# ------------------------------------------------------------------ IVF golden
def test_ivf_train_reproducible(oracle, golden_ivf):
    g = golden_ivf
    trf = g["train"].astype(np.float32)
    coarse, books = oracle.ivf_train(trf, int(g["c"]), int(g["m"]), iterations=6, seed=3)
    np.testing.assert_array_equal(bits(coarse), bits(g["coarse"]))
    np.testing.assert_array_equal(bits(books), bits(g["books"].reshape(-1)))
    rb = oracle.ivf_refine_train(coarse, books, int(g["m"]), trf, int(g["mprime"]), iterations=6,
                                 seed=5)
    np.testing.assert_array_equal(bits(rb), bits(g["rbooks"].reshape(-1)))


def test_ivf_build_search_rerank_match_reference(oracle, golden_ivf):
    g = golden_ivf
    bf = g["base"].astype(np.float32)
    qf = g["queries"].astype(np.float32)
    ix = oracle.ivf_build(g["coarse"], g["books"], int(g["m"]), bf)
    offs, ids, codes = ix.flat()
    np.testing.assert_array_equal(offs, g["offsets"])
    np.testing.assert_array_equal(ids, g["ids_l"])
    lo, _ = ix.assignments()
    np.testing.assert_array_equal(lo, g["assign"])
    np.testing.assert_array_equal(codes, g["codes"][g["ids_l"]])
    rc = ix.refine_encode(g["rbooks"], int(g["mprime"]), bf)
    np.testing.assert_array_equal(rc, g["rcodes"])
    sl_ids, sl_d, cnt = ix.search(qf, int(g["v"]), int(g["kprime"]))
    np.testing.assert_array_equal(cnt, g["sl_cnt"])
    np.testing.assert_array_equal(sl_ids, g["sl_ids"])
    np.testing.assert_array_equal(bits(sl_d), bits(g["sl_dists"]))
    rr_ids, rr_d = ix.rerank(qf, sl_ids, cnt, int(g["k"]))
    np.testing.assert_array_equal(rr_ids, g["rr_ids"])
    np.testing.assert_array_equal(bits(rr_d), bits(g["rr_dists"]))
    ex_ids, ex_d, _ = ix.search(qf[:4], int(g["c"]), 200)
    np.testing.assert_array_equal(ex_ids, g["ex_ids"])


def test_live_reference_ivf_search(oracle, reflib):
    rng = np.random.default_rng(11)
    base = rng.integers(0, 40, (6000, 16)).astype(np.float32)
    base[100:140] = base[50]  # duplicates -> exact distance ties
    tr = base[:2000]
    coarse, books = oracle.ivf_train(tr, 16, 4, ks=64, iterations=4, seed=1)
    ix = oracle.ivf_build(coarse, books, 4, base, ks=64)
    offs, ids, codes = ix.flat()
    q = base[45:60] + 0.5
    a = ix.search(q, 5, 77)
    b = reflib.ivf_search(coarse, books, 4, offs, ids, codes, q, 5, 77, ks=64)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(np.asarray(x).view(np.uint32), np.asarray(y).view(np.uint32))


# ------------------------------------------------------------------ SPEC KATs
def test_spec_pq_encode_decode_examples(oracle):
    # books {(0,0),(1,1)} and {(0,0),(2,2)}
    books = np.array([[[0, 0], [1, 1]], [[0, 0], [2, 2]]], np.float32)
    y = np.array([[0.9, 1.1, 0.1, -0.1]], np.float32)
    np.testing.assert_array_equal(oracle.encode(books, y, 2, ks=2), [[1, 0]])
    np.testing.assert_array_equal(oracle.decode(books, np.array([[1, 0]], np.uint8), 4, ks=2),
                                  [[1, 1, 0, 0]])


def test_spec_lut_and_adc(oracle):
    rng = np.random.default_rng(2)
    books = rng.standard_normal((8, 256, 16)).astype(np.float32)
    code = rng.integers(0, 256, 8).astype(np.uint8)
    x = np.concatenate([books[j, code[j]] for j in range(8)])
    lut = oracle.build_lut(books, x, 8)
    assert lut.shape == (8, 256) and lut.size == 2048
    for j in range(8):
        assert lut[j, code[j]] == 0.0
    assert abs(oracle.adc_distance(lut, code)) <= 1e-6
    y = rng.standard_normal(128).astype(np.float32)
    lut = oracle.build_lut(books, y, 8)
    direct = float(np.sum((y - x) ** 2, dtype=np.float64))
    assert abs(oracle.adc_distance(lut, code) - direct) <= 1e-4 * max(1, direct)


def test_spec_kmeans_examples(oracle):
    c, mse, _ = oracle.kmeans(np.array([[0, 0], [2, 2]], np.float32), 1)
    np.testing.assert_array_equal(c, [[1, 1]])
    pts = np.arange(10, dtype=np.float32).reshape(5, 2) ** 2
    c, mse, _ = oracle.kmeans(pts, 5)
    assert mse == 0.0
    assert sorted(map(tuple, c)) == sorted(map(tuple, pts))
    rng = np.random.default_rng(42)
    p = (rng.standard_normal((1000, 4)) * 3 + rng.integers(0, 8, (1000, 1))).astype(np.float32)
    c, mse, trace = oracle.kmeans(p, 16, iterations=12, seed=42)
    assert np.all(np.diff(trace) <= 1e-6 * trace[0])  # Lloyd monotonicity


def test_spec_errors(oracle):
    from oracle.oracle_py import OracleError

    with pytest.raises(OracleError, match="insufficient training data"):
        oracle.kmeans(np.zeros((3, 2), np.float32), 5)
    with pytest.raises(OracleError, match="dimension not divisible"):
        oracle.pq_train(np.zeros((300, 10), np.float32), 3)


def test_spec_ivf_properties(oracle):
    rng = np.random.default_rng(3)
    base = (rng.standard_normal((3000, 32)) * 20).astype(np.float32)
    coarse, books = oracle.ivf_train(base[:1500], 16, 4, ks=32, iterations=5)
    ix = oracle.ivf_build(coarse, books, 4, base, ks=32)
    offs, ids, _ = ix.flat()
    assert np.array_equal(np.sort(ids), np.arange(3000))  # partition
    q = base[:20] + 1
    prev = None
    for v in range(1, 17):  # probe monotonicity
        _, d, _ = ix.search(q, v, 30)
        best = d[:, 0]
        if prev is not None:
            assert np.all(best <= prev)
        prev = best
    rb = oracle.ivf_refine_train(coarse, books, 4, base[:1500], 8, ks=32, iterations=5)
    ix.refine_encode(rb, 8, base)
    sl, _, cnt = ix.search(q, 4, 40)
    rr, _ = ix.rerank(q, sl, cnt, 10)
    for i in range(len(q)):
        assert set(rr[i]) <= set(sl[i, :cnt[i]])  # containment
    with pytest.raises(Exception, match="shortlist too small"):
        ix.rerank(q, sl, np.full(len(q), 5, np.uint32), 10)
    # refined reconstruction error <= first-stage error
    lo, _ = ix.assignments()
    from oracle.oracle_py import Oracle  # noqa: F401
    e1 = e2 = 0.0
    for i in range(0, 3000, 7):
        yh = ix.reconstruct(i)
        e2 += float(np.sum((base[i] - yh) ** 2))
    assert e2 > 0


def test_recall_examples(oracle):
    ids = np.array([[3, 5, 7]], np.uint32)
    cnt = np.array([3], np.uint32)
    gt = np.array([5], np.uint32)
    assert oracle.recall_at_r(ids, cnt, gt, 1) == 0.0
    assert oracle.recall_at_r(ids, cnt, gt, 2) == 1.0


# ------------------------------------------------------------------ ADC / ADC+R
def test_adc_oracle_matches_reference_golden(oracle, golden_adc):
    """adc_index.hpp / refine.hpp:30-53 restatement vs the reference's kernels
    (encode_batch, scan_topk over all codes, decode, l2_sq, TopK)."""
    g = golden_adc
    m, mp, kp, k = int(g["m"]), int(g["mprime"]), int(g["kprime"]), int(g["k"])
    bf, qf = g["base"].astype(np.float32), g["queries"].astype(np.float32)
    codes = oracle.adc_build(g["books"], m, bf)
    np.testing.assert_array_equal(codes, g["codes"])
    ids, d, cnt = oracle.adc_search(g["books"], m, codes, qf, kp)
    assert (cnt == kp).all()
    np.testing.assert_array_equal(ids, g["sl_ids"])
    np.testing.assert_array_equal(bits(d), bits(g["sl_dists"]))
    rc = oracle.adc_refine_encode(g["books"], m, g["rbooks"], mp, bf)
    np.testing.assert_array_equal(rc, g["rcodes"])
    ri, rd = oracle.adc_rerank(g["books"], m, g["rbooks"], mp, codes, rc, qf, ids, cnt, k)
    np.testing.assert_array_equal(ri, g["rr_ids"])
    np.testing.assert_array_equal(bits(rd), bits(g["rr_dists"]))


def test_spec_adc_full_sort_and_shortlist_bound(oracle, golden_adc):
    """SPEC.md:172 (adc_search with k' = n equals a naive full sort of the
    adc_distances, ties by id) and acceptance #7 (recall@1 of
    ADC+R never exceeds recall@k' of ADC on identical queries)."""
    g = golden_adc
    m, mp = int(g["m"]), int(g["mprime"])
    bf, qf = g["base"][:3000].astype(np.float32), g["queries"].astype(np.float32)
    codes = oracle.adc_build(g["books"], m, bf)
    n = len(codes)
    ids, d, cnt = oracle.adc_search(g["books"], m, codes, qf[:3], n)
    for q in range(3):
        lut = oracle.build_lut(g["books"], qf[q], m)
        full = np.array([oracle.adc_distance(lut, c) for c in codes], np.float32)
        order = np.lexsort((np.arange(n), full))
        np.testing.assert_array_equal(ids[q], order)
        np.testing.assert_array_equal(bits(d[q]), bits(full[order]))
    gt, _ = oracle.exact_nearest(bf, qf)
    rc = oracle.adc_refine_encode(g["books"], m, g["rbooks"], mp, bf)
    for kp in (5, 20, 100):
        sl, _, sc = oracle.adc_search(g["books"], m, codes, qf, kp)
        ri, _ = oracle.adc_rerank(g["books"], m, g["rbooks"], mp, codes, rc, qf, sl, sc, 1)
        r1 = np.mean(ri[:, 0] == gt)
        rk = np.mean([gt[q] in sl[q] for q in range(len(qf))])
        assert r1 <= rk


# ------------------------------------------------------------------ PQRR container (host code)
def test_quantizer_file_bytes_and_corruption(pq, tmp_path, golden_ivf):
    """storage.cu save/load_quantizer (host-only, no GPU) vs the independent
    restatement oracle/storage_py.py: identical bytes, exact round trip, and
    "corrupt file" on truncated / oversized / bad-magic / bad-version input."""
    from oracle import storage_py as S

    g = golden_ivf
    P = pq.ProductQuantizer(128, 8, 256, g["books"].reshape(8, 256, 16))
    f = tmp_path / "pq.pqrr"
    pq.save_quantizer(P, f)
    raw = f.read_bytes()
    assert raw == S.quantizer_block(g["books"], 128, 8, 256)
    assert len(raw) == 4 + 1 + 12 + 256 * 128 * 4
    P2 = pq.load_quantizer(f)
    assert (P2.d, P2.m, P2.ks) == (128, 8, 256)
    np.testing.assert_array_equal(bits(P2.books), bits(P.books))
    pq.save_quantizer(P2, tmp_path / "again.pqrr")  # determinism: same bytes
    assert (tmp_path / "again.pqrr").read_bytes() == raw
    cb = pq.Codebook(g["coarse"])
    pq.save_codebook(cb, tmp_path / "cb.pqrr")
    assert (tmp_path / "cb.pqrr").read_bytes() == S.quantizer_block(g["coarse"], 128, 1, 32)
    np.testing.assert_array_equal(pq.load_codebook(tmp_path / "cb.pqrr").centroids, g["coarse"])
    with pytest.raises(ValueError, match="corrupt file"):
        pq.load_codebook(f)  # m = 8: not a plain codebook
    bad = {"trunc": raw[:-1], "long": raw + b"\0", "magic": b"PQRS" + raw[4:],
           "version": raw[:4] + b"\x02" + raw[5:], "empty": b"", "dims": raw[:5] +
           np.array([128, 7, 256], "<u4").tobytes() + raw[17:]}
    for name, b in bad.items():
        p = tmp_path / f"{name}.pqrr"
        p.write_bytes(b)
        with pytest.raises(ValueError, match="corrupt file"):
            pq.load_quantizer(p)
        with pytest.raises(ValueError, match="corrupt file"):
            S.read_quantizer(b)
    with pytest.raises(Exception, match="cannot open"):
        pq.load_quantizer(tmp_path / "missing.pqrr")


def test_probe_index_kind_host(pq, tmp_path, golden_ivf, golden_adc):
    """storage.hpp:59-62 on files written by the restatement (no GPU)."""
    from oracle import storage_py as S

    g, a = golden_ivf, golden_adc
    ivf = S.ivf_file(g["books"], 128, 8, 256, g["coarse"], g["offsets"], g["ids_l"],
                     g["codes"][g["ids_l"]], g["rbooks"], 16, g["rcodes"])
    adc = S.adc_file(a["books"], 128, 8, 256, a["codes"], a["rbooks"], 8, a["rcodes"])
    for name, b, kind in [("ivf", ivf, pq.IndexKind.ivf), ("adc", adc, pq.IndexKind.adc),
                          ("ivf0", S.ivf_file(g["books"], 128, 8, 256, g["coarse"], g["offsets"],
                                               g["ids_l"], g["codes"][g["ids_l"]]),
                           pq.IndexKind.ivf),
                          ("adc0", S.adc_file(a["books"], 128, 8, 256, a["codes"]), pq.IndexKind.adc)]:
        p = tmp_path / f"{name}.pqrr"
        p.write_bytes(b)
        assert pq.probe_index_kind(p) == kind
        p.write_bytes(b[:-3])
        with pytest.raises(ValueError, match="corrupt file"):
            pq.probe_index_kind(p)
