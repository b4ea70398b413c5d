"""GPU parity suite: the CUDA path (through the C ABI) against the golden
vectors produced by the reference's own code and against the CPU oracle on the
same seeded inputs.  Integer/index outputs must be bit-exact; float distances
too (the arithmetic contract makes them identical)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def pqobj(pq, books, m, d=128, ks=256):
    books = np.asarray(books, np.float32).reshape(m, ks, d // m)
    return pq.ProductQuantizer(d, m, ks, books)


# ------------------------------------------------------------------ kernel seam
def test_assign_batch_golden(pq, golden_ivf):
    g = golden_ivf
    a, d = pq.kernels.assign_batch(g["base"].astype(np.float32), g["coarse"])
    np.testing.assert_array_equal(a, g["assign"])
    np.testing.assert_array_equal(bits(d), bits(g["assign_dist"]))


def test_assign_batch_ties_and_dims(pq, oracle):
    rng = np.random.default_rng(7)
    for d in [4, 8, 12, 16, 24, 32, 64, 128, 130]:
        pts = rng.integers(0, 6, (777, d)).astype(np.float32)
        cen = rng.integers(0, 6, (67, d)).astype(np.float32)
        cen[9] = cen[2]
        a1, d1 = pq.kernels.assign_batch(pts, cen)
        a2, d2 = oracle.assign(pts, cen)
        np.testing.assert_array_equal(a1, a2)
        np.testing.assert_array_equal(bits(d1), bits(d2))


def test_encode_decode_lut_golden(pq, golden_ivf, oracle):
    g = golden_ivf
    bf = g["base"].astype(np.float32)
    res = bf - g["coarse"][g["assign"]]
    P = pqobj(pq, g["books"], 8)
    np.testing.assert_array_equal(pq.kernels.encode_batch(P, res), g["codes"])
    dec = pq.kernels.decode_batch(P, g["codes"][:500])
    np.testing.assert_array_equal(bits(dec), bits(oracle.decode(g["books"], g["codes"][:500], 128)))
    luts = pq.build_lut(P, res[:5])
    for i in range(5):
        np.testing.assert_array_equal(bits(luts[i].values), bits(oracle.build_lut(g["books"], res[i], 8)))


def test_scan_topk_golden(pq, golden_prims):
    g = golden_prims
    lut = pq.LookupTable(g["lut"])
    r = pq.kernels.scan_topk(lut, g["codes"], 100, id_base=7)
    np.testing.assert_array_equal(r.ids, g["scan_ids"])
    np.testing.assert_array_equal(bits(r.dists), bits(g["scan_dists"]))
    r = pq.kernels.scan_topk(lut, g["codes"][:3000], 50)
    np.testing.assert_array_equal(r.ids, g["scan_ids_serial"])


# ------------------------------------------------------------------ generator + training
def test_device_generator_bit_identical(pq, oracle, golden_ivf):
    g = golden_ivf
    base = pq.synth(2, 0, 4000, int(g["clusters"]), seed=int(g["seed"]))
    np.testing.assert_array_equal(base, g["base"])
    centers = oracle.synth_centers(1, 1024, 128)
    for set_id, row0 in [(1, 0), (2, 123_456_789), (3, 9999)]:
        np.testing.assert_array_equal(pq.synth(set_id, row0, 300, 1024, seed=1),
                                      oracle.synth_rows(1, set_id, row0, 300, centers))


def test_kmeans_bit_identical(pq, oracle):
    rng = np.random.default_rng(9)
    p = (rng.standard_normal((5000, 16)) * 7 + rng.integers(0, 5, (5000, 1))).astype(np.float32)
    p[:40] = p[0]  # exact duplicates exercise ties and empty-cluster splits
    for k in [1, 7, 64, 300]:
        tr = []
        cb = pq.kmeans_train(p, k, pq.TrainParams(iterations=8, seed=k, trace=tr))
        c2, mse2, trace2 = oracle.kmeans(p, k, iterations=8, seed=k)
        np.testing.assert_array_equal(bits(cb.centroids), bits(c2))
        assert cb.final_mse == mse2
        np.testing.assert_array_equal(np.array(tr), trace2)


def test_ivf_train_bit_identical(pq, golden_ivf):
    g = golden_ivf
    trf = g["train"].astype(np.float32)
    coarse, P = pq.ivf_train(trf, int(g["c"]), int(g["m"]), params=pq.TrainParams(iterations=6, seed=3))
    np.testing.assert_array_equal(bits(coarse.centroids), bits(g["coarse"]))
    np.testing.assert_array_equal(bits(P.books.reshape(-1)), bits(g["books"]))
    rq = pq.ivf_refine_train(coarse, P, trf, int(g["mprime"]), pq.TrainParams(iterations=6, seed=5))
    np.testing.assert_array_equal(bits(rq.pq.books.reshape(-1)), bits(g["rbooks"]))


# ------------------------------------------------------------------ index: build / search / rerank
def build_small(pq, g, refine=True):
    coarse = pq.Codebook(np.asarray(g["coarse"], np.float32))
    P = pqobj(pq, g["books"], 8)
    rq = pq.RefineQuantizer(pqobj(pq, g["rbooks"], 16)) if refine else None
    return pq.ivf_build(coarse, P, g["base"], rq=rq), coarse, P, rq


def test_ivf_build_layout_golden(pq, golden_ivf):
    g = golden_ivf
    ix, _, _, _ = build_small(pq, g)
    offs, ids, codes, rc = ix.export_lists()
    np.testing.assert_array_equal(offs, g["offsets"])
    np.testing.assert_array_equal(ids, g["ids_l"])
    np.testing.assert_array_equal(codes, g["codes"][g["ids_l"]])
    np.testing.assert_array_equal(rc, g["rcodes"][g["ids_l"]])


def test_ivf_refine_encode_api(pq, golden_ivf):
    g = golden_ivf
    ix, coarse, P, _ = build_small(pq, g, refine=False)
    rq = pq.RefineQuantizer(pqobj(pq, g["rbooks"], 16))
    rc = pq.ivf_refine_encode(ix, rq, g["base"])
    np.testing.assert_array_equal(rc.bytes, g["rcodes"])
    yh = pq.ivf_reconstruct(ix, rq, 17, rc)
    a = int(g["assign"][17])
    B = g["books"].reshape(8, 256, 16)
    R = g["rbooks"].reshape(16, 256, 8)
    p = np.concatenate([B[j, g["codes"][17, j]] for j in range(8)])
    r = np.concatenate([R[j, g["rcodes"][17, j]] for j in range(16)])
    np.testing.assert_array_equal(bits(yh), bits((g["coarse"][a] + p) + r))


def test_search_shortlist_and_rerank_golden(pq, golden_ivf):
    g = golden_ivf
    ix, _, _, _ = build_small(pq, g)
    for q in (g["queries"], g["queries"].astype(np.float32)):
        ids, d, cnt = ix.search(q, int(g["v"]), int(g["kprime"]), 0)
        np.testing.assert_array_equal(cnt, g["sl_cnt"])
        np.testing.assert_array_equal(ids, g["sl_ids"])
        np.testing.assert_array_equal(bits(d), bits(g["sl_dists"]))
        ids, d, cnt = ix.search(q, int(g["v"]), int(g["kprime"]), int(g["k"]))
        np.testing.assert_array_equal(ids, g["rr_ids"])
        np.testing.assert_array_equal(bits(d), bits(g["rr_dists"]))
    # v = c equals the exhaustive scan
    ids, d, _ = ix.search(g["queries"][:4], int(g["c"]), 200, 0)
    np.testing.assert_array_equal(ids, g["ex_ids"])
    np.testing.assert_array_equal(bits(d), bits(g["ex_dists"]))


def test_reference_api_mirror(pq, golden_ivf):
    g = golden_ivf
    ix, coarse, P, rq = build_small(pq, g, refine=False)
    rc = pq.ivf_refine_encode(ix, pq.RefineQuantizer(pqobj(pq, g["rbooks"], 16)), g["base"])
    prm = pq.IvfSearchParams(v=int(g["v"]), kprime=int(g["kprime"]))
    sl = pq.ivf_search_batch(ix, g["queries"], prm)
    one = pq.ivf_search(ix, g["queries"][3], prm)
    np.testing.assert_array_equal(one.ids, sl[3].ids)
    rr = pq.ivf_rerank(g["queries"], sl, ix, ix.rq, rc, int(g["k"]))
    for i in range(len(sl)):
        np.testing.assert_array_equal(rr[i].ids, g["rr_ids"][i])
        np.testing.assert_array_equal(bits(rr[i].dists), bits(g["rr_dists"][i]))
        assert set(rr[i].ids) <= set(sl[i].ids)
    with pytest.raises(ValueError, match="shortlist too small"):
        pq.ivf_rerank(g["queries"][0], pq.SearchResult(sl[0].ids[:5], sl[0].dists[:5]), ix, ix.rq,
                      rc, 10)
    with pytest.raises(ValueError):
        ix.search(g["queries"], 0, 10, 0)
    with pytest.raises(ValueError):
        ix.search(g["queries"], int(g["c"]) + 1, 10, 0)


def test_chunked_add_equals_single_add(pq, golden_ivf):
    g = golden_ivf
    ix, coarse, P, rq = build_small(pq, g)
    ix2 = pq.IvfIndex(coarse, P, rq)
    ix2.add(g["base"][:1000], 0)
    ix2.add(g["base"][1000:2500], 1000)
    ix2.finalize()  # layout built in two rounds: old entries kept, new appended
    ix2.add(g["base"][2500:], 2500)
    for a, b in zip(ix.export_lists(), ix2.export_lists()):
        np.testing.assert_array_equal(a, b)
    with pytest.raises(ValueError):
        ix2.add(g["base"][:10], 5)  # ids must ascend


# ------------------------------------------------------------------ larger: sampled threshold path
@pytest.fixture(scope="module")
def mid_instance(pq, oracle):
    seed, K = 0, 256
    centers = oracle.synth_centers(seed, K, 128)
    base = oracle.synth_rows(seed, 2, 0, 120_000, centers)
    train = oracle.synth_rows(seed, 1, 0, 20_000, centers).astype(np.float32)
    queries = oracle.synth_rows(seed, 3, 0, 64, centers)
    coarse, books = oracle.ivf_train(train, 128, 8, iterations=4, seed=0)
    rbooks = oracle.ivf_refine_train(coarse, books, 8, train, 16, iterations=4, seed=0)
    oix = oracle.ivf_build(coarse, books, 8, base.astype(np.float32))
    oix.refine_encode(rbooks, 16, base.astype(np.float32))
    dix = pq.ivf_build(pq.Codebook(coarse), pqobj(pq, books, 8), base,
                       rq=pq.RefineQuantizer(pqobj(pq, rbooks, 16)))
    return dict(base=base, queries=queries, coarse=coarse, books=books, rbooks=rbooks, oix=oix,
                dix=dix)


@pytest.mark.parametrize("v,kprime,k", [(24, 1000, 100), (8, 100, 10), (40, 300, 300), (3, 2000, 1),
                                        (64, 5000, 100), (40, 10000, 100),
                                        # k' <= 16 over ~15k-38k probed entries (> the 8192 candidate
                                        # buffer): the sampled threshold at stride 1, every entry sampled
                                        (16, 16, 10), (40, 8, 8)])
def test_search_matches_oracle(mid_instance, v, kprime, k):
    oix, dix, q = mid_instance["oix"], mid_instance["dix"], mid_instance["queries"]
    qf = q.astype(np.float32)
    oi, od, oc = oix.search(qf, v, kprime)
    di, dd, dc = dix.search(q, v, kprime, 0)
    np.testing.assert_array_equal(dc, oc)
    for i in range(len(q)):
        n = oc[i]
        np.testing.assert_array_equal(di[i, :n], oi[i, :n])
        np.testing.assert_array_equal(bits(dd[i, :n]), bits(od[i, :n]))
        assert np.all(di[i, n:] == 0xFFFFFFFF) and np.all(np.isinf(dd[i, n:]))
    ri, rd = oix.rerank(qf, oi, oc, k)
    di, dd, dc = dix.search(q, v, kprime, k)
    np.testing.assert_array_equal(di, ri)
    np.testing.assert_array_equal(bits(dd), bits(rd))
    st = dix.last_stats()
    assert st["kernels"] > 5 and st["ms_total"] > 0  # a graph replay (64 queries) reports only the total
    # the synchronising path returns the same bits and per-stage statistics
    dix.set_graph(False)
    try:
        si, sd, sc = dix.search(q, v, kprime, k)
        st = dix.last_stats()
    finally:
        dix.set_graph(True)
    np.testing.assert_array_equal(si, ri)
    np.testing.assert_array_equal(bits(sd), bits(rd))
    assert st["kernels"] > 5 and st["ms_scan"] > 0
    # K4f keeps a superset of the exact candidates (<= tau)
    assert st["exact_candidates"] <= st["candidates"]
    # caller-owned output buffers give the same results
    out = (np.empty((len(q), k), np.uint32), np.empty((len(q), k), np.float32),
           np.empty(len(q), np.uint32))
    oi2, od2, oc2 = dix.search(q, v, kprime, k, out=out)
    assert oi2 is out[0] and od2 is out[1] and oc2 is out[2]
    np.testing.assert_array_equal(out[0], ri)
    np.testing.assert_array_equal(bits(out[1]), bits(rd))
    with pytest.raises(ValueError):
        dix.search(q, v, kprime, k, out=(out[0].astype(np.int64), out[1], out[2]))


def _mid_search_subprocess(**env_over):
    """Runs tools/dbg_filter.py (three mid-size searches against the oracle) in a
    subprocess with the given environment (the switches are read once per
    process) and returns its result lines."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, **env_over)
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "dbg_filter.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if "bad=" in x]
    assert len(lines) == 3, r.stdout
    return lines


def test_exact_scan_fallback_matches_oracle():
    """PQRR_SCAN=exact keeps the fp32 list-major scan."""
    lines = _mid_search_subprocess(PQRR_SCAN="exact")
    assert all("bad=0" in x and "env=exact" in x for x in lines), lines


@pytest.mark.parametrize("scan", ["exact", "filter"])
def test_forced_retries_stay_exact(scan):
    """PQRR_FORCE_RETRY marks every query as failed once (odd: overflow, even:
    under-full).  The retry policy (alpha, denser samples down to stride 1,
    doubled buffer on overflow) must reproduce the oracle exactly; a band
    divisor of 160 additionally forces genuine filter overflows."""
    env = {"PQRR_FORCE_RETRY": "1"}
    if scan == "exact":
        env["PQRR_SCAN"] = "exact"
    lines = _mid_search_subprocess(**env)
    assert all("bad=0" in x for x in lines), lines
    if scan == "filter":
        lines = _mid_search_subprocess(PQRR_BANDDIV="160")
        assert all("bad=0" in x for x in lines), lines
        assert any("retries=0" not in x for x in lines), lines


def test_filter_pass_all_stays_exact():
    """PQRR_FILTER_ALL=1 makes every probed entry of a live pair a K4f
    survivor: it drives the candidate stage through its periodic flushes and
    the direct-append fallback, and the buffers through overflow retries; the
    shortlists must still equal the oracle's."""
    lines = _mid_search_subprocess(PQRR_FILTER_ALL="1")
    assert all("bad=0" in x for x in lines), lines


def test_large_coarse_radix_probe_selection(pq, oracle):
    """Kc > 2048 takes the radix-select top-w path; duplicated centroids force
    exact coarse-distance ties that must resolve to the lowest list index."""
    rng = np.random.default_rng(21)
    base = rng.integers(0, 50, (30000, 128)).astype(np.uint8)
    coarse = base[rng.choice(30000, 4096, replace=False)].astype(np.float32)
    coarse[100:140] = coarse[7]
    books = (rng.standard_normal((8, 256, 16)) * 8).astype(np.float32)
    P = pqobj(pq, books, 8)
    dix = pq.ivf_build(pq.Codebook(coarse), P, base)
    oix = oracle.ivf_build(coarse, books.reshape(-1), 8, base.astype(np.float32))
    q = np.vstack([base[:20], coarse[7:8].astype(np.uint8)])
    for v, kp in [(64, 200), (200, 1000)]:
        oi, od, oc = oix.search(q.astype(np.float32), v, kp)
        di, dd, dc = dix.search(q, v, kp, 0)
        np.testing.assert_array_equal(dc, oc)
        for i in range(len(q)):
            np.testing.assert_array_equal(di[i, :oc[i]], oi[i, :oc[i]])
            np.testing.assert_array_equal(bits(dd[i, :oc[i]]), bits(od[i, :oc[i]]))


@pytest.mark.parametrize("kc", [1024, 2048, 4096])
def test_tensor_core_coarse_certified_probes(pq, oracle, kc):
    """Kc >= 1024 with d = 128 takes the TF32 coarse GEMM + certify path
    (k_coarse_tc.cu).  Fractional centroids make the TF32 rounding real, a
    ragged batch spans several 64-query GEMM tiles, and centroid pairs that
    differ by one ulp in one coordinate put near-ties inside the error bound;
    the probes (hence every shortlist) must still be the exact ones."""
    rng = np.random.default_rng(kc)
    base = rng.integers(0, 120, (30000, 128)).astype(np.uint8)
    coarse = (base[rng.choice(30000, kc, replace=False)].astype(np.float32)
              + rng.standard_normal((kc, 128)).astype(np.float32) * 3.3)
    for a, b in [(11, 900), (12, 901), (13, 1000)]:
        coarse[b] = coarse[a]
        coarse[b, a % 128] = np.nextafter(coarse[a, a % 128], np.float32(np.inf))
    books = (rng.standard_normal((8, 256, 16)) * 6).astype(np.float32)
    dix = pq.ivf_build(pq.Codebook(coarse), pqobj(pq, books, 8), base)
    oix = oracle.ivf_build(coarse, books.reshape(-1), 8, base.astype(np.float32))
    # (more than 256 queries: smaller batches take the exact CUDA-core distances)
    q = np.vstack([base[rng.choice(30000, 300, replace=False)],
                   np.clip(np.rint(coarse[[11, 12, 13]]), 0, 255).astype(np.uint8)])
    # float queries with fractional components (not exact in TF32: the wider
    # error bound applies), one of them half-way between two near-tied centroids
    qf = (q.astype(np.float32) + rng.standard_normal(q.shape).astype(np.float32) * 0.37)
    qf[-1] = (coarse[11] + coarse[900]) * np.float32(0.5)
    for qq in (q, qf):
        for v, kp in [(1, 50), (16, 300), (96, 1000)]:
            oi, od, oc = oix.search(qq.astype(np.float32), v, kp)
            di, dd, dc = dix.search(qq, v, kp, 0)
            np.testing.assert_array_equal(dc, oc)
            for i in range(len(q)):
                np.testing.assert_array_equal(di[i, :oc[i]], oi[i, :oc[i]])
                np.testing.assert_array_equal(bits(dd[i, :oc[i]]), bits(od[i, :oc[i]]))


# ------------------------------------------------------------------ reference-side C++ drop-in
def test_reference_api_shim():
    """integration/test_shim: a caller of the reference's own pqrr:: API
    (compiled against /root/reference headers, prebuilt) linked to the drop-in."""
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration",
                       "build", "test_shim")
    if not os.path.exists(exe):
        pytest.skip("integration/build/test_shim not built (needs the reference headers)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "SHIM OK" in out.stdout, out.stdout + out.stderr


# ------------------------------------------------------------------ K7 merge + list import
def test_merge_topk_kernel_matches_host_merge(pq):
    from paper_1102_3828_b200.sharded import merge_topk_host

    rng = np.random.default_rng(12)
    parts, nq, width, k = 4, 33, 50, 20
    ids = rng.permutation(parts * nq * width).astype(np.uint32).reshape(parts, nq, width)
    d = rng.integers(0, 40, (parts, nq, width)).astype(np.float32)  # many exact ties
    d.sort(axis=2)
    counts = rng.integers(0, width + 1, (parts, nq)).astype(np.uint32)
    counts[:, 0] = 0  # a query with no candidates at all
    oi, od, oc = pq.ivf.merge_topk(ids, d, counts, k)
    ei, ed, ec = merge_topk_host(ids, d, counts, k)
    np.testing.assert_array_equal(oc, ec)
    for q in range(nq):
        n = ec[q]
        np.testing.assert_array_equal(oi[q, :n], ei[q, :n])
        np.testing.assert_array_equal(od[q, :n], ed[q, :n])


def test_load_lists_round_trip(pq, golden_ivf):
    g = golden_ivf
    ix, coarse, P, rq = build_small(pq, g)
    offs, ids, codes, rc = ix.export_lists()
    ix2 = pq.IvfIndex(coarse, P, rq)
    ix2.load_lists(offs, ids, codes, rc)
    for a, b in zip(ix.export_lists(), ix2.export_lists()):
        np.testing.assert_array_equal(a, b)
    a = ix.search(g["queries"], int(g["v"]), int(g["kprime"]), int(g["k"]))
    b = ix2.search(g["queries"], int(g["v"]), int(g["kprime"]), int(g["k"]))
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_massive_boundary_ties_match_oracle(pq, oracle):
    """600 copies of one vector in the base and the same vector as a query: the
    k'-th (and k-th) boundary falls inside > 256 exact distance ties, which the
    selectors must resolve by id exactly like the reference's TopK."""
    seed, K = 3, 64
    centers = oracle.synth_centers(seed, K, 128)
    base = oracle.synth_rows(seed, 2, 0, 30_000, centers)
    train = oracle.synth_rows(seed, 1, 0, 8_000, centers).astype(np.float32)
    dup = base[123].copy()
    base[5000:5600] = dup  # ids 5000..5599 are identical vectors
    queries = np.concatenate([dup[None], oracle.synth_rows(seed, 3, 0, 15, centers)])
    coarse, books = oracle.ivf_train(train, 32, 8, iterations=3, seed=0)
    rbooks = oracle.ivf_refine_train(coarse, books, 8, train, 16, iterations=3, seed=0)
    oix = oracle.ivf_build(coarse, books, 8, base.astype(np.float32))
    oix.refine_encode(rbooks, 16, base.astype(np.float32))
    dix = pq.ivf_build(pq.Codebook(coarse), pqobj(pq, books, 8), base,
                       rq=pq.RefineQuantizer(pqobj(pq, rbooks, 16)))
    qf = queries.astype(np.float32)
    for v, kprime, k in [(4, 300, 100), (32, 300, 250)]:
        oi, od, oc = oix.search(qf, v, kprime)
        ri, rd = oix.rerank(qf, oi, oc, k)
        di, dd, dc = dix.search(queries, v, kprime, k)
        np.testing.assert_array_equal(di, ri)
        np.testing.assert_array_equal(bits(dd), bits(rd))
        # the duplicated query's shortlist is all ties: ids 123, 5000, 5001, ... in order
        expect = np.concatenate([[123], np.arange(5000, 5000 + k - 1)])
        assert np.all(ri[0, :k] == expect)


def test_merge_topk_large_path_matches_sort(pq):
    """K7 above the smem bitonic (parts * width > 25600: exact multi-shard mode
    merges k'-wide shortlists): pack + global radix select + row sort."""
    rng = np.random.default_rng(21)
    parts, nq, width, k = 8, 6, 5000, 3000
    ids = rng.permutation(parts * nq * width).astype(np.uint32).reshape(parts, nq, width)
    d = rng.integers(0, 3000, (parts, nq, width)).astype(np.float32)  # many exact ties
    d.sort(axis=2)
    counts = rng.integers(0, width + 1, (parts, nq)).astype(np.uint32)
    counts[:, 0] = 0
    counts[:, 1] = 100  # fewer candidates than k
    oi, od, oc = pq.ivf.merge_topk(ids, d, counts, k)
    for q in range(nq):
        keys = sorted((float(d[p, q, j]), int(ids[p, q, j])) for p in range(parts)
                      for j in range(counts[p, q]))[:k]
        assert oc[q] == len(keys)
        np.testing.assert_array_equal(oi[q, :len(keys)], np.array([i for _, i in keys], np.uint32))
        np.testing.assert_array_equal(od[q, :len(keys)], np.array([x for x, _ in keys], np.float32))


@pytest.mark.parametrize("nshards,v,kprime,k", [(2, 16, 300, 100), (3, 8, 1000, 50), (2, 40, 10000, 100)])
def test_exact_sharded_mode_equals_single_index(pq, mid_instance, nshards, v, kprime, k):
    """SURVEY §8e exact mode on one GPU: id-range shards (own device indexes,
    global ids), per-shard k' shortlists merged to the global top-k', owned
    re-rank, final merge == the single-index oracle bit for bit."""
    import torch

    from paper_1102_3828_b200.sharded import MultiShardSearch, shard_range

    mi = mid_instance
    base, q = mi["base"], mi["queries"]
    shards = []
    for r in range(nshards):
        lo, hi = shard_range(len(base), r, nshards)
        ix = pq.IvfIndex(pq.Codebook(mi["coarse"]), pqobj(pq, mi["books"], 8),
                         pq.RefineQuantizer(pqobj(pq, mi["rbooks"], 16)))
        ix.add(base[lo:hi], id_base=lo)
        ix.finalize()
        shards.append(ix)
    ms = MultiShardSearch(shards, k, kprime, v, mode="exact")
    dq = torch.from_numpy(q).cuda()
    oi, od, oc = ms.search(dq)
    torch.cuda.synchronize()
    qf = q.astype(np.float32)
    si, _, sc = mi["oix"].search(qf, v, kprime)
    ri, rd = mi["oix"].rerank(qf, si, sc, k)
    np.testing.assert_array_equal(oi.cpu().numpy().view(np.uint32), ri)
    np.testing.assert_array_equal(bits(od.cpu().numpy()), bits(rd))
    assert (oc.cpu().numpy() == k).all()
    # local mode runs too and returns ranked, duplicate-free rows
    li, ld, lc = MultiShardSearch(shards, k, kprime, v, mode="local").search(dq)
    li = li.cpu().numpy()
    for r in range(len(q)):
        assert len(set(li[r].tolist())) == k
    # shortlist ids a shard does not hold are rejected by the explicit re-rank
    from paper_1102_3828_b200._lib import check, lib
    with pytest.raises(Exception, match="not in the index"):
        check(lib.pqrr_dev_rerank_u8(shards[-1].h, np.ascontiguousarray(q[:1]), 1,
                                     np.zeros((1, 1), np.uint32), np.ones(1, np.uint32), 1, 1,
                                     np.zeros((1, 1), np.uint32), np.zeros((1, 1), np.float32)))


@pytest.mark.parametrize("mode", ["exact", "local"])
def test_device_sharded_search_nccl_world1(pq, mid_instance, mode):
    """DeviceShardedSearch through a real NCCL group (world size 1 — gpurun has
    one GPU): all_gather_into_tensor + K7 on the stream; equals the index."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_1102_3828_b200.sharded import DeviceShardedSearch

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        mi = mid_instance
        q = mi["queries"]
        ds = DeviceShardedSearch(mi["dix"], 100, 1000, 24, mode=mode)
        oi, od, oc = ds.search(torch.from_numpy(q).cuda())
        ri, rd, rc = mi["dix"].search(q, 24, 1000, 100)
        np.testing.assert_array_equal(oi.cpu().numpy().view(np.uint32), ri)
        np.testing.assert_array_equal(bits(od.cpu().numpy()), bits(rd))
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------------ ADC / ADC+R (exhaustive)
def test_adc_golden(pq, golden_adc, oracle):
    """adc_build / adc_search_batch / refine_encode / rerank (adc_index.hpp,
    refine.hpp:30-53) on the device == the reference kernels' outputs."""
    g = golden_adc
    m, mp, kp, k = int(g["m"]), int(g["mprime"]), int(g["kprime"]), int(g["k"])
    P = pqobj(pq, g["books"], m)
    R = pq.RefineQuantizer(pqobj(pq, g["rbooks"], mp))
    ix = pq.adc_build(P, g["base"])
    np.testing.assert_array_equal(ix.codes, g["codes"])
    res = pq.adc_search_batch(ix, g["queries"], kp)
    for q, r in enumerate(res):
        np.testing.assert_array_equal(r.ids, g["sl_ids"][q])
        np.testing.assert_array_equal(bits(r.dists), bits(g["sl_dists"][q]))
    one = pq.adc_search(ix, g["queries"][3], kp)
    np.testing.assert_array_equal(one.ids, g["sl_ids"][3])
    codes = pq.refine_encode(ix, R, g["base"])
    np.testing.assert_array_equal(codes.bytes, g["rcodes"])
    rr = pq.rerank(g["queries"], res, ix, R, codes, k)
    for q, r in enumerate(rr):
        np.testing.assert_array_equal(r.ids, g["rr_ids"][q])
        np.testing.assert_array_equal(bits(r.dists), bits(g["rr_dists"][q]))
    # fused ADC+R search (shortlist + re-rank in one call)
    fi, fd, fc = ix.search(g["queries"], kp, k)
    np.testing.assert_array_equal(fi, g["rr_ids"])
    np.testing.assert_array_equal(bits(fd), bits(g["rr_dists"]))
    with pytest.raises(ValueError, match="shortlist too small"):
        pq.rerank(g["queries"][0], pq.SearchResult(res[0].ids[:3], res[0].dists[:3]), ix, R, codes, 4)
    # stand-alone helpers: residual, reconstruct, refine_train
    bf = g["base"][:500].astype(np.float32)
    dec = oracle.decode(g["books"], g["codes"][:500], 128)
    np.testing.assert_array_equal(bits(pq.residual(bf, P)), bits(bf - dec))
    rec = pq.reconstruct(P, R, g["codes"][:500], g["rcodes"][:500])
    for i in (0, 7, 499):
        np.testing.assert_array_equal(bits(rec[i]), bits(oracle.adc_reconstruct(
            g["books"], m, g["rbooks"], mp, g["codes"][i], g["rcodes"][i])))
    tr = g["base"][:4000].astype(np.float32)
    R2 = pq.refine_train(P, tr, 16, pq.TrainParams(iterations=3, seed=4))
    np.testing.assert_array_equal(R2.pq.flat(), oracle.refine_train(g["books"], m, tr, 16,
                                                                    iterations=3, seed=4))


@pytest.mark.parametrize("m,mp,kp,k", [(8, 16, 1000, 100), (8, 8, 300, 50), (8, 32, 5000, 100)])
def test_adc_matches_oracle_large(pq, oracle, mid_instance, m, mp, kp, k):
    """120k-vector exhaustive ADC+R vs the oracle: the single list runs through
    K4f/K4r in 16k-entry work items."""
    mi = mid_instance
    base, q = mi["base"], mi["queries"][:32]
    train = base[:20000].astype(np.float32)
    books = oracle.pq_train(train, m, iterations=3, seed=m)
    rbooks = oracle.refine_train(books, m, train, mp, iterations=3, seed=mp)
    P, R = pqobj(pq, books, m), pq.RefineQuantizer(pqobj(pq, rbooks, mp))
    ix = pq.adc_build(P, base, rq=R)
    bf, qf = base.astype(np.float32), q.astype(np.float32)
    ocodes = oracle.adc_build(books, m, bf)
    np.testing.assert_array_equal(ix.codes, ocodes)
    oi, od, oc = oracle.adc_search(books, m, ocodes, qf, kp)
    di, dd, dc = ix.search(q, kp, 0)
    np.testing.assert_array_equal(di, oi)
    np.testing.assert_array_equal(bits(dd), bits(od))
    orc = oracle.adc_refine_encode(books, m, rbooks, mp, bf)
    np.testing.assert_array_equal(ix.refine_codes.bytes, orc)
    ri, rd = oracle.adc_rerank(books, m, rbooks, mp, ocodes, orc, qf, oi, oc, k)
    fi, fd, _ = ix.search(q, kp, k)
    np.testing.assert_array_equal(fi, ri)
    np.testing.assert_array_equal(bits(fd), bits(rd))


def test_adc_scan_needs_m8(pq, golden_adc):
    """The device scan kernels are specialised to m = 8 (every BASELINE config);
    other m build and encode but fail loudly at search (no CPU fallback)."""
    rng = np.random.default_rng(3)
    books = rng.standard_normal((16, 256, 8)).astype(np.float32)
    ix = pq.adc_build(pqobj(pq, books, 16), golden_adc["base"][:1000])
    assert ix.codes.shape == (1000, 16)
    with pytest.raises(ValueError, match="m = 8"):
        ix.search(golden_adc["queries"], 10, 0)


# ------------------------------------------------------------------ PQRR container (device indexes)
def test_ivf_index_file_round_trip(pq, golden_ivf, tmp_path):
    """save_ivf_index of a device-built index == the restatement's bytes of the
    reference layout (lists id-ascending, refine codes id-aligned); the loaded
    index searches and re-ranks exactly like the golden vectors."""
    from oracle import storage_py as S

    g = golden_ivf
    m, mp = int(g["m"]), int(g["mprime"])
    P, R = pqobj(pq, g["books"], m), pq.RefineQuantizer(pqobj(pq, g["rbooks"], mp))
    ix = pq.ivf_build(pq.Codebook(g["coarse"]), P, g["base"])
    codes = pq.ivf_refine_encode(ix, R, g["base"])
    f = tmp_path / "ivf.pqrr"
    pq.save_ivf_index(ix, R, codes, f)
    raw = f.read_bytes()
    assert raw == S.ivf_file(g["books"], 128, m, 256, g["coarse"], g["offsets"], g["ids_l"],
                             g["codes"][g["ids_l"]], g["rbooks"], mp, g["rcodes"])
    assert pq.probe_index_kind(f) == pq.IndexKind.ivf
    L = pq.load_ivf_index(f)
    np.testing.assert_array_equal(L.refine_codes.bytes, g["rcodes"])
    v, kp, k = int(g["v"]), int(g["kprime"]), int(g["k"])
    si, sd, sc = L.index.search(g["queries"], v, kp, 0)
    for q in range(len(sc)):
        n = sc[q]
        np.testing.assert_array_equal(si[q, :n], g["sl_ids"][q, :n])
    ri, rd, _ = L.index.search(g["queries"], v, kp, k)
    np.testing.assert_array_equal(ri, g["rr_ids"])
    np.testing.assert_array_equal(bits(rd), bits(g["rr_dists"]))
    pq.save_ivf_index(L.index, L.refine_quantizer, L.refine_codes, tmp_path / "again.pqrr")
    assert (tmp_path / "again.pqrr").read_bytes() == raw
    # without refinement
    ix0 = pq.ivf_build(pq.Codebook(g["coarse"]), P, g["base"])
    pq.save_ivf_index(ix0, None, None, tmp_path / "plain.pqrr")
    assert (tmp_path / "plain.pqrr").read_bytes() == S.ivf_file(
        g["books"], 128, m, 256, g["coarse"], g["offsets"], g["ids_l"], g["codes"][g["ids_l"]])
    for cut in (1, 100, len(raw) // 2):
        (tmp_path / "t.pqrr").write_bytes(raw[:-cut])
        with pytest.raises(ValueError, match="corrupt file"):
            pq.load_ivf_index(tmp_path / "t.pqrr")
    # a list whose ids are not ascending is rejected
    hdr = 17 + 256 * 128 * 4 + 4 + 32 * 128 * 4 + 32 * 8
    lens = np.frombuffer(raw[hdr - 32 * 8:hdr], "<u8")
    l0 = int(np.argmax(lens >= 2))
    e0 = hdr + int(lens[:l0].sum()) * (4 + m)
    swapped = bytearray(raw)
    swapped[e0:e0 + 4], swapped[e0 + 12:e0 + 16] = raw[e0 + 12:e0 + 16], raw[e0:e0 + 4]
    (tmp_path / "s.pqrr").write_bytes(bytes(swapped))
    with pytest.raises(ValueError, match="corrupt file"):
        pq.load_ivf_index(tmp_path / "s.pqrr")


def test_adc_index_file_round_trip(pq, golden_adc, tmp_path):
    from oracle import storage_py as S

    g = golden_adc
    m, mp, kp, k = int(g["m"]), int(g["mprime"]), int(g["kprime"]), int(g["k"])
    P, R = pqobj(pq, g["books"], m), pq.RefineQuantizer(pqobj(pq, g["rbooks"], mp))
    ix = pq.adc_build(P, g["base"])
    codes = pq.refine_encode(ix, R, g["base"])
    f = tmp_path / "adc.pqrr"
    pq.save_adc_index(ix, R, codes, f)
    raw = f.read_bytes()
    assert raw == S.adc_file(g["books"], 128, m, 256, g["codes"], g["rbooks"], mp, g["rcodes"])
    assert pq.probe_index_kind(f) == pq.IndexKind.adc
    L = pq.load_adc_index(f)
    np.testing.assert_array_equal(L.index.codes, g["codes"])
    np.testing.assert_array_equal(L.refine_codes.bytes, g["rcodes"])
    fi, fd, _ = L.index.search(g["queries"], kp, k)
    np.testing.assert_array_equal(fi, g["rr_ids"])
    np.testing.assert_array_equal(bits(fd), bits(g["rr_dists"]))
    (tmp_path / "t.pqrr").write_bytes(raw[:-1])
    with pytest.raises(ValueError, match="corrupt file"):
        pq.load_adc_index(tmp_path / "t.pqrr")
    with pytest.raises(ValueError, match="not an ADC index"):
        ivf = pq.ivf_build(pq.Codebook(np.ones((2, 128), np.float32)), P, g["base"][:100])
        pq.save_adc_index(ivf, None, None, tmp_path / "x.pqrr")


def test_export_lists_subset(pq, golden_ivf):
    g = golden_ivf
    ix = pq.ivf_build(pq.Codebook(g["coarse"]), pqobj(pq, g["books"], 8), g["base"],
                      rq=pq.RefineQuantizer(pqobj(pq, g["rbooks"], 16)))
    offs, ids, codes, rc = ix.export_lists()
    sub = np.array([5, 0, 31, 7], np.uint32)
    so, si, sc, sr = ix.export_lists_subset(sub)
    for i, l in enumerate(sub):
        a, b = offs[l], offs[l + 1]
        np.testing.assert_array_equal(si[so[i]:so[i + 1]], ids[a:b])
        np.testing.assert_array_equal(sc[so[i]:so[i + 1]], codes[a:b])
        np.testing.assert_array_equal(sr[so[i]:so[i + 1]], rc[a:b])


def test_far_pair_bound_is_a_certified_lower_bound(pq, oracle, mid_instance):
    """k_bound.cu (two-phase LUT pass): the tensor-core bound never exceeds the
    exact fp32 sum of the LUT minima (the quantity the live-pair test uses),
    for u8 and fractional queries, and stays tight (it only selects work)."""
    from paper_1102_3828_b200._lib import check, lib

    mi = mid_instance
    coarse, books = mi["coarse"], mi["books"]
    rng = np.random.default_rng(5)
    for qs in (mi["queries"][:24].astype(np.float32),
               (mi["queries"][:24] + rng.standard_normal((24, 128)) * 3.7).astype(np.float32)):
        nq, w, R1 = len(qs), 40, 5
        probes, _ = oracle.coarse_probe(coarse, qs, w)
        out = np.zeros(nq * w, np.float32)
        check(lib.pqrr_dev_pair_bounds(0, np.ascontiguousarray(qs), nq, 128, coarse, coarse.shape[0],
                                       np.ascontiguousarray(books, np.float32).reshape(-1), 8, 256,
                                       np.ascontiguousarray(probes, np.uint32).reshape(-1), w, R1, out))
        out = out.reshape(nq, w)
        ratios = []
        for q in range(nq):
            for r in range(R1, w):
                lut = oracle.build_lut(books, qs[q] - coarse[probes[q, r]], 8).reshape(8, 256)
                sm = np.float32(0)
                for j in range(8):
                    sm = np.float32(sm + lut[j].min())
                assert out[q, r] <= sm, (q, r, out[q, r], sm)
                ratios.append(out[q, r] / sm)
        assert np.all(out[:, :R1] == 0)
        assert np.median(ratios) > 0.98


def test_exact_knn_groundtruth(pq, oracle, mid_instance):
    """compute_groundtruth / exact_search (eval.hpp:13-19) on the integer tensor
    cores == a float64 brute force under (dist, id), incl. duplicated base rows
    (ties broken by id), k > n, and the device-generated base set."""
    mi = mid_instance
    base, q = mi["base"][:30000].copy(), mi["queries"][:40]
    base[777] = base[5]  # exact ties
    base[20001] = q[3]   # distance 0
    gt = pq.compute_groundtruth(base, q, 50)
    bf, qf = base.astype(np.float64), q.astype(np.float64)
    d = (qf * qf).sum(1)[:, None] + (bf * bf).sum(1)[None, :] - 2 * qf @ bf.T
    for i in range(len(q)):
        order = np.lexsort((np.arange(len(base)), d[i]))[:50]
        np.testing.assert_array_equal(gt.ids[i], order)
        np.testing.assert_array_equal(gt.dists[i], d[i, order].astype(np.float32))
    nn, _ = oracle.exact_nearest(base.astype(np.float32), q.astype(np.float32))
    np.testing.assert_array_equal(gt.ids[:, 0], nn)
    g1 = pq.compute_groundtruth(base, q, 1)  # k = 1: the fused-argmin path
    np.testing.assert_array_equal(g1.ids[:, 0], nn)
    np.testing.assert_array_equal(g1.dists[:, 0], gt.dists[:, 0])
    assert pq.groundtruth_synthetic(0, 256, 120_000, q, 1).ids[:, 0].tolist() == \
        pq.compute_groundtruth(mi["base"], q, 1).ids[:, 0].tolist()
    one = pq.exact_search(base, q[7], 3)
    np.testing.assert_array_equal(one.ids, gt.ids[7, :3])
    small = pq.compute_groundtruth(base[:20], q[:2], 50)  # k > n returns n entries
    assert small.k == 20
    gs = pq.groundtruth_synthetic(0, 256, 120_000, q, 10)
    full = pq.compute_groundtruth(mi["base"], q, 10)
    np.testing.assert_array_equal(gs.ids, full.ids)
    res = [pq.SearchResult(full.ids[i, :10].astype(np.uint32), full.dists[i, :10]) for i in range(len(q))]
    assert pq.recall_at_r(res, full, 1) == 1.0


# ------------------------------------------------------------------ round 2: tensor-core add path
def _near_tie_centroids(rng, rows, k):
    """Centroids that put many rows inside the certification window: pairs of
    centroids mirrored about a row (equal distances, or within a few ulps),
    exact duplicates, and ordinary k-means-like means."""
    cen = rng.uniform(0, 120, (k, 128)).astype(np.float32)
    for j in range(0, k // 4, 2):  # mirrored pairs around row j: exact or near ties
        r = rows[j].astype(np.float32)
        delta = rng.uniform(-3, 3, 128).astype(np.float32)
        cen[j] = r + delta
        cen[j + 1] = r - delta
        if j % 4 == 2:
            cen[j + 1] = np.nextafter(cen[j + 1], np.float32(1e9))
    cen[k // 2] = cen[k // 2 + 1]  # exact duplicate: ties go to the lower index
    cen[k // 2 + 2:k // 2 + 8] = cen[k // 2 + 2]  # 6 copies: overflow path
    return cen


@pytest.mark.parametrize("k", [128, 1024, 8192])
def test_assign_u8_tensor_core_equals_reference(pq, reflib, k):
    """tcgen05 add-path assignment (k_assign_tc.cu) vs the reference's own
    kernels::assign_batch (kernels.cpp:21-39) on the widened rows."""
    rng = np.random.default_rng(100 + k)
    n = 20_000 + 77  # ragged last tile
    rows = rng.integers(0, 256, (n, 128)).astype(np.uint8)
    rows[:300] = rows[0]  # repeated rows
    cen = _near_tie_centroids(rng, rows, k)
    # rows sitting exactly between the mirrored pairs
    for j in range(0, k // 4, 2):
        rows[1000 + j] = np.clip(np.rint((cen[j] + cen[j + 1]) / 2), 0, 255).astype(np.uint8)
    # rows equal to the duplicated centroids (rounded): many candidates
    rows[2000:2100] = np.clip(np.rint(cen[k // 2 + 2]), 0, 255).astype(np.uint8)
    got = pq.kernels.assign_u8(rows, cen)
    want, _ = reflib.assign(rows.astype(np.float32), cen)
    np.testing.assert_array_equal(got, want)


def test_assign_u8_other_shapes_exact(pq, reflib):
    rng = np.random.default_rng(5)
    rows = rng.integers(0, 256, (3000, 64)).astype(np.uint8)
    cen = rng.uniform(0, 255, (100, 64)).astype(np.float32)
    np.testing.assert_array_equal(pq.kernels.assign_u8(rows, cen), reflib.assign(rows.astype(np.float32), cen)[0])


@pytest.mark.parametrize("nshards", [2, 3])
def test_index_group_exact_equals_single_index(pq, mid_instance, nshards):
    """pqrr_dev_group_* (one process, several id-range shards; here all on one
    GPU, so the all-gathers are device copies): exact mode equals the
    single-index oracle bit for bit; local mode equals MultiShardSearch's."""
    import torch

    from paper_1102_3828_b200.sharded import IndexGroup, MultiShardSearch, shard_range

    mi = mid_instance
    base, q = mi["base"], mi["queries"]
    shards = []
    for r in range(nshards):
        lo, hi = shard_range(len(base), r, nshards)
        ix = pq.IvfIndex(pq.Codebook(mi["coarse"]), pqobj(pq, mi["books"], 8),
                         pq.RefineQuantizer(pqobj(pq, mi["rbooks"], 16)))
        ix.add(base[lo:hi], id_base=lo)
        ix.finalize()
        shards.append(ix)
    qf = q.astype(np.float32)
    for v, kprime, k in [(8, 300, 50), (32, 2000, 100)]:
        g = IndexGroup(shards, "exact")
        assert not g.uses_nccl()
        gi, gd, gc = g.search(q, v, kprime, k)
        si, _, sc = mi["oix"].search(qf, v, kprime)
        ri, rd = mi["oix"].rerank(qf, si, sc, k)
        np.testing.assert_array_equal(gi, ri)
        np.testing.assert_array_equal(bits(gd), bits(rd))
        assert (gc == k).all()
        # shortlists only (k = 0): the global IVFADC top-k'
        si2, sd2, sc2 = g.search(q, v, kprime, 0)
        np.testing.assert_array_equal(sc2, sc)
        for r in range(len(q)):
            np.testing.assert_array_equal(si2[r, :sc[r]], si[r, :sc[r]])
        g.close()
        lg = IndexGroup(shards, "local")
        li, ld, lc = lg.search(q, v, kprime, k)
        mi_, md_, mc_ = MultiShardSearch(shards, k, kprime, v, mode="local").search(torch.from_numpy(q).cuda())
        np.testing.assert_array_equal(li, mi_.cpu().numpy().view(np.uint32))
        np.testing.assert_array_equal(bits(ld), bits(md_.cpu().numpy()))
        lg.close()
    g = IndexGroup(shards, "exact")
    with pytest.raises(ValueError, match="shortlist too small"):
        g.search(q[:4], 1, 5, 100)
    g.close()


def test_two_phase_search_large_batch_matches_oracle(pq, mid_instance, oracle):
    """A batch large enough for the two-phase LUT pass (query-list pairs >=
    64 x SMs): far probes go through the tcgen05 far-pair bound (k_bound.cu)
    and, at Kc = 128, the coarse distances through the tcgen05 D~ kernel;
    shortlists and re-ranked lists must equal the oracle's bit for bit."""
    from oracle.oracle_py import Oracle

    o = Oracle()
    centers = o.synth_centers(0, 256, 128)
    q = o.synth_rows(0, 3, 1000, 320, centers)
    oix, dix = mid_instance["oix"], mid_instance["dix"]
    qf = q.astype(np.float32)
    for v, kprime, k in [(40, 1000, 100), (96, 300, 50)]:
        oi, od, oc = oix.search(qf, v, kprime)
        ri, rd = oix.rerank(qf, oi, oc, k)
        di, dd, dc = dix.search(q, v, kprime, k)
        np.testing.assert_array_equal(di, ri)
        np.testing.assert_array_equal(bits(dd), bits(rd))
        si, sd, sc = dix.search(q, v, kprime, 0)
        np.testing.assert_array_equal(sc, oc)
        for i in range(len(q)):
            np.testing.assert_array_equal(si[i, :oc[i]], oi[i, :oc[i]])


@pytest.mark.parametrize("nq,v,kprime,k", [(1, 24, 1000, 100), (5, 8, 100, 10), (64, 64, 5000, 100),
                                           (300, 40, 1000, 100), (16, 40, 8, 8), (7, 16, 300, 0)])
def test_graph_replay_equals_oracle(pq, mid_instance, oracle, nq, v, kprime, k):
    """Small batches run as one captured CUDA graph (host-side bounds instead
    of count readbacks, a device status word instead of the retry round trip).
    The capture call and the replays — with different queries in the same
    buffers — must equal the oracle bit for bit, and the graph must hold the
    whole search (no kernel launched outside it on a replay)."""
    from oracle.oracle_py import Oracle

    o = Oracle()
    centers = o.synth_centers(0, 256, 128)
    oix, dix = mid_instance["oix"], mid_instance["dix"]
    for rep in range(3):
        q = o.synth_rows(0, 3, 5000 + 1000 * rep, nq, centers)
        qf = q.astype(np.float32)
        oi, od, oc = oix.search(qf, v, kprime)
        l0 = pq.launch_count()
        di, dd, dc = dix.search(q, v, kprime, k)
        launched = pq.launch_count() - l0
        # a replay launches exactly the captured kernels (a batch whose status
        # word flags a failed threshold is redone on the synchronising path,
        # which reports stage times)
        if rep and dix.last_stats()["ms_scan"] == 0:
            assert launched == dix.last_stats()["kernels"], launched
        if k:
            ri, rd = oix.rerank(qf, oi, oc, k)
            np.testing.assert_array_equal(di, ri)
            np.testing.assert_array_equal(bits(dd), bits(rd))
        else:
            np.testing.assert_array_equal(dc, oc)
            for i in range(nq):
                np.testing.assert_array_equal(di[i, :oc[i]], oi[i, :oc[i]])
                np.testing.assert_array_equal(bits(dd[i, :oc[i]]), bits(od[i, :oc[i]]))
        st = dix.last_stats()
        assert st["ms_total"] > 0  # (a graph replay times only the total; a flagged batch is redone with stage times)


def test_enqueue_finish_device_api(pq, mid_instance, oracle):
    """pqrr_dev_search_u8_enqueue launches the captured search without blocking;
    pqrr_dev_search_finish returns the blocking call's outcome: the same bits,
    'shortlist too small' when k exceeds a row's candidates, and
    NotImplementedError for a batch outside the envelope."""
    import torch

    oix, dix, q = mid_instance["oix"], mid_instance["dix"], mid_instance["queries"]
    v, kprime, k = 24, 1000, 100
    qf = q.astype(np.float32)
    oi, od, oc = oix.search(qf, v, kprime)
    ri, rd = oix.rerank(qf, oi, oc, k)
    dq = torch.from_numpy(q).cuda()
    ids = torch.zeros((len(q), k), dtype=torch.int32, device="cuda")
    dists = torch.zeros((len(q), k), dtype=torch.float32, device="cuda")
    cnt = torch.zeros(len(q), dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        ids.zero_()
        dix.search_enqueue(dq.data_ptr(), len(q), v, kprime, k, ids.data_ptr(), dists.data_ptr(),
                           cnt.data_ptr(), st)
        with pytest.raises(ValueError, match="pending"):
            dix.search_enqueue(dq.data_ptr(), len(q), v, kprime, k, ids.data_ptr(), dists.data_ptr(),
                               cnt.data_ptr(), st)
        dix.search_finish()
        torch.cuda.synchronize()
        np.testing.assert_array_equal(ids.cpu().numpy().view(np.uint32), ri)
        np.testing.assert_array_equal(bits(dists.cpu().numpy()), bits(rd))
    dix.search_finish()  # nothing pending: a no-op
    # a row with fewer than k candidates: the error arrives at finish
    big = torch.zeros((len(q), 3000), dtype=torch.int32, device="cuda")
    bigd = torch.zeros((len(q), 3000), dtype=torch.float32, device="cuda")
    dix.search_enqueue(dq.data_ptr(), len(q), 1, 3000, 3000, big.data_ptr(), bigd.data_ptr(),
                       cnt.data_ptr(), st)
    with pytest.raises(ValueError, match="shortlist too small"):
        dix.search_finish()
    many = torch.zeros((2000, 128), dtype=torch.uint8, device="cuda")
    with pytest.raises(NotImplementedError):
        dix.search_enqueue(many.data_ptr(), 2000, v, kprime, 0, ids.data_ptr(), dists.data_ptr(),
                           cnt.data_ptr(), st)


def test_large_batch_warp_selections_match_oracle(pq, mid_instance, oracle):
    """A batch that fills the GPU with warps (>= 2 x 148 x 8 queries) takes the
    warp-per-query kernels: the single-pass threshold (each lane keeps its 8
    smallest samples; k_wselect.cu), the warp top-w / shortlist / top-k
    selections.  Shortlists and re-ranked lists must equal the oracle's."""
    from oracle.oracle_py import Oracle

    o = Oracle()
    centers = o.synth_centers(0, 256, 128)
    q = o.synth_rows(0, 3, 20000, 2400, centers)
    oix, dix = mid_instance["oix"], mid_instance["dix"]
    qf = q.astype(np.float32)
    for v, kprime, k in [(24, 300, 50), (8, 1000, 100)]:
        oi, od, oc = oix.search(qf, v, kprime)
        ri, rd = oix.rerank(qf, oi, oc, k)
        di, dd, dc = dix.search(q, v, kprime, k)
        np.testing.assert_array_equal(di, ri)
        np.testing.assert_array_equal(bits(dd), bits(rd))
        st = dix.last_stats()
        assert st["ms_threshold"] > 0  # the synchronising path (more than 1024 queries)


@pytest.mark.parametrize("graph", [True, False])
def test_narrow_lut_pass_many_lanes_per_list(pq, mid_instance, oracle, graph):
    """Small batches (no more query-list pairs than lists) take the narrow LUT
    pass (k_lutnarrow.cu: code book resident, two query lanes per LUT).  Seven
    copies of two queries put up to 14 lanes on every probed list, so items
    run through several lane pairs, odd lane counts included; shortlists
    (every list sampled at k' = 8: stride 1) and re-ranked lists must equal
    the oracle's on both search paths."""
    oix, dix = mid_instance["oix"], mid_instance["dix"]
    q = np.repeat(mid_instance["queries"][:2], 7, axis=0)[:13]
    qf = q.astype(np.float32)
    dix.set_graph(graph)
    try:
        for v, kprime, k in [(16, 300, 50), (19, 8, 8), (3, 2000, 100)]:
            assert len(q) * v <= 256
            oi, od, oc = oix.search(qf, v, kprime)
            ri, rd = oix.rerank(qf, oi, oc, min(k, int(oc.min())))
            di, dd, dc = dix.search(q, v, kprime, min(k, int(oc.min())))
            np.testing.assert_array_equal(di, ri)
            np.testing.assert_array_equal(bits(dd), bits(rd))
            si, sd, sc = dix.search(q, v, kprime, 0)
            np.testing.assert_array_equal(sc, oc)
            for i in range(len(q)):
                np.testing.assert_array_equal(si[i, :oc[i]], oi[i, :oc[i]])
                np.testing.assert_array_equal(bits(sd[i, :oc[i]]), bits(od[i, :oc[i]]))
    finally:
        dix.set_graph(True)


def test_graph_cache_eviction_and_recapture(pq, mid_instance, oracle):
    """More batch shapes than the index caches graphs for (16): the least
    recently used graph is destroyed (its graph memory trimmed) and a shape
    that comes back is captured again; every search still equals the oracle."""
    oix, dix, q = mid_instance["oix"], mid_instance["dix"], mid_instance["queries"]
    v, kprime = 8, 100
    oi, od, oc = oix.search(q.astype(np.float32), v, kprime)
    for rnd in range(2):
        for nq in range(1, 21):
            di, dd, dc = dix.search(q[:nq], v, kprime, 0)
            np.testing.assert_array_equal(dc, oc[:nq])
            for i in range(nq):
                np.testing.assert_array_equal(di[i, :oc[i]], oi[i, :oc[i]])
                np.testing.assert_array_equal(bits(dd[i, :oc[i]]), bits(od[i, :oc[i]]))
