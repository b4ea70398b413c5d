"""The reference-side harness of bench.py's parity legs (oracle/ref_harness.py),
on the CPU: the host-built index equals the oracle's ivf_build + refine encode,
the reference search equals the oracle's search + re-rank, the probed-list
path equals the full-index search, and the add-path re-encode sample equals
the host index."""
import numpy as np

from oracle import ref_harness as H
from oracle.oracle_py import Oracle, RefLib


def test_ref_harness_matches_oracle(reflib):
    cfg = dict(n=30000, train=6000, nq=50, clusters=64, kc=64, m=8, mprime=16, w=8, kprime=200, k=50)
    hx = H.cpu_build(cfg, 0, None, chunk=7000)
    o = Oracle()
    centers = o.synth_centers(0, 64, 128)
    base = o.synth_rows(0, 2, 0, cfg['n'], centers).astype(np.float32)
    oix = o.ivf_build(hx.coarse, hx.books, 8, base)
    oix.refine_encode(hx.rbooks, 16, base)
    offs, ids, codes = oix.flat()
    assert np.array_equal(offs, hx.offs) and np.array_equal(ids, hx.ids) and np.array_equal(codes, hx.codes)
    assert np.array_equal(oix.rcodes, hx.rcodes_by_id)
    q = o.synth_rows(0, 3, 0, cfg['nq'], centers)
    ref = RefLib(); ref.set_threads(0)
    ri, rd, _ = H.ref_search(ref, hx, q, cfg['w'], cfg['kprime'], cfg['k'])
    sl, _, sc = oix.search(q.astype(np.float32), cfg['w'], cfg['kprime'])
    oi, od = oix.rerank(q.astype(np.float32), sl, sc, cfg['k'])
    assert np.array_equal(ri, oi) and np.array_equal(rd.view(np.uint32), od.view(np.uint32))
    # probed path with an export function from the host index
    def export_subset(U):
        o_ = [0]; I=[]; Cc=[]; R=[]
        for l in U:
            a, b = int(hx.offs[l]), int(hx.offs[l+1])
            I.append(hx.ids[a:b]); Cc.append(hx.codes[a:b]); R.append(hx.rcodes_by_id[hx.ids[a:b]]); o_.append(o_[-1]+b-a)
        return np.array(o_, np.uint64), np.concatenate(I), np.concatenate(Cc), np.concatenate(R)
    pi, pd, ts, nl = H.probed_reference(ref, export_subset, hx.coarse, hx.books, hx.rbooks, 8, 16, 64, q, cfg['w'], cfg['kprime'], cfg['k'], batch=16)
    assert np.array_equal(pi, oi) and np.array_equal(pd.view(np.uint32), od.view(np.uint32)), (pi[:2], oi[:2])
    starts, block = H.sample_ids(cfg['n'], nblocks=4, block=100)
    sid, a, c, rc = H.reencode_sample(cfg, hx.coarse, hx.books, hx.rbooks, starts, block)
    assert np.array_equal(a, hx.list_of_id[sid]) and np.array_equal(c, hx.codes_by_id[sid]) and np.array_equal(rc, hx.rcodes_by_id[sid])
    assert H.host_cores() >= 1 and H.cpu_model()


def test_reference_arm_file_lists(tmp_path):
    """bench.FileLists: the reference arm's view of the lists a setup process
    exported (no product code loaded) returns each requested list's rows."""
    import bench

    U = np.array([3, 7, 9], np.uint32)
    offs = np.array([0, 2, 5, 6], np.uint64)
    ids = np.array([1, 4, 2, 3, 8, 5], np.uint32)
    codes = np.arange(48, dtype=np.uint8).reshape(6, 8)
    rc = np.arange(96, dtype=np.uint8).reshape(6, 16)
    for name, a in (("lists", U), ("offs", offs), ("ids", ids), ("codes", codes), ("rcodes", rc)):
        np.save(tmp_path / f"{name}.npy", a)
    fl = bench.FileLists(str(tmp_path))
    o, i, c, r = fl(np.array([9, 3], np.uint32))
    np.testing.assert_array_equal(o, [0, 1, 3])
    np.testing.assert_array_equal(i, [5, 1, 4])
    np.testing.assert_array_equal(c[:, 0], [40, 0, 8])
    np.testing.assert_array_equal(r[:, 0], [80, 0, 16])
    assert fl.nbytes() > 0
