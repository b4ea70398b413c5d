"""CPU multi-process tests of the id-range sharded search (world_size 2, gloo):
the host orchestration, the all-gather and the (dist, id) merge.  The
per-shard searcher is the CPU oracle (test infrastructure); the GPU path
swaps in IvfIndex.search + the K7 merge kernel (tests/test_gpu_parity.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _instance():
    from oracle.oracle_py import Oracle

    o = Oracle()
    o.set_threads(2)
    rng = np.random.default_rng(4)
    base = (rng.integers(0, 30, (6000, 16)) + rng.integers(0, 40, (1, 16))).astype(np.float32)
    base[3000:3010] = base[10]  # duplicates straddling the shard boundary -> ties by id
    coarse, books = o.ivf_train(base[:2000], 12, 4, ks=32, iterations=4, seed=1)
    rbooks = o.ivf_refine_train(coarse, books, 4, base[:2000], 8, ks=32, iterations=4, seed=2)
    queries = base[5:25] + 0.25
    return o, base, coarse, books, rbooks, queries


def _shard_search(o, base, coarse, books, rbooks, queries, lo, hi, v, kprime, k):
    ix = o.ivf_build(coarse, books, 4, base[lo:hi], ks=32)
    ix.refine_encode(rbooks, 8, base[lo:hi])
    sl, _, cnt = ix.search(queries, v, kprime)
    ids, d = ix.rerank(queries, sl, cnt, min(k, int(cnt.min())))
    counts = np.full(len(queries), ids.shape[1], np.uint32)
    return ids + np.uint32(lo), d, counts


def _shard_shortlist(o, base, coarse, books, queries, lo, hi, v, kprime):
    ix = o.ivf_build(coarse, books, 4, base[lo:hi], ks=32)
    sl, d, cnt = ix.search(queries, v, kprime)
    return sl + np.uint32(lo), d, cnt


def _shard_rerank_owned(o, base, coarse, books, rbooks, queries, lo, hi, sl_ids, sl_cnt, k):
    """Oracle stand-in for pqrr_dev_rerank_owned_u8_device: re-rank the entries of
    the global shortlist this shard holds, top-min(k, owned) per query."""
    ix = o.ivf_build(coarse, books, 4, base[lo:hi], ks=32)
    ix.refine_encode(rbooks, 8, base[lo:hi])
    nq = len(queries)
    ids = np.full((nq, k), 0xFFFFFFFF, np.uint32)
    d = np.full((nq, k), np.inf, np.float32)
    cnt = np.zeros(nq, np.uint32)
    for q in range(nq):
        row = sl_ids[q, :sl_cnt[q]]
        own = row[(row >= lo) & (row < hi)] - np.uint32(lo)
        if len(own) == 0:
            continue
        kk = min(k, len(own))
        ri, rd = ix.rerank(queries[q:q + 1], own[None, :], np.array([len(own)], np.uint32), kk)
        ids[q, :kk], d[q, :kk], cnt[q] = ri[0] + np.uint32(lo), rd[0], kk
    return ids, d, cnt


def _worker_exact(rank, world, port, v, kprime, k, out_path):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1102_3828_b200.sharded import ShardedSearch, shard_range

    o, base, coarse, books, rbooks, queries = _instance()
    lo, hi = shard_range(len(base), rank, world)
    ss = ShardedSearch(
        lambda q: _shard_shortlist(o, base, coarse, books, q, lo, hi, v, kprime), width=k,
        mode="exact", kprime=kprime,
        local_rerank=lambda q, si, sc: _shard_rerank_owned(o, base, coarse, books, rbooks, q, lo, hi,
                                                           si, sc, k))
    try:
        ids, d, c = ss.search(queries)
        res = dict(ids=ids, d=d, c=c)
    except ValueError as e:
        res = dict(err=np.array(str(e)))
    if rank == 0:
        np.savez(out_path, **res)
    dist.barrier()
    dist.destroy_process_group()


def _worker(rank, world, port, v, kprime, k, out_path):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1102_3828_b200.sharded import ShardedSearch, shard_range

    o, base, coarse, books, rbooks, queries = _instance()
    lo, hi = shard_range(len(base), rank, world)
    ss = ShardedSearch(lambda q: _shard_search(o, base, coarse, books, rbooks, q, lo, hi, v, kprime,
                                               k), width=k)
    ids, d, c = ss.search(queries)
    if rank == 0:
        np.savez(out_path, ids=ids, d=d, c=c)
    dist.barrier()
    dist.destroy_process_group()


def _run(tmp_path, v, kprime, k, worker=_worker, world=2):
    out = str(tmp_path / "res.npz")
    mp.spawn(worker, args=(world, _free_port(), v, kprime, k, out), nprocs=world, join=True)
    return dict(np.load(out))


def test_sharded_merge_equals_per_shard_oracle(tmp_path):
    from paper_1102_3828_b200.sharded import merge_topk_host, shard_range

    v, kprime, k = 4, 40, 10
    res = _run(tmp_path, v, kprime, k)
    o, base, coarse, books, rbooks, queries = _instance()
    parts = [_shard_search(o, base, coarse, books, rbooks, queries, *shard_range(6000, r, 2), v,
                           kprime, k) for r in range(2)]
    ei, ed, ec = merge_topk_host(np.stack([p[0] for p in parts]), np.stack([p[1] for p in parts]),
                                 np.stack([p[2] for p in parts]), k)
    np.testing.assert_array_equal(res["ids"], ei)
    np.testing.assert_array_equal(res["d"].view(np.uint32), ed.view(np.uint32))
    for q in range(len(queries)):  # ascending (dist, id), no duplicates
        keys = list(zip(res["d"][q].tolist(), res["ids"][q].tolist()))
        assert keys == sorted(keys) and len(set(res["ids"][q])) == k


def test_sharded_equals_single_index_when_shortlists_are_complete(tmp_path):
    """With k' covering every candidate, local mode reranks the same set as one
    index, so the merged top-k equals the single-index oracle exactly."""
    v, kprime, k = 3, 6000, 10
    res = _run(tmp_path, v, kprime, k)
    o, base, coarse, books, rbooks, queries = _instance()
    ix = o.ivf_build(coarse, books, 4, base, ks=32)
    ix.refine_encode(rbooks, 8, base)
    sl, _, cnt = ix.search(queries, v, kprime)
    ri, rd = ix.rerank(queries, sl, cnt, k)
    np.testing.assert_array_equal(res["ids"], ri)
    np.testing.assert_array_equal(res["d"].view(np.uint32), rd.view(np.uint32))


@pytest.mark.parametrize("world,v,kprime,k", [(2, 4, 40, 10), (2, 2, 25, 25), (3, 5, 60, 7)])
def test_exact_mode_equals_single_index_oracle(tmp_path, world, v, kprime, k):
    """Exact mode (global top-k' shortlist, owned re-rank, final merge)
    reproduces ONE index's ivf_search_batch + ivf_rerank bit for bit, with
    k' far below the candidate count (where local mode may differ)."""
    res = _run(tmp_path, v, kprime, k, worker=_worker_exact, world=world)
    o, base, coarse, books, rbooks, queries = _instance()
    ix = o.ivf_build(coarse, books, 4, base, ks=32)
    ix.refine_encode(rbooks, 8, base)
    sl, _, cnt = ix.search(queries, v, kprime)
    ri, rd = ix.rerank(queries, sl, cnt, k)
    np.testing.assert_array_equal(res["ids"], ri)
    np.testing.assert_array_equal(res["d"].view(np.uint32), rd.view(np.uint32))
    assert (res["c"] == k).all()


def test_exact_mode_shortlist_too_small(tmp_path):
    res = _run(tmp_path, 1, 5, 6, worker=_worker_exact)
    assert "shortlist too small" in str(res["err"])
