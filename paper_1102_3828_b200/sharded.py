"""Multi-GPU IVFADC+R: id-range sharding, one process per GPU (north star).

Every rank holds all Kc inverted lists over its id range
[n*rank/world, n*(rank+1)/world) — the add path needs no communication, since
each rank generates/encodes its own rows.  A search replicates the query batch,
each rank runs the fused search on its shard, the per-rank top-k (id, dist)
lists are all-gathered, and K7 merges them under (dist, id)
(types.hpp:47-50).  Ids are global, so the merge is a pure k-way merge.

Two modes:

* ``"local"`` — the north star's literal flow: each shard keeps its own top-k'
  shortlist, so up to world*k' candidates are re-ranked (results can only be
  as good as or better than one index with one k' shortlist).
* ``"exact"`` — reproduces the single index (ivf_search_batch + ivf_rerank,
  ivf_index.hpp:58-64,79-81) bit for bit: every shard returns its local top-k'
  IVFADC shortlist; the all-gathered shortlists are merged to the global top-k'
  (the union's k' smallest under (dist, id) are the single index's shortlist,
  because an entry's ADC distance does not depend on which shard holds it);
  each shard re-ranks the global-shortlist entries it holds; a second
  all-gather + merge of the per-shard top-k gives the final list.  Cost: one
  extra all-gather of Q*k'*8 B per rank.

The collective is torch.distributed (NCCL over NVLink on GPUs; gloo in the
CPU tests, which plug an oracle searcher into ``local_search``).
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import numpy as np


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    return n * rank // world, n * (rank + 1) // world


def merge_topk_host(ids: np.ndarray, dists: np.ndarray, counts: np.ndarray, k: int):
    """Reference (numpy) merge of [parts, nq, width] ranked lists — used by the
    CPU multi-process tests; the GPU path uses the K7 kernel (merge_topk)."""
    parts, nq, width = ids.shape
    out_i = np.full((nq, k), 0xFFFFFFFF, np.uint32)
    out_d = np.full((nq, k), np.inf, np.float32)
    out_c = np.zeros(nq, np.uint32)
    for q in range(nq):
        cand = []
        for p in range(parts):
            c = int(counts[p, q])
            cand.extend(zip(dists[p, q, :c].tolist(), ids[p, q, :c].tolist()))
        cand.sort(key=lambda t: (np.float32(t[0]), t[1]))
        cand = cand[:k]
        out_c[q] = len(cand)
        for j, (d, i) in enumerate(cand):
            out_i[q, j] = i
            out_d[q, j] = d
    return out_i, out_d, out_c


class ShardedSearch:
    """Host orchestration of one rank.

    local mode: local_search(queries) -> (ids[nq, width], dists[nq, width],
    counts[nq]), the shard's re-ranked top-k (the product passes
    IvfIndex.search; tests pass an oracle).
    exact mode: local_search returns the shard's IVFADC shortlist (width k'),
    and local_rerank(queries, sl_ids, sl_counts) re-ranks the global-shortlist
    entries the shard holds -> (ids[nq, k], dists[nq, k], counts[nq]).
    ``merge`` defaults to the numpy merge (the GPU path uses the K7 kernel).
    """

    def __init__(self, local_search: Callable, width: int, group=None,
                 merge: Optional[Callable] = None, mode: str = "local",
                 local_rerank: Optional[Callable] = None, kprime: int = 0):
        import torch.distributed as dist

        if mode not in ("local", "exact"):
            raise ValueError(f"unknown sharded mode {mode!r}")
        if mode == "exact" and (local_rerank is None or kprime <= 0):
            raise ValueError("exact mode needs local_rerank and kprime")
        self.dist = dist
        self.group = group
        self.local_search = local_search
        self.local_rerank = local_rerank
        self.width = width
        self.kprime = kprime
        self.mode = mode
        self.world = dist.get_world_size(group)
        self.merge = merge or merge_topk_host

    def search(self, queries):
        if self.mode == "local":
            return self._gather_merge(*self.local_search(queries), self.width)
        sl_i, sl_d, sl_c = self._gather_merge(*self.local_search(queries), self.kprime)
        if len(sl_c) and int(sl_c.min()) < self.width:
            raise ValueError("shortlist too small")  # SPEC.md:256, as one index would
        return self._gather_merge(*self.local_rerank(queries, sl_i, sl_c), self.width)

    def _gather_merge(self, ids, dists, counts, k):
        import torch

        ti = torch.from_numpy(np.ascontiguousarray(ids).view(np.int32))
        td = torch.from_numpy(np.ascontiguousarray(dists, np.float32))
        tc = torch.from_numpy(np.ascontiguousarray(counts).view(np.int32))
        gi = [torch.empty_like(ti) for _ in range(self.world)]
        gd = [torch.empty_like(td) for _ in range(self.world)]
        gc = [torch.empty_like(tc) for _ in range(self.world)]
        self.dist.all_gather(gi, ti, group=self.group)
        self.dist.all_gather(gd, td, group=self.group)
        self.dist.all_gather(gc, tc, group=self.group)
        all_i = np.stack([g.numpy().view(np.uint32) for g in gi])
        all_d = np.stack([g.numpy() for g in gd])
        all_c = np.stack([g.numpy().view(np.uint32) for g in gc])
        return self.merge(all_i, all_d, all_c, k)


def _merge_device(all_i, all_d, all_c, k, stream):
    """K7 on stacked [parts, nq, width] device tensors -> top-k (ids, dists, counts)."""
    import torch

    from ._lib import check, lib

    parts, nq, width = all_i.shape
    dev = all_i.device
    out_i = torch.empty((nq, k), dtype=torch.int32, device=dev)
    out_d = torch.empty((nq, k), dtype=torch.float32, device=dev)
    out_c = torch.empty(nq, dtype=torch.int32, device=dev)
    check(lib.pqrr_dev_merge_topk_device(dev.index, all_i.data_ptr(), all_d.data_ptr(),
                                         all_c.data_ptr(), nq, parts, width, k, out_i.data_ptr(),
                                         out_d.data_ptr(), out_c.data_ptr(), stream.cuda_stream))
    return out_i, out_d, out_c


def _local_search(ix, d_queries, w, kprime, k, stream):
    """One shard's fused search; k = 0 returns its IVFADC shortlist (width k')."""
    import torch

    nq, dev = d_queries.shape[0], d_queries.device
    width = k or kprime
    i = torch.empty((nq, width), dtype=torch.int32, device=dev)
    d = torch.empty((nq, width), dtype=torch.float32, device=dev)
    c = torch.empty(nq, dtype=torch.int32, device=dev)
    ix.search_device(d_queries.data_ptr(), nq, w, kprime, k, i.data_ptr(), d.data_ptr(),
                     c.data_ptr(), stream.cuda_stream)
    return i, d, c


def _rerank_owned(ix, d_queries, sl_i, sl_c, k, stream):
    import torch

    nq, dev = d_queries.shape[0], d_queries.device
    i = torch.empty((nq, k), dtype=torch.int32, device=dev)
    d = torch.empty((nq, k), dtype=torch.float32, device=dev)
    c = torch.empty(nq, dtype=torch.int32, device=dev)
    ix.rerank_owned_device(d_queries.data_ptr(), nq, sl_i.data_ptr(), sl_c.data_ptr(),
                           sl_i.shape[1], k, i.data_ptr(), d.data_ptr(), c.data_ptr(),
                           stream.cuda_stream)
    return i, d, c


def _check_shortlist(sl_c, k):
    if sl_c.numel() and int(sl_c.min()) < k:
        raise ValueError("shortlist too small")  # SPEC.md:256, as one index would


def _packed(nq, width, dev):
    """One rank's search output as ONE buffer, [ids nq x width | dists nq x
    width | counts nq] 32-bit words, so a merge needs a single all-gather
    (pqrr_dev_merge_packed_device); returns (buffer, ids, dists, counts) views."""
    import torch

    buf = torch.empty(2 * nq * width + nq, dtype=torch.int32, device=dev)
    ids = buf[:nq * width].view(nq, width)
    dists = buf[nq * width:2 * nq * width].view(torch.float32).view(nq, width)
    counts = buf[2 * nq * width:]
    return buf, ids, dists, counts


class DeviceShardedSearch:
    """GPU rank: device-resident queries; each search writes its rows straight
    into a packed buffer, ONE NCCL all-gather per merge, and the K7 merge
    kernel on the same stream (mode as in the module docstring).  The
    collectives run with `stream` current, so they are ordered after the
    shard's search whichever stream the caller passes.  Exact mode's
    "shortlist too small" check reads the shortlist counts back only after
    the whole batch is enqueued."""

    def __init__(self, index, k: int, kprime: int, w: int, group=None, mode: str = "local"):
        import torch
        import torch.distributed as dist

        if mode not in ("local", "exact"):
            raise ValueError(f"unknown sharded mode {mode!r}")
        self.ix, self.k, self.kprime, self.w, self.mode = index, k, kprime, w, mode
        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.torch = torch

    def _gather_merge(self, buf, nq, width, k, stream):
        torch = self.torch
        dev = buf.device
        allb = torch.empty((self.world, buf.numel()), dtype=torch.int32, device=dev)
        with torch.cuda.stream(stream):
            self.dist.all_gather_into_tensor(allb, buf, group=self.group)
        out_i = torch.empty((nq, k), dtype=torch.int32, device=dev)
        out_d = torch.empty((nq, k), dtype=torch.float32, device=dev)
        out_c = torch.empty(nq, dtype=torch.int32, device=dev)
        from ._lib import check, lib

        check(lib.pqrr_dev_merge_packed_device(dev.index, allb.data_ptr(), nq, self.world, width, k,
                                               out_i.data_ptr(), out_d.data_ptr(), out_c.data_ptr(),
                                               stream.cuda_stream))
        return out_i, out_d, out_c

    def search(self, d_queries, stream=None):
        """d_queries: uint8 CUDA tensor [nq, d] -> (ids, dists, counts) CUDA tensors."""
        stream = stream or self.torch.cuda.current_stream(d_queries.device)
        nq, dev = d_queries.shape[0], d_queries.device
        if self.mode == "local":
            buf, i, d, c = _packed(nq, self.k, dev)
            self.ix.search_device(d_queries.data_ptr(), nq, self.w, self.kprime, self.k, i.data_ptr(),
                                  d.data_ptr(), c.data_ptr(), stream.cuda_stream)
            return self._gather_merge(buf, nq, self.k, self.k, stream)
        buf, i, d, c = _packed(nq, self.kprime, dev)
        self.ix.search_device(d_queries.data_ptr(), nq, self.w, self.kprime, 0, i.data_ptr(),
                              d.data_ptr(), c.data_ptr(), stream.cuda_stream)
        sl_i, _, sl_c = self._gather_merge(buf, nq, self.kprime, self.kprime, stream)
        buf2, i2, d2, c2 = _packed(nq, self.k, dev)
        self.ix.rerank_owned_device(d_queries.data_ptr(), nq, sl_i.data_ptr(), sl_c.data_ptr(),
                                    self.kprime, self.k, i2.data_ptr(), d2.data_ptr(), c2.data_ptr(),
                                    stream.cuda_stream)
        out = self._gather_merge(buf2, nq, self.k, self.k, stream)
        with self.torch.cuda.stream(stream):
            short = (sl_c.min() < self.k) if sl_c.numel() else None
        if short is not None and bool(short):
            raise ValueError("shortlist too small")  # SPEC.md:256, as one index would
        return out


class MultiShardSearch:
    """Several id-range shards on ONE device in one process (more shards than
    GPUs, or the one-GPU parity test of the sharded flow): the same steps as
    DeviceShardedSearch with the all-gather replaced by a device-side stack."""

    def __init__(self, indexes, k: int, kprime: int, w: int, mode: str = "exact"):
        import torch

        if mode not in ("local", "exact"):
            raise ValueError(f"unknown sharded mode {mode!r}")
        self.ixs, self.k, self.kprime, self.w, self.mode = list(indexes), k, kprime, w, mode
        self.torch = torch

    def _stack_merge(self, parts, k, stream):
        t = self.torch
        return _merge_device(t.stack([p[0] for p in parts]), t.stack([p[1] for p in parts]),
                             t.stack([p[2] for p in parts]), k, stream)

    def search(self, d_queries, stream=None):
        stream = stream or self.torch.cuda.current_stream(d_queries.device)
        if self.mode == "local":
            return self._stack_merge([_local_search(ix, d_queries, self.w, self.kprime, self.k,
                                                    stream) for ix in self.ixs], self.k, stream)
        sl_i, _, sl_c = self._stack_merge([_local_search(ix, d_queries, self.w, self.kprime, 0,
                                                         stream) for ix in self.ixs],
                                          self.kprime, stream)
        _check_shortlist(sl_c, self.k)
        return self._stack_merge([_rerank_owned(ix, d_queries, sl_i, sl_c, self.k, stream)
                                  for ix in self.ixs], self.k, stream)


class IndexGroup:
    """One process driving several id-range shards (pqrr_dev_group_*): NCCL
    all-gathers when the shards sit on distinct GPUs, device copies when they
    share one.  mode "exact" (default) is bit-identical to one index holding
    every id; "local" merges each shard's fused top-k."""

    MODES = {"exact": 0, "local": 1}

    def __init__(self, shards, mode: str = "exact"):
        import ctypes as C

        from ._lib import check, lib

        if mode not in self.MODES:
            raise ValueError(f"unknown group mode {mode!r}")
        self.shards, self.mode = list(shards), mode
        arr = (C.c_void_p * len(self.shards))(*[s.h.value for s in self.shards])
        self.h = C.c_void_p()
        check(lib.pqrr_dev_group_create(len(self.shards), arr, C.byref(self.h)))

    def uses_nccl(self) -> bool:
        import ctypes as C

        from ._lib import check, lib

        n, u = C.c_uint32(), C.c_int()
        check(lib.pqrr_dev_group_size(self.h, C.byref(n), C.byref(u)))
        return bool(u.value)

    def search(self, queries, v: int, kprime: int, k: int = 0, out=None):
        """u8 host queries [nq, d] -> (ids, dists, counts), rows of k (k' if k = 0)."""
        from ._lib import check, lib

        q = np.ascontiguousarray(queries, np.uint8)
        nq, width = q.shape[0], (k or kprime)
        if out is None:
            out = (np.zeros((nq, width), np.uint32), np.zeros((nq, width), np.float32),
                   np.zeros(nq, np.uint32))
        ids, dists, counts = out
        check(lib.pqrr_dev_group_search_u8(self.h, q, nq, v, kprime, k, self.MODES[self.mode], ids, dists,
                                           counts))
        return ids, dists, counts

    def close(self):
        from ._lib import lib

        if getattr(self, "h", None) and self.h.value:
            lib.pqrr_dev_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
