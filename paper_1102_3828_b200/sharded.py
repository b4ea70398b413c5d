"""Multi-GPU IVFADC+R: id-range sharding, one process per GPU (north star).

Every rank holds all Kc inverted lists over its id range
[n*rank/world, n*(rank+1)/world) — the add path needs no communication, since
each rank generates/encodes its own rows.  A search replicates the query batch,
each rank runs the fused search on its shard, the per-rank top-k (id, dist)
lists are all-gathered, and K7 merges them under (dist, id)
(types.hpp:47-50).  Ids are global, so the merge is a pure k-way merge.

This is the north star's "local mode": each shard keeps its own top-k'
shortlist, so up to world*k' candidates are re-ranked (results can only be
as good as or better than one index with one k' shortlist).

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

    local_search(queries) -> (ids[nq, width], dists[nq, width], counts[nq]) for
    this rank's shard (the product passes IvfIndex.search; tests pass an
    oracle).  ``merge`` defaults to the device K7 kernel when a GPU is used.
    """

    def __init__(self, local_search: Callable, width: int, group=None,
                 merge: Optional[Callable] = None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.local_search = local_search
        self.width = width
        self.world = dist.get_world_size(group)
        self.merge = merge or merge_topk_host

    def search(self, queries):
        import torch

        ids, dists, counts = self.local_search(queries)
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
        return self.merge(all_i, all_d, all_c, self.width)


class DeviceShardedSearch:
    """GPU rank: device-resident queries, NCCL all-gather into one buffer and
    the K7 merge kernel on the same stream."""

    def __init__(self, index, k: int, kprime: int, w: int, group=None):
        import torch
        import torch.distributed as dist

        self.ix, self.k, self.kprime, self.w = index, k, kprime, w
        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.torch = torch

    def search(self, d_queries, stream=None):
        """d_queries: uint8 CUDA tensor [nq, d] -> (ids, dists, counts) CUDA tensors."""
        from ._lib import check, lib

        torch = self.torch
        nq = d_queries.shape[0]
        k = self.k
        dev = d_queries.device
        stream = stream or torch.cuda.current_stream(dev)
        loc_i = torch.empty((nq, k), dtype=torch.int32, device=dev)
        loc_d = torch.empty((nq, k), dtype=torch.float32, device=dev)
        loc_c = torch.empty(nq, dtype=torch.int32, device=dev)
        self.ix.search_device(d_queries.data_ptr(), nq, self.w, self.kprime, k, loc_i.data_ptr(),
                              loc_d.data_ptr(), loc_c.data_ptr(), stream.cuda_stream)
        all_i = torch.empty((self.world, nq, k), dtype=torch.int32, device=dev)
        all_d = torch.empty((self.world, nq, k), dtype=torch.float32, device=dev)
        all_c = torch.empty((self.world, nq), dtype=torch.int32, device=dev)
        self.dist.all_gather_into_tensor(all_i, loc_i, group=self.group)
        self.dist.all_gather_into_tensor(all_d, loc_d, group=self.group)
        self.dist.all_gather_into_tensor(all_c, loc_c, group=self.group)
        out_i = torch.empty((nq, k), dtype=torch.int32, device=dev)
        out_d = torch.empty((nq, k), dtype=torch.float32, device=dev)
        out_c = torch.empty(nq, dtype=torch.int32, device=dev)
        check(lib.pqrr_dev_merge_topk_device(dev.index, all_i.data_ptr(), all_d.data_ptr(),
                                             all_c.data_ptr(), nq, self.world, k, k,
                                             out_i.data_ptr(), out_d.data_ptr(), out_c.data_ptr(),
                                             stream.cuda_stream))
        return out_i, out_d, out_c
