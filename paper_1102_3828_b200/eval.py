"""Ground truth and recall (eval.hpp:13-27) on the device: exact k-NN of u8
vectors on the integer tensor cores (k_exact.cu), ties by id."""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from ._lib import check, lib
from .ivf import DEFAULT_DEVICE, SearchResult, _vectorset


@dataclass
class GroundTruth:
    """dataset_io.hpp:66-74: k neighbour ids (and distances) per query."""
    k: int
    ids: np.ndarray    # (nq, k) int32
    dists: np.ndarray  # (nq, k) float32

    def nq(self) -> int:
        return self.ids.shape[0]

    def nearest(self, q: int) -> int:
        return int(self.ids[q, 0])

    def row(self, q: int) -> np.ndarray:
        return self.ids[q]


def _u8(a, d=None) -> np.ndarray:
    a = _vectorset(a, d)
    if a.dtype != np.uint8:
        if not np.all((a >= 0) & (a <= 255) & (np.asarray(a) == np.round(a))):
            raise ValueError("the device ground truth takes u8 vectors")
        a = a.astype(np.uint8)
    return np.ascontiguousarray(a)


def _knn(base: Optional[np.ndarray], queries, k: int, device: int, synth=None):
    q = _u8(queries, 128)
    nq = q.shape[0]
    ids = np.zeros((nq, k), np.uint32)
    d = np.zeros((nq, k), np.float32)
    cnt = np.zeros(nq, np.uint32)
    if synth is None:
        b = _u8(base, 128)
        check(lib.pqrr_dev_exact_knn_u8(device, b.ctypes.data, b.shape[0], q, nq, 128, k, ids, d, cnt))
    else:
        seed, clusters, row0, n = synth
        check(lib.pqrr_dev_exact_knn_synthetic(device, seed, clusters, row0, n, q, nq, k, ids, d, cnt))
    return ids, d, cnt


def exact_search(base, x, k: int, device: int = DEFAULT_DEVICE) -> SearchResult:
    """eval.hpp:15: min(k, n) true nearest neighbours under (dist, id)."""
    ids, d, cnt = _knn(base, _vectorset(x), k, device)
    return SearchResult(ids[0, :cnt[0]].copy(), d[0, :cnt[0]].copy())


def compute_groundtruth(base, queries, k: int, device: int = DEFAULT_DEVICE) -> GroundTruth:
    """eval.hpp:18-19 (k > n returns n entries)."""
    ids, d, cnt = _knn(base, queries, k, device)
    kk = int(cnt.min()) if len(cnt) else 0
    return GroundTruth(kk, ids[:, :kk].astype(np.int32), d[:, :kk].copy())


def groundtruth_synthetic(seed: int, clusters: int, n: int, queries, k: int, row0: int = 0,
                          device: int = DEFAULT_DEVICE) -> GroundTruth:
    """compute_groundtruth over rows [row0, row0 + n) of the synthetic base set,
    generated on the device (1B-scale ground truth without a host copy)."""
    ids, d, cnt = _knn(None, queries, k, device, synth=(seed, clusters, row0, n))
    kk = int(cnt.min()) if len(cnt) else 0
    return GroundTruth(kk, ids[:, :kk].astype(np.int32), d[:, :kk].copy())


def recall_at_r(results: List[SearchResult], gt: GroundTruth, r: int) -> float:
    """eval.hpp:21-25: share of queries whose true nearest neighbour is within
    the first min(r, |result|) entries."""
    if not results:
        return 0.0
    hit = sum(int(gt.nearest(q)) in set(res.ids[:r].tolist()) for q, res in enumerate(results))
    return hit / len(results)
