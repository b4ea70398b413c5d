"""pqrr::kernels (kernels.hpp:13-43) on the device: the link-time hot-kernel
seam of the reference, one batch per call."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, lib
from .ivf import DEFAULT_DEVICE, LookupTable, ProductQuantizer, SearchResult, _f32, _vectorset


def set_threads(t: int) -> None:
    """kernels.hpp:16 — thread caps do not apply to the device; accepted for API parity."""


def max_threads() -> int:
    return 1


def assign_batch(points, centroids, device: int = DEFAULT_DEVICE):
    """kernels.hpp:23-25 -> (assign u32[n], dist f32[n]); ties to the lowest index."""
    p = _f32(_vectorset(points))
    c = _f32(_vectorset(centroids, p.shape[1]))
    n = p.shape[0]
    a = np.zeros(n, np.uint32)
    d = np.zeros(n, np.float32)
    check(lib.pqrr_dev_assign_batch(device, p, n, p.shape[1], c, c.shape[0], a, d))
    return a, d


def assign_u8(points, centroids, device: int = DEFAULT_DEVICE) -> np.ndarray:
    """The add path's assignment of u8 rows (ivf_index.hpp:54-56): equal to
    assign_batch's indices; d = 128, k % 128 == 0 run on the tensor cores
    (certified, pqrr_dev_assign_u8)."""
    p = np.ascontiguousarray(points, np.uint8)
    c = _f32(_vectorset(centroids, p.shape[1]))
    a = np.zeros(p.shape[0], np.uint32)
    check(lib.pqrr_dev_assign_u8(device, p, p.shape[0], p.shape[1], c, c.shape[0], a))
    return a


def encode_batch(pq: ProductQuantizer, data, device: int = DEFAULT_DEVICE) -> np.ndarray:
    """kernels.hpp:28-29."""
    x = _f32(_vectorset(data, pq.d))
    out = np.zeros((x.shape[0], pq.m), np.uint8)
    check(lib.pqrr_dev_encode_batch(device, pq.flat(), pq.d, pq.m, pq.ks, x, x.shape[0], out))
    return out


def decode_batch(pq: ProductQuantizer, codes, device: int = DEFAULT_DEVICE) -> np.ndarray:
    """kernels.hpp:32-33."""
    c = np.ascontiguousarray(np.asarray(codes, np.uint8).reshape(-1, pq.m))
    out = np.zeros((c.shape[0], pq.d), np.float32)
    check(lib.pqrr_dev_decode_batch(device, pq.flat(), pq.d, pq.m, pq.ks, c, c.shape[0], out))
    return out


def scan_topk(lut: LookupTable, codes, kprime: int, id_base: int = 0,
              device: int = DEFAULT_DEVICE) -> SearchResult:
    """kernels.hpp:40-41: kprime smallest (dist, id), ids = id_base + position."""
    t = _f32(lut.values)
    c = np.ascontiguousarray(np.asarray(codes, np.uint8).reshape(-1, t.shape[0]))
    ids = np.zeros(max(kprime, 1), np.uint32)
    dists = np.zeros(max(kprime, 1), np.float32)
    cnt = C.c_size_t(0)
    check(lib.pqrr_dev_scan_topk(device, t, t.shape[0], t.shape[1], c, c.shape[0], kprime, id_base,
                                 ids, dists, C.byref(cnt)))
    return SearchResult(ids[:cnt.value].copy(), dists[:cnt.value].copy())
