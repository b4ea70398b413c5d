"""Exhaustive ADC and ADC+R (adc_index.hpp:13-31, refine.hpp:13-53) on the device.

The paper's first system (§3.2): every database vector is PQ-encoded as is
(no coarse quantizer), a query builds ONE lookup table and scans all n codes,
and ADC+R re-ranks the k' shortlist with the residual quantizer.  The device
index is the IVF machinery with a single all-zero coarse centroid
(pqrr_dev_adc_index_create): y - 0 = y and x - 0 = x exactly in fp32 and
(0 + p) + q_r = p + q_r, so codes, LUTs, ADC sums and re-rank distances are
the ADC / ADC+R ones bit for bit (tests/test_gpu_parity.py::test_adc_*).
The scan runs through the same list-major K4f/K4r kernels (the single list is
split into 16k-entry work items).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import check, lib
from .ivf import (DEFAULT_DEVICE, ProductQuantizer, RefineCodes, RefineQuantizer, SearchResult,
                  TrainParams, _f32, _vectorset)


class AdcIndex:
    """adc_index.hpp:13-19: n m-byte codes in id order, resident in HBM."""

    def __init__(self, pq: ProductQuantizer, rq: Optional[RefineQuantizer] = None,
                 device: int = DEFAULT_DEVICE):
        self.pq, self.rq, self.device = pq, rq, device
        self.refine_codes: Optional[RefineCodes] = None
        h = C.c_void_p()
        rb = rq.pq.flat() if rq is not None else None
        check(lib.pqrr_dev_adc_index_create(device, pq.d, pq.m, pq.flat(),
                                            rq.pq.m if rq is not None else 0,
                                            rb.ctypes.data if rb is not None else None, pq.ks,
                                            C.byref(h)))
        self._rb = rb
        self.h = h

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            lib.pqrr_dev_index_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _add(self, base) -> None:
        if base.shape[0]:
            if base.dtype == np.uint8:
                check(lib.pqrr_dev_add_u8(self.h, np.ascontiguousarray(base), base.shape[0], 0))
            else:
                check(lib.pqrr_dev_add_f32(self.h, _f32(base), base.shape[0], 0))
        check(lib.pqrr_dev_finalize(self.h))

    @property
    def n(self) -> int:
        inf = _lib.IndexInfo()
        check(lib.pqrr_dev_index_get_info(self.h, C.byref(inf)))
        return inf.n

    def _export(self):
        n = self.n
        offs = np.zeros(2, np.uint64)
        ids = np.zeros(n, np.uint32)
        codes = np.zeros((n, self.pq.m), np.uint8)
        mp = self.rq.pq.m if self.rq is not None else 0
        rc = np.zeros((n, mp), np.uint8) if mp else None
        check(lib.pqrr_dev_export_lists(self.h, offs.ctypes.data, ids.ctypes.data,
                                        codes.ctypes.data, rc.ctypes.data if rc is not None else None))
        return ids, codes, rc

    @property
    def codes(self) -> np.ndarray:
        """n x m code bytes in id order (adc_index.hpp:17)."""
        ids, codes, _ = self._export()
        out = np.zeros_like(codes)
        out[ids] = codes
        return out

    def code(self, i: int) -> np.ndarray:
        return self.codes[i]

    def search(self, queries, kprime: int, k: int = 0, out=None):
        """Batched device search: (ids, dists, counts) of width k or kprime.
        k = 0 -> the ADC shortlist; k > 0 -> fused ADC+R re-rank."""
        q = _vectorset(queries, self.pq.d)
        nq = q.shape[0]
        width = k if k else kprime
        if out is None:
            ids = np.zeros((nq, width), np.uint32)
            dists = np.zeros((nq, width), np.float32)
            counts = np.zeros(nq, np.uint32)
        else:
            ids, dists, counts = out
        if q.dtype == np.uint8:
            check(lib.pqrr_dev_search_u8(self.h, np.ascontiguousarray(q), nq, 1, kprime, k, ids,
                                         dists, counts))
        else:
            check(lib.pqrr_dev_search_f32(self.h, _f32(q), nq, 1, kprime, k, ids, dists, counts))
        return ids, dists, counts

    def last_stats(self) -> dict:
        st = _lib.SearchStats()
        check(lib.pqrr_dev_last_search_stats(self.h, C.byref(st)))
        return st.as_dict()


def adc_build(pq: ProductQuantizer, base, device: int = DEFAULT_DEVICE,
              rq: Optional[RefineQuantizer] = None) -> AdcIndex:
    """adc_index.hpp:22: encodes the base set; ids are 0-based positions.
    ``rq`` (extension) also encodes the refinement codes in the same pass."""
    ix = AdcIndex(pq, rq, device)
    ix._add(_vectorset(base, pq.d))
    if rq is not None:
        ix.refine_codes = _refine_codes_by_id(ix)
    return ix


def adc_search(index: AdcIndex, x, kprime: int) -> SearchResult:
    """adc_index.hpp:24-26: min(kprime, n) smallest estimates under (dist, id)."""
    ids, dists, cnt = index.search(_vectorset(x, index.pq.d), kprime, 0)
    return SearchResult(ids[0, :cnt[0]].copy(), dists[0, :cnt[0]].copy())


def adc_search_batch(index: AdcIndex, queries, kprime: int) -> List[SearchResult]:
    """adc_index.hpp:28-31: element-wise identical to adc_search, order kept."""
    ids, dists, cnt = index.search(queries, kprime, 0)
    return [SearchResult(ids[q, :cnt[q]].copy(), dists[q, :cnt[q]].copy()) for q in range(len(cnt))]


def residual(y, pq_c: ProductQuantizer, device: int = DEFAULT_DEVICE) -> np.ndarray:
    """refine.hpp:30-31: y - decode(encode(y)) (rows of a batch, or one vector)."""
    yy = _f32(_vectorset(y, pq_c.d))
    out = np.zeros_like(yy)
    check(lib.pqrr_dev_residual(device, pq_c.flat(), pq_c.d, pq_c.m, pq_c.ks, yy, yy.shape[0], out))
    return out[0] if np.asarray(y).ndim == 1 else out


def refine_train(pq_c: ProductQuantizer, training, mprime: int, params: TrainParams = TrainParams(),
                 device: int = DEFAULT_DEVICE) -> RefineQuantizer:
    """refine.hpp:33-36: pq_train on the residual set, 8 bits per sub-quantizer."""
    t = _f32(_vectorset(training, pq_c.d))
    n, d = t.shape
    if mprime == 0 or d % mprime:
        raise ValueError("dimension not divisible")
    rb = np.zeros(mprime * pq_c.ks * (d // mprime), np.float32)
    check(lib.pqrr_dev_refine_train(device, pq_c.flat(), d, pq_c.m, pq_c.ks, t, n, mprime,
                                    params.iterations, params.seed, rb))
    return RefineQuantizer(ProductQuantizer(d, mprime, pq_c.ks, rb.reshape(mprime, pq_c.ks, d // mprime)))


def _refine_codes_by_id(index: AdcIndex) -> RefineCodes:
    ids, _, rc = index._export()
    byid = np.zeros((len(ids), index.rq.pq.m), np.uint8)
    byid[ids] = rc
    return RefineCodes(index.rq.pq.m, byid)


def refine_encode(index: AdcIndex, rq: RefineQuantizer, base) -> RefineCodes:
    """refine.hpp:38-40: id-aligned codes of y - decode(encode(y)).  The device
    keeps refinement codes beside the first-stage codes, so the index is
    re-encoded with ``rq`` attached and the codes exported."""
    base = _vectorset(base, index.pq.d)
    if base.shape[0] != index.n:
        raise ValueError("count mismatch")
    new = adc_build(index.pq, base, index.device, rq)
    index.close()
    index.h, index.rq, index._rb, index.refine_codes = new.h, rq, new._rb, new.refine_codes
    new.h = C.c_void_p()
    return index.refine_codes


def reconstruct(pq_c: ProductQuantizer, rq: RefineQuantizer, code_c, code_r,
                device: int = DEFAULT_DEVICE) -> np.ndarray:
    """refine.hpp:42-45: decode_c(code_c) + decode_r(code_r)."""
    cc = np.ascontiguousarray(np.asarray(code_c, np.uint8).reshape(-1, pq_c.m))
    cr = np.ascontiguousarray(np.asarray(code_r, np.uint8).reshape(-1, rq.pq.m))
    if cc.shape[0] != cr.shape[0]:
        raise ValueError("count mismatch")
    out = np.zeros((cc.shape[0], pq_c.d), np.float32)
    check(lib.pqrr_dev_reconstruct_codes(device, pq_c.flat(), pq_c.d, pq_c.m, rq.pq.flat(), rq.pq.m,
                                         pq_c.ks, cc, cr, cc.shape[0], out))
    return out[0] if np.asarray(code_c).ndim == 1 else out


def rerank(x, shortlist, index: AdcIndex, rq: RefineQuantizer, codes: RefineCodes, k: int):
    """refine.hpp:47-53: k best of the shortlist under l2_sq(x, reconstruct);
    one vector + SearchResult, or a batch + list.  "shortlist too small"."""
    if index.rq is None or index.refine_codes is not codes:
        raise ValueError("refinement codes are not attached to this index")
    single = isinstance(shortlist, SearchResult)
    sls = [shortlist] if single else list(shortlist)
    q = _vectorset(x, index.pq.d)
    nq = q.shape[0]
    if nq != len(sls):
        raise ValueError("query / shortlist count mismatch")
    stride = max(1, max((len(s) for s in sls), default=1))
    sl_ids = np.zeros((nq, stride), np.uint32)
    sl_cnt = np.zeros(nq, np.uint32)
    for i, s in enumerate(sls):
        sl_ids[i, :len(s)] = s.ids
        sl_cnt[i] = len(s)
    ids = np.zeros((nq, max(k, 1)), np.uint32)
    dists = np.zeros((nq, max(k, 1)), np.float32)
    if q.dtype == np.uint8:
        check(lib.pqrr_dev_rerank_u8(index.h, np.ascontiguousarray(q), nq, sl_ids, sl_cnt, stride,
                                     k, ids, dists))
    else:
        check(lib.pqrr_dev_rerank_f32(index.h, _f32(q), nq, sl_ids, sl_cnt, stride, k, ids, dists))
    res = [SearchResult(ids[i, :k].copy(), dists[i, :k].copy()) for i in range(nq)]
    return res[0] if single else res
