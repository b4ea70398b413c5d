"""Host-side mirror of the reference's pqrr C++ API for the IVFADC+R path.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/pqrr/): ``ivf_train`` / ``ivf_build`` /
``ivf_search`` / ``ivf_search_batch`` / ``ivf_refine_train`` /
``ivf_refine_encode`` / ``ivf_reconstruct`` / ``ivf_rerank``
(ivf_index.hpp:48-81), ``kmeans_train`` (kmeans.hpp:38), ``pq_train`` /
``pq_encode`` / ``pq_decode`` / ``build_lut`` / ``adc_distance``
(product_quantizer.hpp:39-59).  A ``VectorSet`` is a C-contiguous float32
(n, d) numpy array; u8 arrays are accepted wherever the reference would read
bvecs (widened exactly, dataset_io.hpp:29-31).  Every call runs on the GPU
through libpqrr_b200.so; errors raise ValueError with the reference's messages.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, lib

DEFAULT_DEVICE = 0


# ----------------------------------------------------------------------- types
@dataclass
class TrainParams:
    """kmeans.hpp:21-28."""
    iterations: int = 25
    seed: int = 0
    redo: int = 1
    trace: Optional[list] = None


@dataclass
class Codebook:
    """kmeans.hpp:11-19: k centroids of dimensionality dim."""
    centroids: np.ndarray  # (k, dim) float32
    final_mse: float = 0.0

    @property
    def k(self) -> int:
        return self.centroids.shape[0]

    @property
    def dim(self) -> int:
        return self.centroids.shape[1]

    def centroid(self, i: int) -> np.ndarray:
        return self.centroids[i]


@dataclass
class ProductQuantizer:
    """product_quantizer.hpp:15-24; books is (m, ks, d/m) float32."""
    d: int
    m: int
    ks: int
    books: np.ndarray

    def dsub(self) -> int:
        return self.d // self.m

    def code_size(self) -> int:
        return self.m

    def bits_per_sub(self) -> int:
        return int(np.ceil(np.log2(self.ks))) if self.ks > 1 else 0

    def flat(self) -> np.ndarray:
        return np.ascontiguousarray(self.books.reshape(-1), np.float32)


@dataclass
class LookupTable:
    """product_quantizer.hpp:28-35: (m, ks) squared distances."""
    values: np.ndarray

    @property
    def m(self):
        return self.values.shape[0]

    @property
    def ks(self):
        return self.values.shape[1]

    def at(self, j, i):
        return float(self.values[j, i])


@dataclass
class RefineQuantizer:
    """refine.hpp:15-19."""
    pq: ProductQuantizer

    def mprime(self) -> int:
        return self.pq.m


@dataclass
class RefineCodes:
    """refine.hpp:22-28: n id-aligned codes of m' bytes."""
    m: int
    bytes: np.ndarray  # (n, m') uint8

    def n(self) -> int:
        return self.bytes.shape[0]

    def code(self, i: int) -> np.ndarray:
        return self.bytes[i]


@dataclass
class SearchResult:
    """types.hpp:53-59: ascending (dist, id)."""
    ids: np.ndarray
    dists: np.ndarray

    def size(self) -> int:
        return len(self.ids)

    def __len__(self):
        return len(self.ids)

    def empty(self) -> bool:
        return len(self.ids) == 0


@dataclass
class IvfSearchParams:
    """ivf_index.hpp:43-46."""
    v: int = 8
    kprime: int = 100


def _f32(x) -> np.ndarray:
    x = np.asarray(x)
    if x.dtype != np.float32:
        x = x.astype(np.float32)
    return np.ascontiguousarray(x)


def _vectorset(x, d=None) -> np.ndarray:
    x = np.asarray(x)
    if x.ndim == 1:
        x = x.reshape(1, -1)
    if d is not None and x.shape[1] != d:
        raise ValueError("dimension mismatch")
    return x


# ----------------------------------------------------------------------- training
def kmeans_train(points, k: int, params: TrainParams = TrainParams(), device: int = DEFAULT_DEVICE) -> Codebook:
    """kmeans.hpp:38 (exact device assignment, id-order fp64 update)."""
    p = _f32(_vectorset(points))
    n, d = p.shape
    cent = np.zeros((max(k, 1), d), np.float32)
    mse = C.c_double(0)
    trace = np.zeros(max(params.iterations, 1), np.float64)
    check(lib.pqrr_dev_kmeans_train(device, p, n, d, k, params.iterations, params.seed, params.redo,
                                    cent, C.byref(mse), trace.ctypes.data))
    if params.trace is not None:
        params.trace[:] = list(trace[: params.iterations])
    return Codebook(cent, mse.value)


def pq_train(training, m: int, ks: int = 256, params: TrainParams = TrainParams(),
             device: int = DEFAULT_DEVICE) -> ProductQuantizer:
    """product_quantizer.hpp:39-40: sub-book j seeded seed + j."""
    t = _f32(_vectorset(training))
    n, d = t.shape
    if m == 0 or d % m:
        raise ValueError("dimension not divisible")
    books = np.zeros(m * ks * (d // m), np.float32)
    check(lib.pqrr_dev_pq_train(device, t, n, d, m, ks, params.iterations, params.seed, params.redo,
                                books))
    return ProductQuantizer(d, m, ks, books.reshape(m, ks, d // m))


def ivf_train(training, c: int, m: int, ks: int = 256, params: TrainParams = TrainParams(),
              device: int = DEFAULT_DEVICE):
    """ivf_index.hpp:50-52 -> (Codebook, ProductQuantizer)."""
    t = _f32(_vectorset(training))
    n, d = t.shape
    if m == 0 or d % m:
        raise ValueError("dimension not divisible")
    coarse = np.zeros((c, d), np.float32)
    books = np.zeros(m * ks * (d // m), np.float32)
    check(lib.pqrr_dev_ivf_train(device, t, n, d, c, m, ks, params.iterations, params.seed, coarse,
                                 books))
    return Codebook(coarse), ProductQuantizer(d, m, ks, books.reshape(m, ks, d // m))


def ivf_refine_train(coarse: Codebook, pq: ProductQuantizer, training, mprime: int,
                     params: TrainParams = TrainParams(), device: int = DEFAULT_DEVICE) -> RefineQuantizer:
    """ivf_index.hpp:68-70: residuals against coarse + PQ decode."""
    t = _f32(_vectorset(training, pq.d))
    n, d = t.shape
    if mprime == 0 or d % mprime:
        raise ValueError("dimension not divisible")
    rb = np.zeros(mprime * pq.ks * (d // mprime), np.float32)
    check(lib.pqrr_dev_ivf_refine_train(device, _f32(coarse.centroids), coarse.k, pq.flat(), d,
                                        pq.m, pq.ks, t, n, mprime, params.iterations, params.seed,
                                        rb))
    return RefineQuantizer(ProductQuantizer(d, mprime, pq.ks, rb.reshape(mprime, pq.ks, d // mprime)))


# ----------------------------------------------------------------------- PQ codec
def pq_encode(pq: ProductQuantizer, y, device: int = DEFAULT_DEVICE) -> np.ndarray:
    """product_quantizer.hpp:42-43 (batched over rows)."""
    y = _f32(_vectorset(y))
    if y.shape[1] != pq.d:
        raise ValueError("length mismatch")
    out = np.zeros((y.shape[0], pq.m), np.uint8)
    check(lib.pqrr_dev_encode_batch(device, pq.flat(), pq.d, pq.m, pq.ks, y, y.shape[0], out))
    return out


def pq_decode(pq: ProductQuantizer, codes, device: int = DEFAULT_DEVICE) -> np.ndarray:
    """product_quantizer.hpp:45-46."""
    c = np.ascontiguousarray(np.asarray(codes, np.uint8).reshape(-1, pq.m))
    out = np.zeros((c.shape[0], pq.d), np.float32)
    check(lib.pqrr_dev_decode_batch(device, pq.flat(), pq.d, pq.m, pq.ks, c, c.shape[0], out))
    return out


def build_lut(pq: ProductQuantizer, x, device: int = DEFAULT_DEVICE) -> LookupTable:
    """product_quantizer.hpp:48-49."""
    x = _f32(_vectorset(x))
    if x.shape[1] != pq.d:
        raise ValueError("length mismatch")
    out = np.zeros((x.shape[0], pq.m, pq.ks), np.float32)
    check(lib.pqrr_dev_build_lut(device, pq.flat(), pq.d, pq.m, pq.ks, x, x.shape[0], out))
    if x.shape[0] == 1:
        return LookupTable(out[0])
    return [LookupTable(t) for t in out]


def adc_distance(lut: LookupTable, code) -> float:
    """product_quantizer.hpp:53-57: j-ascending float32 sum (host helper)."""
    acc = np.float32(0.0)
    for j, c in enumerate(np.asarray(code, np.uint8)):
        acc = np.float32(acc + lut.values[j, c])
    return float(acc)


# ----------------------------------------------------------------------- index
class IvfIndex:
    """ivf_index.hpp:27-41 resident in HBM (plus refinement when attached)."""

    def __init__(self, coarse: Codebook, pq: ProductQuantizer, rq: Optional[RefineQuantizer] = None,
                 device: int = DEFAULT_DEVICE):
        self.coarse = coarse
        self.pq = pq
        self.rq = rq
        self.device = device
        self.refine_codes: Optional[RefineCodes] = None
        h = C.c_void_p()
        rb = rq.pq.flat() if rq is not None else None
        mprime = rq.pq.m if rq is not None else 0
        check(lib.pqrr_dev_index_create(device, pq.d, coarse.k, _f32(coarse.centroids), pq.m,
                                        pq.flat(), mprime, rb.ctypes.data if rb is not None else None,
                                        pq.ks, C.byref(h)))
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

    # -- add path
    def add(self, base, id_base: int = 0) -> None:
        base = _vectorset(base, self.pq.d)
        if base.dtype == np.uint8:
            check(lib.pqrr_dev_add_u8(self.h, np.ascontiguousarray(base), base.shape[0], id_base))
        else:
            check(lib.pqrr_dev_add_f32(self.h, _f32(base), base.shape[0], id_base))

    def add_synthetic(self, seed: int, clusters: int, row0: int, n: int, id_base: int = 0) -> None:
        check(lib.pqrr_dev_add_synthetic(self.h, seed, clusters, row0, n, id_base))

    def finalize(self) -> None:
        check(lib.pqrr_dev_finalize(self.h))

    def info(self) -> dict:
        inf = _lib.IndexInfo()
        check(lib.pqrr_dev_index_get_info(self.h, C.byref(inf)))
        return {k: getattr(inf, k) for k, _ in inf._fields_}

    @property
    def n(self) -> int:
        return self.info()["n"]

    def c(self) -> int:
        return self.coarse.k

    def export_lists(self):
        """(offsets[c+1], ids[n], codes[n, m], rcodes[n, m'] or None) in list order."""
        inf = self.info()
        n, c = inf["n"], inf["c"]
        offs = np.zeros(c + 1, np.uint64)
        ids = np.zeros(n, np.uint32)
        codes = np.zeros((n, self.pq.m), np.uint8)
        rc = np.zeros((n, inf["mprime"]), np.uint8) if inf["mprime"] else None
        check(lib.pqrr_dev_export_lists(self.h, offs.ctypes.data, ids.ctypes.data, codes.ctypes.data,
                                        rc.ctypes.data if rc is not None else None))
        return offs, ids, codes, rc

    def export_lists_subset(self, lists):
        """(offsets[len(lists)+1], ids, codes, rcodes or None) of the given lists,
        each id-ascending (host copies of those lists only)."""
        lists = np.ascontiguousarray(lists, np.uint32)
        offs = np.zeros(len(lists) + 1, np.uint64)
        check(lib.pqrr_dev_export_lists_subset(self.h, lists, len(lists), offs, None, None, None))
        n = int(offs[-1])
        mp = self.info()["mprime"]
        ids = np.zeros(n, np.uint32)
        codes = np.zeros((n, self.pq.m), np.uint8)
        rc = np.zeros((n, mp), np.uint8) if mp else None
        check(lib.pqrr_dev_export_lists_subset(self.h, lists, len(lists), offs, ids.ctypes.data,
                                               codes.ctypes.data,
                                               rc.ctypes.data if rc is not None else None))
        return offs, ids, codes, rc

    def load_lists(self, offsets, ids, codes, rcodes=None) -> None:
        """Inverse of export_lists (an existing inverted file into an empty index)."""
        rc = None
        if rcodes is not None:
            rc = np.ascontiguousarray(rcodes, np.uint8)
        check(lib.pqrr_dev_load_lists(self.h, np.ascontiguousarray(offsets, np.uint64),
                                      np.ascontiguousarray(ids, np.uint32),
                                      np.ascontiguousarray(codes, np.uint8),
                                      rc.ctypes.data if rc is not None else None))

    @property
    def lists(self):
        offs, ids, codes, _ = self.export_lists()
        return [(ids[offs[l]:offs[l + 1]], codes[offs[l]:offs[l + 1]]) for l in range(len(offs) - 1)]

    def assignments(self):
        """list_of_id / pos_of_id (ivf_index.hpp:34-35) from the device layout."""
        offs, ids, _, _ = self.export_lists()
        n = len(ids)
        lo = np.zeros(int(ids.max()) + 1 if n else 0, np.uint32)
        po = np.zeros_like(lo)
        for l in range(len(offs) - 1):
            seg = ids[offs[l]:offs[l + 1]]
            lo[seg] = l
            po[seg] = np.arange(len(seg), dtype=np.uint32)
        return lo, po

    # -- search
    def search(self, queries, v: int, kprime: int, k: int = 0, out=None):
        """Batched fused search; returns (ids, dists, counts) arrays of width k or kprime.

        ``out`` (optional) = caller-owned (ids uint32 [nq, width], dists float32
        [nq, width], counts uint32 [nq]) C-contiguous arrays written in place —
        e.g. page-locked buffers reused across batches, so the device-to-host
        copy of the results runs at full PCIe / C2C bandwidth."""
        q = _vectorset(queries, self.pq.d)
        nq = q.shape[0]
        width = k if k else kprime
        if out is None:
            ids = np.zeros((nq, width), np.uint32)
            dists = np.zeros((nq, width), np.float32)
            counts = np.zeros(nq, np.uint32)
        else:
            ids, dists, counts = out
            for a, dt, shp in ((ids, np.uint32, (nq, width)), (dists, np.float32, (nq, width)),
                               (counts, np.uint32, (nq,))):
                if a.dtype != dt or a.shape != shp or not a.flags["C_CONTIGUOUS"]:
                    raise ValueError("out arrays: expected C-contiguous %s %s" % (np.dtype(dt), shp))
        if q.dtype == np.uint8:
            check(lib.pqrr_dev_search_u8(self.h, np.ascontiguousarray(q), nq, v, kprime, k, ids, dists,
                                         counts))
        else:
            check(lib.pqrr_dev_search_f32(self.h, _f32(q), nq, v, kprime, k, ids, dists, counts))
        return ids, dists, counts

    def search_device(self, d_queries_ptr: int, nq: int, v: int, kprime: int, k: int,
                      d_ids_ptr: int, d_dists_ptr: int, d_counts_ptr: int, stream_ptr: int = 0):
        check(lib.pqrr_dev_search_u8_device(self.h, d_queries_ptr, nq, v, kprime, k, d_ids_ptr,
                                            d_dists_ptr, d_counts_ptr, stream_ptr or None))

    def search_enqueue(self, d_queries_ptr: int, nq: int, v: int, kprime: int, k: int,
                       d_ids_ptr: int, d_dists_ptr: int, d_counts_ptr: int, stream_ptr: int = 0):
        """Small-batch search as one captured CUDA graph, launched without
        blocking the host (pqrr_dev_search_u8_enqueue); ``search_finish`` waits
        and raises what the blocking call would."""
        check(lib.pqrr_dev_search_u8_enqueue(self.h, d_queries_ptr, nq, v, kprime, k, d_ids_ptr,
                                             d_dists_ptr, d_counts_ptr, stream_ptr or None))

    def search_finish(self):
        check(lib.pqrr_dev_search_finish(self.h))

    def set_graph(self, enabled: bool):
        """False: every search takes the synchronising path (per-stage times in
        ``last_stats``); True (default): batches of <= 1024 queries replay graphs."""
        check(lib.pqrr_dev_index_set_graph(self.h, 1 if enabled else 0))

    def rerank_owned_device(self, d_queries_ptr: int, nq: int, d_sl_ids_ptr: int,
                            d_sl_counts_ptr: int, sl_stride: int, k: int, d_ids_ptr: int,
                            d_dists_ptr: int, d_counts_ptr: int, stream_ptr: int = 0):
        """Exact multi-shard mode: re-rank the ids of a global shortlist that this
        shard holds (device pointers; see pqrr_dev_rerank_owned_u8_device)."""
        check(lib.pqrr_dev_rerank_owned_u8_device(self.h, d_queries_ptr, nq, d_sl_ids_ptr,
                                                  d_sl_counts_ptr, sl_stride, k, d_ids_ptr,
                                                  d_dists_ptr, d_counts_ptr, stream_ptr or None))

    def lookup_ids(self, ids):
        """(list_of_id, codes [n, m], rcodes [n, m'] or None) of the given ids
        (code_of_id, ivf_index.hpp:33-40; RefineCodes::code, refine.hpp:27);
        list = 0xffffffff for ids never added."""
        ids = np.ascontiguousarray(ids, np.uint32)
        n = len(ids)
        mp = self.info()["mprime"]
        lst = np.zeros(n, np.uint32)
        codes = np.zeros((n, self.pq.m), np.uint8)
        rc = np.zeros((n, mp), np.uint8) if mp else None
        check(lib.pqrr_dev_lookup_ids(self.h, ids, n, lst.ctypes.data, codes.ctypes.data,
                                      rc.ctypes.data if rc is not None else None))
        return lst, codes, rc

    def last_stats(self) -> dict:
        st = _lib.SearchStats()
        check(lib.pqrr_dev_last_search_stats(self.h, C.byref(st)))
        return st.as_dict()


def ivf_build(coarse: Codebook, pq: ProductQuantizer, base, device: int = DEFAULT_DEVICE,
              rq: Optional[RefineQuantizer] = None) -> IvfIndex:
    """ivf_index.hpp:56: every base vector to its nearest list, coding y - C_a.

    ``rq`` (extension) encodes the refinement codes in the same pass, which is
    what ivf_refine_encode would produce (the fused device add path)."""
    ix = IvfIndex(coarse, pq, rq, device)
    base = _vectorset(base, pq.d)
    if base.shape[0]:
        ix.add(base, 0)
    ix.finalize()
    ix._base_n = base.shape[0]
    return ix


def ivf_refine_encode(index: IvfIndex, rq: RefineQuantizer, base) -> RefineCodes:
    """ivf_index.hpp:72-73: id-aligned codes of y - (C_a + p).

    The device index keeps refinement codes next to the first-stage codes, so
    this (re)builds the device index with ``rq`` attached and exports them."""
    base = _vectorset(base, index.pq.d)
    if base.shape[0] != index.n:
        raise ValueError("count mismatch")
    new = IvfIndex(index.coarse, index.pq, rq, index.device)
    if base.shape[0]:
        new.add(base, 0)
    new.finalize()
    index.close()
    index.h, index.rq, index._rb = new.h, rq, new._rb
    new.h = C.c_void_p()
    offs, ids, _, rc = index.export_lists()
    byid = np.zeros((len(ids), rq.pq.m), np.uint8)
    byid[ids] = rc
    codes = RefineCodes(rq.pq.m, byid)
    index.refine_codes = codes
    return codes


def ivf_search(index: IvfIndex, x, params: IvfSearchParams) -> SearchResult:
    """ivf_index.hpp:60-61."""
    ids, dists, cnt = index.search(_vectorset(x, index.pq.d), params.v, params.kprime, 0)
    return SearchResult(ids[0, :cnt[0]].copy(), dists[0, :cnt[0]].copy())


def ivf_search_batch(index: IvfIndex, queries, params: IvfSearchParams) -> List[SearchResult]:
    """ivf_index.hpp:63-64: element-wise identical to ivf_search, query order kept."""
    ids, dists, cnt = index.search(queries, params.v, params.kprime, 0)
    return [SearchResult(ids[q, :cnt[q]].copy(), dists[q, :cnt[q]].copy()) for q in range(len(cnt))]


def ivf_reconstruct(index: IvfIndex, rq: RefineQuantizer, id_: int, codes: RefineCodes) -> np.ndarray:
    """ivf_index.hpp:76-77: coarse centroid + decode + refinement decode."""
    if index.rq is None or index.refine_codes is not codes:
        raise ValueError("refinement codes are not attached to this index")
    out = np.zeros((1, index.pq.d), np.float32)
    check(lib.pqrr_dev_reconstruct(index.h, np.array([id_], np.uint32), 1, out))
    return out[0]


def ivf_rerank(x, shortlist, index: IvfIndex, rq: RefineQuantizer, codes: RefineCodes,
               k: int):
    """ivf_index.hpp:79-81; x may be one vector (shortlist: SearchResult) or a
    batch (shortlist: list of SearchResult).  Errors "shortlist too small"."""
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
        check(lib.pqrr_dev_rerank_u8(index.h, np.ascontiguousarray(q), nq, sl_ids, sl_cnt, stride, k,
                                     ids, dists))
    else:
        check(lib.pqrr_dev_rerank_f32(index.h, _f32(q), nq, sl_ids, sl_cnt, stride, k, ids, dists))
    res = [SearchResult(ids[i, :k].copy(), dists[i, :k].copy()) for i in range(nq)]
    return res[0] if single else res


def merge_topk(ids, dists, counts, k: int, device: int = DEFAULT_DEVICE):
    """K7 on the device: per-shard ranked lists [parts, nq, width] -> top-k (dist, id)."""
    ids = np.ascontiguousarray(ids, np.uint32)
    dists = np.ascontiguousarray(dists, np.float32)
    counts = np.ascontiguousarray(counts, np.uint32)
    parts, nq, width = ids.shape
    oi = np.zeros((nq, k), np.uint32)
    od = np.zeros((nq, k), np.float32)
    oc = np.zeros(nq, np.uint32)
    check(lib.pqrr_dev_merge_topk(device, ids, dists, counts, nq, parts, width, k, oi, od, oc))
    return oi, od, oc


# ----------------------------------------------------------------------- data
def synth(set_id: int, row0: int, n: int, clusters: int, seed: int = 0, d: int = 128,
          device: int = DEFAULT_DEVICE) -> np.ndarray:
    """Rows of the BASELINE.json SIFT-like generator (set 1 train, 2 base, 3 query)."""
    out = np.zeros((n, d), np.uint8)
    check(lib.pqrr_dev_synth(device, seed, clusters, d, set_id, row0, n, out))
    return out
