"""ctypes bindings for the CPU oracle (build/liboracle.so) and the
reference-backed library (_ref/libpqrr_ref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package
(paper_1102_3828_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libpqrr_ref.so")
REF_SRC = "/root/reference/proj"

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_sz = C.c_size_t
_u32 = C.c_uint32
_u64 = C.c_uint64


def build(ref: bool | None = None) -> None:
    """Compile the oracle (and, when the reference tree exists, oracle/_ref)."""
    targets = ["all"]
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        targets.append("ref")
    subprocess.check_call(["make", "-s", "-C", HERE] + targets)


class OracleError(RuntimeError):
    pass


def _sig(lib, name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


class Oracle:
    """Thin numpy wrapper over liboracle.so (the C++ restatement)."""

    def __init__(self, path: str = LIB_PATH):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        _sig(L, "orc_last_error", C.c_char_p, [])
        _sig(L, "orc_set_threads", C.c_int, [C.c_int])
        _sig(L, "orc_l2_sq", C.c_float, [_f32p, _f32p, _sz])
        _sig(L, "orc_l2_sq_d", C.c_double, [_f32p, _f32p, _sz])
        _sig(L, "orc_topk", _sz, [_u32p, _f32p, _sz, _sz, _u32p, _f32p])
        _sig(L, "orc_assign_batch", C.c_int, [_f32p, _sz, _u32, _f32p, _u32, _u32p, _f32p])
        _sig(L, "orc_encode_batch", C.c_int, [_f32p, _u32, _u32, _u32, _f32p, _sz, _u8p])
        _sig(L, "orc_decode_batch", C.c_int, [_f32p, _u32, _u32, _u32, _u8p, _sz, _f32p])
        _sig(L, "orc_build_lut", C.c_int, [_f32p, _u32, _u32, _u32, _f32p, _f32p])
        _sig(L, "orc_adc_distance", C.c_float, [_f32p, _u32, _u32, _u8p])
        _sig(L, "orc_scan_topk", _sz, [_f32p, _u32, _u32, _u8p, _sz, _sz, _u32, _u32p, _f32p])
        _sig(L, "orc_kmeans_train", C.c_int,
             [_f32p, _sz, _u32, _u32, _u32, _u64, _u32, _f32p, C.POINTER(C.c_double), C.c_void_p])
        _sig(L, "orc_pq_train", C.c_int, [_f32p, _sz, _u32, _u32, _u32, _u32, _u64, _u32, _f32p])
        _sig(L, "orc_ivf_train", C.c_int,
             [_f32p, _sz, _u32, _u32, _u32, _u32, _u32, _u64, _f32p, _f32p])
        _sig(L, "orc_ivf_refine_train", C.c_int,
             [_f32p, _u32, _f32p, _u32, _u32, _u32, _f32p, _sz, _u32, _u32, _u64, _f32p])
        _sig(L, "orc_ivf_build", C.c_void_p, [_f32p, _u32, _f32p, _u32, _u32, _u32, _f32p, _sz])
        _sig(L, "orc_ivf_free", None, [C.c_void_p])
        _sig(L, "orc_ivf_list_size", _sz, [C.c_void_p, _u32])
        _sig(L, "orc_ivf_list_get", C.c_int, [C.c_void_p, _u32, _u32p, _u8p])
        _sig(L, "orc_ivf_assignments", C.c_int, [C.c_void_p, _u32p, _u32p])
        _sig(L, "orc_ivf_refine_encode", C.c_int, [C.c_void_p, _f32p, _u32, _f32p, _sz, _u8p])
        _sig(L, "orc_ivf_search_batch", C.c_int,
             [C.c_void_p, _f32p, _sz, _u32, _sz, _u32p, _f32p, _u32p])
        _sig(L, "orc_ivf_reconstruct", C.c_int, [C.c_void_p, _u32, _f32p])
        _sig(L, "orc_ivf_rerank_batch", C.c_int,
             [C.c_void_p, _f32p, _sz, _u32p, _u32p, _sz, _sz, _u32p, _f32p])
        _sig(L, "orc_coarse_probe", C.c_int, [_f32p, _u32, _u32, _f32p, _sz, _u32, _u32p, _f32p])
        _sig(L, "orc_exact_nearest", C.c_int, [_f32p, _sz, _u32, _f32p, _sz, _u32p, _f64p])
        _sig(L, "orc_recall_at_r", C.c_double, [_u32p, _u32p, _sz, _sz, _u32p, _sz])
        _sig(L, "orc_splitmix_stream_state", _u64, [_u64, _u32, _u64])
        _sig(L, "orc_splitmix_next", _u64, [C.POINTER(_u64)])
        _sig(L, "orc_bounded_u32", None, [_u32, _u32, _sz, _u32p])
        _sig(L, "orc_uniform01", None, [_u32, _sz, _f32p])
        _sig(L, "orc_ln", C.c_double, [C.c_double])
        _sig(L, "orc_sincos_2pi", None, [C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double)])
        _sig(L, "orc_synth_centers", C.c_int, [_u64, _u32, _u32, _f64p])
        _sig(L, "orc_synth_rows", C.c_int, [_u64, _u32, _u64, _sz, _u32, _f64p, _u32, _u8p])
        _sig(L, "orc_adc_encode", C.c_int, [_f32p, _u32, _u32, _u32, _f32p, _sz, _u8p])
        _sig(L, "orc_adc_search_batch", C.c_int,
             [_f32p, _u32, _u32, _u32, _u8p, _sz, _f32p, _sz, _sz, _u32p, _f32p, _u32p])
        _sig(L, "orc_refine_train", C.c_int,
             [_f32p, _u32, _u32, _u32, _f32p, _sz, _u32, _u32, _u64, _f32p])
        _sig(L, "orc_adc_refine_encode", C.c_int,
             [_f32p, _u32, _u32, _f32p, _u32, _u32, _f32p, _sz, _u8p])
        _sig(L, "orc_adc_reconstruct", C.c_int,
             [_f32p, _u32, _u32, _f32p, _u32, _u32, _u8p, _u8p, _f32p])
        _sig(L, "orc_adc_rerank_batch", C.c_int,
             [_f32p, _u32, _u32, _f32p, _u32, _u32, _u8p, _u8p, _f32p, _sz, _u32p, _u32p, _sz,
              _sz, _u32p, _f32p])

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(self.lib.orc_last_error().decode())

    def set_threads(self, t: int) -> int:
        return self.lib.orc_set_threads(t)

    # ---- primitives
    def l2_sq(self, a, b) -> float:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return self.lib.orc_l2_sq(a, b, a.size)

    def l2_sq_d(self, a, b) -> float:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return self.lib.orc_l2_sq_d(a, b, a.size)

    def topk(self, ids, dists, k):
        ids = np.ascontiguousarray(ids, np.uint32)
        dists = np.ascontiguousarray(dists, np.float32)
        oi = np.zeros(k, np.uint32)
        od = np.zeros(k, np.float32)
        n = self.lib.orc_topk(ids, dists, ids.size, k, oi, od)
        return oi[:n], od[:n]

    def assign(self, points, centroids):
        points = np.ascontiguousarray(points, np.float32)
        centroids = np.ascontiguousarray(centroids, np.float32)
        n, d = points.shape
        a = np.zeros(n, np.uint32)
        dist = np.zeros(n, np.float32)
        self._chk(self.lib.orc_assign_batch(points, n, d, centroids, centroids.shape[0], a, dist))
        return a, dist

    def encode(self, books, data, m, ks=256):
        data = np.ascontiguousarray(data, np.float32)
        books = np.ascontiguousarray(books, np.float32)
        n, d = data.shape
        out = np.zeros((n, m), np.uint8)
        self._chk(self.lib.orc_encode_batch(books, d, m, ks, data, n, out))
        return out

    def decode(self, books, codes, d, ks=256):
        codes = np.ascontiguousarray(codes, np.uint8)
        books = np.ascontiguousarray(books, np.float32)
        n, m = codes.shape
        out = np.zeros((n, d), np.float32)
        self._chk(self.lib.orc_decode_batch(books, d, m, ks, codes, n, out))
        return out

    def build_lut(self, books, x, m, ks=256):
        x = np.ascontiguousarray(x, np.float32)
        books = np.ascontiguousarray(books, np.float32)
        out = np.zeros((m, ks), np.float32)
        self._chk(self.lib.orc_build_lut(books, x.size, m, ks, x, out))
        return out

    def adc_distance(self, lut, code):
        lut = np.ascontiguousarray(lut, np.float32)
        code = np.ascontiguousarray(code, np.uint8)
        return self.lib.orc_adc_distance(lut, lut.shape[0], lut.shape[1], code)

    def scan_topk(self, lut, codes, kprime, id_base=0):
        lut = np.ascontiguousarray(lut, np.float32)
        codes = np.ascontiguousarray(codes, np.uint8)
        oi = np.zeros(kprime, np.uint32)
        od = np.zeros(kprime, np.float32)
        n = self.lib.orc_scan_topk(lut, lut.shape[0], lut.shape[1], codes, codes.shape[0],
                                   kprime, id_base, oi, od)
        return oi[:n], od[:n]

    # ---- training
    def kmeans(self, points, k, iterations=25, seed=0, redo=1):
        points = np.ascontiguousarray(points, np.float32)
        n, d = points.shape
        cent = np.zeros((k, d), np.float32)
        mse = C.c_double()
        trace = np.zeros(max(iterations, 1), np.float64)
        self._chk(self.lib.orc_kmeans_train(points, n, d, k, iterations, seed, redo, cent,
                                            C.byref(mse), trace.ctypes.data))
        return cent, mse.value, trace[:iterations]

    def pq_train(self, training, m, ks=256, iterations=25, seed=0, redo=1):
        training = np.ascontiguousarray(training, np.float32)
        n, d = training.shape
        if m == 0 or d % m:
            raise OracleError("dimension not divisible")
        books = np.zeros(m * ks * (d // m), np.float32)
        self._chk(self.lib.orc_pq_train(training, n, d, m, ks, iterations, seed, redo, books))
        return books

    def ivf_train(self, training, c, m, ks=256, iterations=25, seed=0):
        training = np.ascontiguousarray(training, np.float32)
        n, d = training.shape
        coarse = np.zeros((c, d), np.float32)
        books = np.zeros(m * ks * (d // m), np.float32)
        self._chk(self.lib.orc_ivf_train(training, n, d, c, m, ks, iterations, seed, coarse, books))
        return coarse, books

    def ivf_refine_train(self, coarse, books, m, training, mprime, ks=256, iterations=25, seed=0):
        training = np.ascontiguousarray(training, np.float32)
        n, d = training.shape
        rbooks = np.zeros(mprime * ks * (d // mprime), np.float32)
        self._chk(self.lib.orc_ivf_refine_train(np.ascontiguousarray(coarse, np.float32),
                                                coarse.shape[0], np.ascontiguousarray(books),
                                                d, m, ks, training, n, mprime, iterations, seed,
                                                rbooks))
        return rbooks

    # ---- ADC / ADC+R (adc_index.hpp:13-31, refine.hpp:30-53)
    def adc_build(self, books, m, base, ks=256):
        base = np.ascontiguousarray(base, np.float32)
        n, d = base.shape
        out = np.zeros((n, m), np.uint8)
        self._chk(self.lib.orc_adc_encode(np.ascontiguousarray(books, np.float32).reshape(-1), d, m,
                                          ks, base, n, out))
        return out

    def adc_search(self, books, m, codes, queries, kprime, ks=256):
        queries = np.ascontiguousarray(queries, np.float32)
        codes = np.ascontiguousarray(codes, np.uint8)
        nq, d = queries.shape
        ids = np.zeros((nq, kprime), np.uint32)
        dists = np.zeros((nq, kprime), np.float32)
        counts = np.zeros(nq, np.uint32)
        self._chk(self.lib.orc_adc_search_batch(np.ascontiguousarray(books, np.float32).reshape(-1),
                                                d, m, ks, codes, codes.shape[0], queries, nq,
                                                kprime, ids, dists, counts))
        return ids, dists, counts

    def refine_train(self, books, m, training, mprime, ks=256, iterations=25, seed=0):
        training = np.ascontiguousarray(training, np.float32)
        n, d = training.shape
        out = np.zeros(mprime * ks * (d // mprime), np.float32)
        self._chk(self.lib.orc_refine_train(np.ascontiguousarray(books, np.float32).reshape(-1), d,
                                            m, ks, training, n, mprime, iterations, seed, out))
        return out

    def adc_refine_encode(self, books, m, rbooks, mprime, base, ks=256):
        base = np.ascontiguousarray(base, np.float32)
        n, d = base.shape
        out = np.zeros((n, mprime), np.uint8)
        self._chk(self.lib.orc_adc_refine_encode(
            np.ascontiguousarray(books, np.float32).reshape(-1), d, m,
            np.ascontiguousarray(rbooks, np.float32).reshape(-1), mprime, ks, base, n, out))
        return out

    def adc_reconstruct(self, books, m, rbooks, mprime, code, rcode, d=128, ks=256):
        out = np.zeros(d, np.float32)
        self._chk(self.lib.orc_adc_reconstruct(
            np.ascontiguousarray(books, np.float32).reshape(-1), d, m,
            np.ascontiguousarray(rbooks, np.float32).reshape(-1), mprime, ks,
            np.ascontiguousarray(code, np.uint8), np.ascontiguousarray(rcode, np.uint8), out))
        return out

    def adc_rerank(self, books, m, rbooks, mprime, codes, rcodes, queries, sl_ids, sl_counts, k,
                   ks=256):
        queries = np.ascontiguousarray(queries, np.float32)
        sl_ids = np.ascontiguousarray(sl_ids, np.uint32)
        nq, d = queries.shape
        ids = np.zeros((nq, k), np.uint32)
        dists = np.zeros((nq, k), np.float32)
        self._chk(self.lib.orc_adc_rerank_batch(
            np.ascontiguousarray(books, np.float32).reshape(-1), d, m,
            np.ascontiguousarray(rbooks, np.float32).reshape(-1), mprime, ks,
            np.ascontiguousarray(codes, np.uint8), np.ascontiguousarray(rcodes, np.uint8), queries,
            nq, sl_ids, np.ascontiguousarray(sl_counts, np.uint32), sl_ids.shape[1], k, ids, dists))
        return ids, dists

    def ivf_build(self, coarse, books, m, base, ks=256) -> "OracleIvf":
        return OracleIvf(self, coarse, books, m, base, ks)

    def coarse_probe(self, coarse, queries, v):
        queries = np.ascontiguousarray(queries, np.float32)
        coarse = np.ascontiguousarray(coarse, np.float32)
        nq, d = queries.shape
        lists = np.zeros((nq, v), np.uint32)
        dists = np.zeros((nq, v), np.float32)
        self._chk(self.lib.orc_coarse_probe(coarse, coarse.shape[0], d, queries, nq, v, lists,
                                            dists))
        return lists, dists

    # ---- eval
    def exact_nearest(self, base, queries):
        base = np.ascontiguousarray(base, np.float32)
        queries = np.ascontiguousarray(queries, np.float32)
        ids = np.zeros(queries.shape[0], np.uint32)
        d = np.zeros(queries.shape[0], np.float64)
        self._chk(self.lib.orc_exact_nearest(base, base.shape[0], base.shape[1], queries,
                                             queries.shape[0], ids, d))
        return ids, d

    def recall_at_r(self, ids, counts, gt, r):
        ids = np.ascontiguousarray(ids, np.uint32)
        return self.lib.orc_recall_at_r(ids, np.ascontiguousarray(counts, np.uint32),
                                        ids.shape[1], ids.shape[0],
                                        np.ascontiguousarray(gt, np.uint32), r)

    # ---- generator
    def synth_centers(self, seed, clusters, d=128):
        out = np.zeros((clusters, d), np.float64)
        self._chk(self.lib.orc_synth_centers(seed, clusters, d, out))
        return out

    def synth_rows(self, seed, set_id, row0, n, centers):
        clusters, d = centers.shape
        out = np.zeros((n, d), np.uint8)
        self._chk(self.lib.orc_synth_rows(seed, set_id, row0, n, d,
                                          np.ascontiguousarray(centers), clusters, out))
        return out

    def bounded_u32(self, seed, bound, n):
        out = np.zeros(n, np.uint32)
        self.lib.orc_bounded_u32(seed, bound, n, out)
        return out

    def uniform01(self, seed, n):
        out = np.zeros(n, np.float32)
        self.lib.orc_uniform01(seed, n, out)
        return out

    def splitmix_raw(self, state, n):
        st = _u64(state)
        return np.array([self.lib.orc_splitmix_next(C.byref(st)) for _ in range(n)], np.uint64)

    def ln(self, u):
        return self.lib.orc_ln(u)

    def sincos_2pi(self, u):
        s, c = C.c_double(), C.c_double()
        self.lib.orc_sincos_2pi(u, C.byref(s), C.byref(c))
        return s.value, c.value

    def stream(self, seed, set_id, row, n):
        st = _u64(self.lib.orc_splitmix_stream_state(seed, set_id, row))
        return np.array([self.lib.orc_splitmix_next(C.byref(st)) for _ in range(n)], np.uint64)


class OracleIvf:
    """Oracle IvfIndex handle (ivf_index.hpp:27-41) with refinement attached."""

    def __init__(self, orc: Oracle, coarse, books, m, base, ks=256):
        self.o = orc
        self.coarse = np.ascontiguousarray(coarse, np.float32)
        self.books = np.ascontiguousarray(books, np.float32)
        base = np.ascontiguousarray(base, np.float32)
        self.n, self.d = base.shape
        self.c = self.coarse.shape[0]
        self.m = m
        self.ks = ks
        self.mprime = 0
        self.h = orc.lib.orc_ivf_build(self.coarse, self.c, self.books, self.d, m, ks, base, self.n)
        if not self.h:
            raise OracleError(orc.lib.orc_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.orc_ivf_free(self.h)
            self.h = None

    def list_sizes(self):
        return np.array([self.o.lib.orc_ivf_list_size(self.h, l) for l in range(self.c)], np.uint64)

    def list(self, l):
        n = self.o.lib.orc_ivf_list_size(self.h, l)
        ids = np.zeros(n, np.uint32)
        codes = np.zeros((n, self.m), np.uint8)
        self.o._chk(self.o.lib.orc_ivf_list_get(self.h, l, ids, codes))
        return ids, codes

    def flat(self):
        """Lists flattened in list order: offsets[c+1], ids[n], codes[n, m]."""
        sizes = self.list_sizes()
        offs = np.zeros(self.c + 1, np.uint64)
        offs[1:] = np.cumsum(sizes)
        ids = np.zeros(self.n, np.uint32)
        codes = np.zeros((self.n, self.m), np.uint8)
        for l in range(self.c):
            i, c = self.list(l)
            ids[offs[l]:offs[l + 1]] = i
            codes[offs[l]:offs[l + 1]] = c
        return offs, ids, codes

    def assignments(self):
        lo = np.zeros(self.n, np.uint32)
        po = np.zeros(self.n, np.uint32)
        self.o._chk(self.o.lib.orc_ivf_assignments(self.h, lo, po))
        return lo, po

    def refine_encode(self, rbooks, mprime, base):
        base = np.ascontiguousarray(base, np.float32)
        self.rbooks = np.ascontiguousarray(rbooks, np.float32)
        self.mprime = mprime
        out = np.zeros((self.n, mprime), np.uint8)
        self.o._chk(self.o.lib.orc_ivf_refine_encode(self.h, self.rbooks, mprime, base, self.n, out))
        self.rcodes = out
        return out

    def search(self, queries, v, kprime):
        queries = np.ascontiguousarray(queries, np.float32)
        nq = queries.shape[0]
        ids = np.zeros((nq, kprime), np.uint32)
        dists = np.zeros((nq, kprime), np.float32)
        counts = np.zeros(nq, np.uint32)
        self.o._chk(self.o.lib.orc_ivf_search_batch(self.h, queries, nq, v, kprime, ids, dists,
                                                    counts))
        return ids, dists, counts

    def reconstruct(self, i):
        out = np.zeros(self.d, np.float32)
        self.o._chk(self.o.lib.orc_ivf_reconstruct(self.h, i, out))
        return out

    def rerank(self, queries, sl_ids, sl_counts, k):
        queries = np.ascontiguousarray(queries, np.float32)
        sl_ids = np.ascontiguousarray(sl_ids, np.uint32)
        nq = queries.shape[0]
        ids = np.zeros((nq, k), np.uint32)
        dists = np.zeros((nq, k), np.float32)
        self.o._chk(self.o.lib.orc_ivf_rerank_batch(self.h, queries, nq, sl_ids,
                                                    np.ascontiguousarray(sl_counts, np.uint32),
                                                    sl_ids.shape[1], k, ids, dists))
        return ids, dists


class RefLib:
    """The reference's own kernels.cpp + header code (oracle/_ref/libpqrr_ref.so)."""

    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        _sig(L, "ref_set_threads", None, [C.c_int])
        _sig(L, "ref_max_threads", C.c_int, [])
        _sig(L, "ref_l2_sq", C.c_float, [_f32p, _f32p, _sz])
        _sig(L, "ref_l2_sq_d", C.c_double, [_f32p, _f32p, _sz])
        _sig(L, "ref_assign_batch", None, [_f32p, _sz, _u32, _f32p, _u32, _u32p, _f32p])
        _sig(L, "ref_encode_batch", None, [_f32p, _u32, _u32, _u32, _f32p, _sz, _u8p])
        _sig(L, "ref_decode_batch", None, [_f32p, _u32, _u32, _u32, _u8p, _sz, _f32p])
        _sig(L, "ref_build_lut", None, [_f32p, _u32, _u32, _u32, _f32p, _f32p])
        _sig(L, "ref_adc_distance", C.c_float, [_f32p, _u32, _u32, _u8p])
        _sig(L, "ref_scan_topk", _sz, [_f32p, _u32, _u32, _u8p, _sz, _sz, _u32, _u32p, _f32p])
        _sig(L, "ref_topk", _sz, [_u32p, _f32p, _sz, _sz, _u32p, _f32p])
        _sig(L, "ref_splitmix", None, [_u64, _sz, _u64p])
        _sig(L, "ref_bounded_u32", None, [_u32, _u32, _sz, _u32p])
        _sig(L, "ref_uniform01", None, [_u32, _sz, _f32p])
        _sig(L, "ref_ivf_search_batch", None,
             [_f32p, _u32, _f32p, _u32, _u32, _u32, _u64p, _u32p, _u8p, _f32p, _sz, _u32, _sz,
              _u32p, _f32p, _u32p])
        _sig(L, "ref_ivf_rerank_batch", C.c_int,
             [_f32p, _f32p, _f32p, _u32, _u32, _u32, _u32, _u32p, _u8p, _u8p, _f32p, _sz, _u32p,
              _u32p, _sz, _sz, _u32p, _f32p])

    def set_threads(self, t):
        self.lib.ref_set_threads(t)

    def l2_sq(self, a, b):
        a = np.ascontiguousarray(a, np.float32)
        return self.lib.ref_l2_sq(a, np.ascontiguousarray(b, np.float32), a.size)

    def assign(self, points, centroids):
        points = np.ascontiguousarray(points, np.float32)
        centroids = np.ascontiguousarray(centroids, np.float32)
        n, d = points.shape
        a = np.zeros(n, np.uint32)
        dist = np.zeros(n, np.float32)
        self.lib.ref_assign_batch(points, n, d, centroids, centroids.shape[0], a, dist)
        return a, dist

    def encode(self, books, data, m, ks=256):
        data = np.ascontiguousarray(data, np.float32)
        n, d = data.shape
        out = np.zeros((n, m), np.uint8)
        self.lib.ref_encode_batch(np.ascontiguousarray(books, np.float32), d, m, ks, data, n, out)
        return out

    def decode(self, books, codes, d, ks=256):
        codes = np.ascontiguousarray(codes, np.uint8)
        n, m = codes.shape
        out = np.zeros((n, d), np.float32)
        self.lib.ref_decode_batch(np.ascontiguousarray(books, np.float32), d, m, ks, codes, n, out)
        return out

    def build_lut(self, books, x, m, ks=256):
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros((m, ks), np.float32)
        self.lib.ref_build_lut(np.ascontiguousarray(books, np.float32), x.size, m, ks, x, out)
        return out

    def scan_topk(self, lut, codes, kprime, id_base=0):
        lut = np.ascontiguousarray(lut, np.float32)
        codes = np.ascontiguousarray(codes, np.uint8)
        oi = np.zeros(kprime, np.uint32)
        od = np.zeros(kprime, np.float32)
        n = self.lib.ref_scan_topk(lut, lut.shape[0], lut.shape[1], codes, codes.shape[0],
                                   kprime, id_base, oi, od)
        return oi[:n], od[:n]

    def topk(self, ids, dists, k):
        ids = np.ascontiguousarray(ids, np.uint32)
        oi = np.zeros(k, np.uint32)
        od = np.zeros(k, np.float32)
        n = self.lib.ref_topk(ids, np.ascontiguousarray(dists, np.float32), ids.size, k, oi, od)
        return oi[:n], od[:n]

    def splitmix(self, seed, n):
        out = np.zeros(n, np.uint64)
        self.lib.ref_splitmix(seed, n, out)
        return out

    def bounded_u32(self, seed, bound, n):
        out = np.zeros(n, np.uint32)
        self.lib.ref_bounded_u32(seed, bound, n, out)
        return out

    def uniform01(self, seed, n):
        out = np.zeros(n, np.float32)
        self.lib.ref_uniform01(seed, n, out)
        return out

    def ivf_search(self, coarse, books, m, offsets, ids, codes, queries, v, kprime, ks=256):
        queries = np.ascontiguousarray(queries, np.float32)
        coarse = np.ascontiguousarray(coarse, np.float32)
        nq, d = queries.shape
        oi = np.zeros((nq, kprime), np.uint32)
        od = np.zeros((nq, kprime), np.float32)
        cnt = np.zeros(nq, np.uint32)
        self.lib.ref_ivf_search_batch(coarse, coarse.shape[0], np.ascontiguousarray(books), d, m,
                                      ks, np.ascontiguousarray(offsets, np.uint64),
                                      np.ascontiguousarray(ids, np.uint32),
                                      np.ascontiguousarray(codes, np.uint8), queries, nq, v,
                                      kprime, oi, od, cnt)
        return oi, od, cnt

    def ivf_rerank(self, coarse, books, rbooks, m, mprime, list_of_id, codes_by_id, rcodes_by_id,
                   queries, sl_ids, sl_counts, k, ks=256):
        queries = np.ascontiguousarray(queries, np.float32)
        sl_ids = np.ascontiguousarray(sl_ids, np.uint32)
        nq, d = queries.shape
        oi = np.zeros((nq, k), np.uint32)
        od = np.zeros((nq, k), np.float32)
        rc = self.lib.ref_ivf_rerank_batch(
            np.ascontiguousarray(coarse, np.float32), np.ascontiguousarray(books, np.float32),
            np.ascontiguousarray(rbooks, np.float32), d, m, mprime, ks,
            np.ascontiguousarray(list_of_id, np.uint32), np.ascontiguousarray(codes_by_id, np.uint8),
            np.ascontiguousarray(rcodes_by_id, np.uint8), queries, nq, sl_ids,
            np.ascontiguousarray(sl_counts, np.uint32), sl_ids.shape[1], k, oi, od)
        if rc != 0:
            raise OracleError("shortlist too small")
        return oi, od


def ref_available() -> bool:
    return os.path.exists(REF_PATH)
