"""The "PQRR" binary container (storage.hpp:14-62) for quantizers, codebooks and
device-resident ADC / IVF indexes.  The reader/writer is host C++ inside
libpqrr_b200.so (csrc/storage.cu); this module mirrors the reference API.
Layouts: DESIGN.md §10.  Errors: "corrupt file" (ValueError) on any size or
header mismatch, OSError-like PqrrError when the file cannot be opened."""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from ._lib import check, lib
from .adc import AdcIndex
from .ivf import (DEFAULT_DEVICE, Codebook, IvfIndex, ProductQuantizer, RefineCodes,
                  RefineQuantizer, _f32)


class IndexKind(enum.Enum):
    adc = 0
    ivf = 1


def _p(path) -> bytes:
    return os.fsencode(os.fspath(path))


def save_quantizer(pq: ProductQuantizer, path) -> None:
    """storage.hpp:33."""
    check(lib.pqrr_dev_save_quantizer(_p(path), pq.d, pq.m, pq.ks, pq.flat()))


def _load_block(path):
    d, m, ks = _lib._u32(), _lib._u32(), _lib._u32()
    check(lib.pqrr_dev_load_quantizer(_p(path), C.byref(d), C.byref(m), C.byref(ks), None))
    books = np.zeros(ks.value * d.value, np.float32)
    check(lib.pqrr_dev_load_quantizer(_p(path), C.byref(d), C.byref(m), C.byref(ks),
                                      books.ctypes.data))
    return d.value, m.value, ks.value, books


def load_quantizer(path) -> ProductQuantizer:
    """storage.hpp:34."""
    d, m, ks, books = _load_block(path)
    return ProductQuantizer(d, m, ks, books.reshape(m, ks, d // m))


def save_codebook(book: Codebook, path) -> None:
    """storage.hpp:36 (the quantizer layout with m = 1, storage.hpp:28-29)."""
    c = _f32(book.centroids)
    check(lib.pqrr_dev_save_quantizer(_p(path), c.shape[1], 1, c.shape[0], c.reshape(-1)))


def load_codebook(path) -> Codebook:
    """storage.hpp:37."""
    d, m, ks, books = _load_block(path)
    if m != 1:
        raise ValueError("corrupt file")  # a product quantizer, not a plain codebook
    return Codebook(books.reshape(ks, d))


def _check_refine(index, rq, codes):
    if (rq is None) != (codes is None):
        raise ValueError("refine quantizer and codes go together")
    if rq is None and index.rq is not None:
        raise ValueError("the device index carries refinement codes: pass rq and codes")
    if rq is not None and (index.rq is None or index.refine_codes is not codes):
        raise ValueError("refinement codes are not attached to this index")


def save_adc_index(index: AdcIndex, rq: Optional[RefineQuantizer], codes: Optional[RefineCodes],
                   path) -> None:
    """storage.hpp:39-40."""
    _check_refine(index, rq, codes)
    check(lib.pqrr_dev_save_adc_index(index.h, _p(path)))


def save_ivf_index(index: IvfIndex, rq: Optional[RefineQuantizer], codes: Optional[RefineCodes],
                   path) -> None:
    """storage.hpp:49-50."""
    _check_refine(index, rq, codes)
    check(lib.pqrr_dev_save_index(index.h, _p(path)))


@dataclass
class LoadedAdcIndex:
    """storage.hpp:42-46."""
    index: AdcIndex
    refine_quantizer: Optional[RefineQuantizer]
    refine_codes: Optional[RefineCodes]


@dataclass
class LoadedIvfIndex:
    """storage.hpp:52-56."""
    index: IvfIndex
    refine_quantizer: Optional[RefineQuantizer]
    refine_codes: Optional[RefineCodes]


def _codebooks(h, info):
    d, c, m, mp, ks = info["d"], info["c"], info["m"], info["mprime"], info["ks"]
    coarse = np.zeros((c, d), np.float32)
    books = np.zeros(ks * d, np.float32)
    rbooks = np.zeros(ks * d, np.float32) if mp else None
    check(lib.pqrr_dev_export_codebooks(h, coarse.ctypes.data, books.ctypes.data,
                                        rbooks.ctypes.data if mp else None))
    P = ProductQuantizer(d, m, ks, books.reshape(m, ks, d // m))
    R = RefineQuantizer(ProductQuantizer(d, mp, ks, rbooks.reshape(mp, ks, d // mp))) if mp else None
    return coarse, P, R


def _info(h) -> dict:
    inf = _lib.IndexInfo()
    check(lib.pqrr_dev_index_get_info(h, C.byref(inf)))
    return {k: getattr(inf, k) for k, _ in inf._fields_}


def load_adc_index(path, device: int = DEFAULT_DEVICE) -> LoadedAdcIndex:
    """storage.hpp:47."""
    h = C.c_void_p()
    check(lib.pqrr_dev_load_adc_index(device, _p(path), C.byref(h)))
    _, P, R = _codebooks(h, _info(h))
    ix = AdcIndex.__new__(AdcIndex)
    ix.pq, ix.rq, ix.device, ix.h, ix._rb, ix.refine_codes = P, R, device, h, None, None
    if R is not None:
        from .adc import _refine_codes_by_id

        ix.refine_codes = _refine_codes_by_id(ix)
    return LoadedAdcIndex(ix, R, ix.refine_codes)


def load_ivf_index(path, device: int = DEFAULT_DEVICE) -> LoadedIvfIndex:
    """storage.hpp:57."""
    h = C.c_void_p()
    check(lib.pqrr_dev_load_index(device, _p(path), C.byref(h)))
    coarse, P, R = _codebooks(h, _info(h))
    ix = IvfIndex.__new__(IvfIndex)
    ix.coarse, ix.pq, ix.rq, ix.device, ix.h, ix._rb = Codebook(coarse), P, R, device, h, None
    ix.refine_codes = None
    if R is not None:
        offs, ids, _, rc = ix.export_lists()
        order = np.argsort(ids, kind="stable")
        ix.refine_codes = RefineCodes(R.pq.m, np.ascontiguousarray(rc[order]))
    return LoadedIvfIndex(ix, R, ix.refine_codes)


def probe_index_kind(path) -> IndexKind:
    """storage.hpp:59-62: the layout whose section sizes fit the file exactly."""
    k = C.c_int()
    check(lib.pqrr_dev_probe_index_kind(_p(path), C.byref(k)))
    return IndexKind(k.value)
