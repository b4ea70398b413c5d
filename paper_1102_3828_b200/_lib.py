"""ctypes binding of libpqrr_b200.so (include/pqrr_dev.h).

The library is built in-tree (paper_1102_3828_b200/lib/) by
``__graft_entry__.build()`` / ``make -C paper_1102_3828_b200/csrc``.  There is
no fallback: if the shared object is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# PQRR_LIB_PATH: an alternative build of the same library (A/B timing runs)
LIB_PATH = os.environ.get("PQRR_LIB_PATH") or os.path.join(HERE, "lib", "libpqrr_b200.so")

PQRR_OK = 0
PQRR_EINVAL = -1
PQRR_ECUDA = -2
PQRR_ENODEV = -3
PQRR_EUNSUPPORTED = -4
PQRR_ESHORTLIST = -5
PQRR_EINTERNAL = -6

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA library first "
        "(python -c 'import __graft_entry__ as g; g.build()')")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_sz = C.c_size_t
_u32 = C.c_uint32
_u64 = C.c_uint64
_vp = C.c_void_p
_int = C.c_int


class IndexInfo(C.Structure):
    _fields_ = [("n", C.c_uint64), ("slots", C.c_uint64), ("d", C.c_uint32), ("c", C.c_uint32),
                ("m", C.c_uint32), ("mprime", C.c_uint32), ("ks", C.c_uint32),
                ("max_list_len", C.c_uint32), ("device_bytes", C.c_uint64)]


class SearchStats(C.Structure):
    _fields_ = [("ms_total", C.c_float), ("ms_coarse", C.c_float), ("ms_invert", C.c_float),
                ("ms_sample_scan", C.c_float), ("ms_threshold", C.c_float),
                ("ms_scan", C.c_float), ("ms_select", C.c_float), ("ms_rerank", C.c_float),
                ("nq", C.c_uint64), ("scanned_entries", C.c_uint64),
                ("sampled_entries", C.c_uint64), ("candidates", C.c_uint64),
                ("work_items", C.c_uint32), ("retries", C.c_uint32), ("stride", C.c_uint32),
                ("kernels", C.c_uint32), ("ms_filter", C.c_float),
                ("exact_candidates", C.c_uint64), ("ms_recheck", C.c_float),
                ("ms_rerank_dist", C.c_float), ("rerank_candidates", C.c_uint64),
                ("filter_live_entries", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


lib = C.CDLL(LIB_PATH)


def _sig(name, args, res=_int):
    f = getattr(lib, name)
    f.argtypes = args
    f.restype = res
    return f


_sig("pqrr_dev_last_error", [], C.c_char_p)
_sig("pqrr_dev_device_count", [C.POINTER(_int)])
_sig("pqrr_dev_launch_count", [], _u64)
_sig("pqrr_dev_assign_batch", [_int, _f32p, _sz, _u32, _f32p, _u32, _u32p, _f32p])
_sig("pqrr_dev_encode_batch", [_int, _f32p, _u32, _u32, _u32, _f32p, _sz, _u8p])
_sig("pqrr_dev_decode_batch", [_int, _f32p, _u32, _u32, _u32, _u8p, _sz, _f32p])
_sig("pqrr_dev_build_lut", [_int, _f32p, _u32, _u32, _u32, _f32p, _sz, _f32p])
_sig("pqrr_dev_scan_topk", [_int, _f32p, _u32, _u32, _u8p, _sz, _sz, _u32, _u32p, _f32p,
                            C.POINTER(_sz)])
_sig("pqrr_dev_kmeans_train", [_int, _f32p, _sz, _u32, _u32, _u32, _u64, _u32, _f32p,
                               C.POINTER(C.c_double), _vp])
_sig("pqrr_dev_pq_train", [_int, _f32p, _sz, _u32, _u32, _u32, _u32, _u64, _u32, _f32p])
_sig("pqrr_dev_ivf_train", [_int, _f32p, _sz, _u32, _u32, _u32, _u32, _u32, _u64, _f32p, _f32p])
_sig("pqrr_dev_ivf_refine_train", [_int, _f32p, _u32, _f32p, _u32, _u32, _u32, _f32p, _sz, _u32,
                                   _u32, _u64, _f32p])
_sig("pqrr_dev_synth", [_int, _u64, _u32, _u32, _u32, _u64, _sz, _u8p])
_sig("pqrr_dev_index_create", [_int, _u32, _u32, _f32p, _u32, _f32p, _u32, _vp, _u32,
                               C.POINTER(_vp)])
_sig("pqrr_dev_index_destroy", [_vp])
_sig("pqrr_dev_add_u8", [_vp, _u8p, _sz, _u32])
_sig("pqrr_dev_add_f32", [_vp, _f32p, _sz, _u32])
_sig("pqrr_dev_add_synthetic", [_vp, _u64, _u32, _u64, _sz, _u32])
_sig("pqrr_dev_finalize", [_vp])
_sig("pqrr_dev_index_get_info", [_vp, C.POINTER(IndexInfo)])
_sig("pqrr_dev_export_lists", [_vp, _vp, _vp, _vp, _vp])
_sig("pqrr_dev_search_u8", [_vp, _u8p, _sz, _u32, _sz, _sz, _u32p, _f32p, _u32p])
_sig("pqrr_dev_search_f32", [_vp, _f32p, _sz, _u32, _sz, _sz, _u32p, _f32p, _u32p])
_sig("pqrr_dev_search_u8_device", [_vp, _vp, _sz, _u32, _sz, _sz, _vp, _vp, _vp, _vp])
_sig("pqrr_dev_search_u8_enqueue", [_vp, _vp, _sz, _u32, _sz, _sz, _vp, _vp, _vp, _vp])
_sig("pqrr_dev_search_finish", [_vp])
_sig("pqrr_dev_index_set_graph", [_vp, _int])
_sig("pqrr_dev_rerank_u8", [_vp, _u8p, _sz, _u32p, _u32p, _sz, _sz, _u32p, _f32p])
_sig("pqrr_dev_rerank_f32", [_vp, _f32p, _sz, _u32p, _u32p, _sz, _sz, _u32p, _f32p])
_sig("pqrr_dev_reconstruct", [_vp, _u32p, _sz, _f32p])
_sig("pqrr_dev_lookup_ids", [_vp, _u32p, _sz, _vp, _vp, _vp])
_sig("pqrr_dev_rerank_owned_u8_device", [_vp, _vp, _sz, _vp, _vp, _sz, _sz, _vp, _vp, _vp, _vp])
_sig("pqrr_dev_last_search_stats", [_vp, C.POINTER(SearchStats)])
_sig("pqrr_dev_load_lists", [_vp, _u64p, _u32p, _u8p, _vp])
_sig("pqrr_dev_merge_topk", [_int, _u32p, _f32p, _u32p, _sz, _u32, _u32, _u32, _u32p, _f32p, _u32p])
_sig("pqrr_dev_merge_topk_device", [_int, _vp, _vp, _vp, _sz, _u32, _u32, _u32, _vp, _vp, _vp, _vp])
_sig("pqrr_dev_assign_u8", [_int, _u8p, _sz, _u32, _f32p, _u32, _u32p])
_sig("pqrr_dev_index_device", [_vp, C.POINTER(_int)])
_sig("pqrr_dev_group_create", [_u32, C.POINTER(_vp), C.POINTER(_vp)])
_sig("pqrr_dev_group_search_u8", [_vp, _u8p, _sz, _u32, _sz, _sz, _int, _u32p, _f32p, _u32p])
_sig("pqrr_dev_group_size", [_vp, C.POINTER(_u32), C.POINTER(_int)])
_sig("pqrr_dev_group_destroy", [_vp])
_sig("pqrr_dev_merge_packed_device", [_int, _vp, _sz, _u32, _u32, _u32, _vp, _vp, _vp, _vp])
_sig("pqrr_dev_adc_index_create", [_int, _u32, _u32, _f32p, _u32, _vp, _u32, C.POINTER(_vp)])
_sig("pqrr_dev_refine_train", [_int, _f32p, _u32, _u32, _u32, _f32p, _sz, _u32, _u32, _u64, _f32p])
_sig("pqrr_dev_residual", [_int, _f32p, _u32, _u32, _u32, _f32p, _sz, _f32p])
_sig("pqrr_dev_export_codebooks", [_vp, _vp, _vp, _vp])
_sig("pqrr_dev_exact_knn_u8", [_int, _vp, _sz, _u8p, _sz, _u32, _u32, _u32p, _f32p, _u32p])
_sig("pqrr_dev_exact_knn_synthetic", [_int, _u64, _u32, _u64, _sz, _u8p, _sz, _u32, _u32p, _f32p, _u32p])
_sig("pqrr_dev_pair_bounds", [_int, _f32p, _sz, _u32, _f32p, _u32, _f32p, _u32, _u32, _u32p, _u32, _u32,
                              _f32p])
_sig("pqrr_dev_export_lists_subset", [_vp, _u32p, _u32, _u64p, _vp, _vp, _vp])
_cs = C.c_char_p
_sig("pqrr_dev_save_quantizer", [_cs, _u32, _u32, _u32, _f32p])
_sig("pqrr_dev_load_quantizer", [_cs, C.POINTER(_u32), C.POINTER(_u32), C.POINTER(_u32), _vp])
_sig("pqrr_dev_save_index", [_vp, _cs])
_sig("pqrr_dev_load_index", [_int, _cs, C.POINTER(_vp)])
_sig("pqrr_dev_save_adc_index", [_vp, _cs])
_sig("pqrr_dev_load_adc_index", [_int, _cs, C.POINTER(_vp)])
_sig("pqrr_dev_probe_index_kind", [_cs, C.POINTER(_int)])
_sig("pqrr_dev_reconstruct_codes", [_int, _f32p, _u32, _u32, _f32p, _u32, _u32, _u8p, _u8p, _sz,
                                    _f32p])

# Symbols include/pqrr_dev.h declares (checked by the CPU test suite).
EXPORTED = [
    "pqrr_dev_last_error", "pqrr_dev_device_count", "pqrr_dev_launch_count",
    "pqrr_dev_assign_batch", "pqrr_dev_assign_u8", "pqrr_dev_encode_batch", "pqrr_dev_decode_batch",
    "pqrr_dev_build_lut", "pqrr_dev_scan_topk", "pqrr_dev_kmeans_train", "pqrr_dev_pq_train",
    "pqrr_dev_ivf_train", "pqrr_dev_ivf_refine_train", "pqrr_dev_synth",
    "pqrr_dev_index_create", "pqrr_dev_index_destroy", "pqrr_dev_add_u8", "pqrr_dev_add_f32",
    "pqrr_dev_add_synthetic", "pqrr_dev_finalize", "pqrr_dev_index_get_info",
    "pqrr_dev_export_lists", "pqrr_dev_search_u8", "pqrr_dev_search_f32",
    "pqrr_dev_search_u8_device", "pqrr_dev_search_u8_enqueue", "pqrr_dev_search_finish",
    "pqrr_dev_index_set_graph", "pqrr_dev_rerank_u8", "pqrr_dev_rerank_f32",
    "pqrr_dev_reconstruct", "pqrr_dev_lookup_ids", "pqrr_dev_last_search_stats", "pqrr_dev_load_lists",
    "pqrr_dev_merge_topk", "pqrr_dev_merge_topk_device", "pqrr_dev_merge_packed_device",
    "pqrr_dev_index_device", "pqrr_dev_group_create", "pqrr_dev_group_search_u8", "pqrr_dev_group_size",
    "pqrr_dev_group_destroy",
    "pqrr_dev_rerank_owned_u8_device",
    "pqrr_dev_adc_index_create", "pqrr_dev_refine_train", "pqrr_dev_residual",
    "pqrr_dev_reconstruct_codes", "pqrr_dev_export_codebooks", "pqrr_dev_export_lists_subset",
    "pqrr_dev_pair_bounds", "pqrr_dev_exact_knn_u8", "pqrr_dev_exact_knn_synthetic", "pqrr_dev_save_quantizer",
    "pqrr_dev_load_quantizer", "pqrr_dev_save_index", "pqrr_dev_load_index",
    "pqrr_dev_save_adc_index", "pqrr_dev_load_adc_index", "pqrr_dev_probe_index_kind",
]


class PqrrError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class DeviceUnavailable(PqrrError):
    pass


def check(rc: int) -> None:
    """Map a status to the reference's exception types (SPEC.md error strings)."""
    if rc == PQRR_OK:
        return
    msg = lib.pqrr_dev_last_error().decode()
    if rc in (PQRR_EINVAL, PQRR_ESHORTLIST):
        raise ValueError(msg)  # std::invalid_argument in the reference
    if rc == PQRR_ENODEV:
        raise DeviceUnavailable(rc, msg)
    if rc == PQRR_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise PqrrError(rc, msg)


def device_count() -> int:
    n = _int(0)
    lib.pqrr_dev_device_count(C.byref(n))
    return n.value


def launch_count() -> int:
    return int(lib.pqrr_dev_launch_count())
