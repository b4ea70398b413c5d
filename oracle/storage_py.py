"""Independent restatement of the "PQRR" container (storage.hpp:14-28,
SPEC.md:131,194,275) in plain Python struct/numpy — TEST INFRASTRUCTURE ONLY
(the product's reader/writer is paper_1102_3828_b200/csrc/storage.cu).  The
reference declares these functions without bodies; the byte layout below is
our reading of its header comment, stated once in DESIGN.md §10, and the
tests check the product byte-for-byte against it.
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"PQRR"
VERSION = 1


class Corrupt(ValueError):
    def __init__(self):
        super().__init__("corrupt file")


def quantizer_block(books, d, m, ks) -> bytes:
    """magic, version u8, d/m/ks u32, m*ks*(d/m) f32 (storage.hpp:18-19)."""
    b = np.ascontiguousarray(books, "<f4").reshape(-1)
    assert b.size == ks * d
    return MAGIC + struct.pack("<BIII", VERSION, d, m, ks) + b.tobytes()


def adc_file(books, d, m, ks, codes, rbooks=None, mprime=0, rcodes=None) -> bytes:
    """quantizer block, n u64, n*m code bytes, optional refine section."""
    codes = np.ascontiguousarray(codes, np.uint8)
    out = quantizer_block(books, d, m, ks) + struct.pack("<Q", codes.shape[0]) + codes.tobytes()
    if mprime:
        out += refine_section(rbooks, d, mprime, ks, rcodes)
    return out


def refine_section(rbooks, d, mprime, ks, rcodes) -> bytes:
    """refine quantizer block, m' u32, n*m' bytes."""
    return (quantizer_block(rbooks, d, mprime, ks) + struct.pack("<I", mprime)
            + np.ascontiguousarray(rcodes, np.uint8).tobytes())


def ivf_file(books, d, m, ks, coarse, offsets, ids, codes, rbooks=None, mprime=0,
             rcodes_by_id=None) -> bytes:
    """residual quantizer block, c u32, coarse f32, c x u64 lengths, per-list
    (id u32, m code bytes) entries, optional refine section (id order)."""
    coarse = np.ascontiguousarray(coarse, "<f4")
    c = coarse.shape[0]
    offsets = np.asarray(offsets, np.uint64)
    lens = (offsets[1:] - offsets[:-1]).astype("<u8")
    rec = np.zeros(len(ids), dtype=[("id", "<u4"), ("code", np.uint8, (m,))])
    rec["id"] = ids
    rec["code"] = np.asarray(codes, np.uint8).reshape(-1, m)
    out = (quantizer_block(books, d, m, ks) + struct.pack("<I", c) + coarse.tobytes()
           + lens.tobytes() + rec.tobytes())
    if mprime:
        out += refine_section(rbooks, d, mprime, ks, rcodes_by_id)
    return out


class _R:
    def __init__(self, b: bytes):
        self.b, self.p = b, 0

    def take(self, n):
        if n > len(self.b) - self.p:
            raise Corrupt()
        v = self.b[self.p:self.p + n]
        self.p += n
        return v

    def unpack(self, fmt):
        return struct.unpack(fmt, self.take(struct.calcsize(fmt)))


def read_quantizer_block(r: _R):
    if r.take(4) != MAGIC:
        raise Corrupt()
    ver, d, m, ks = r.unpack("<BIII")
    if ver != VERSION or d == 0 or m == 0 or ks == 0 or d % m:
        raise Corrupt()
    books = np.frombuffer(r.take(4 * ks * d), "<f4").reshape(m, ks, d // m)
    return d, m, ks, books


def read_quantizer(b: bytes):
    r = _R(b)
    q = read_quantizer_block(r)
    if r.p != len(b):
        raise Corrupt()
    return q
