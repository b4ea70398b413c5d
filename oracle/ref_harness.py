"""Reference-side harness of the parity checks and the CPU baseline.

TEST INFRASTRUCTURE ONLY: imported by tests/ and by the cpu_baseline /
--impl reference legs of bench.py, never by the product package.  Everything
here runs on the host:

* ``cpu_build``      — the whole IVFADC+R index built WITHOUT the device:
  codebooks by the oracle's k-means restatement (kmeans.hpp:30-38,
  ivf_index.hpp:48-52,66-70), then the reference's own
  ``kernels::assign_batch`` / ``encode_batch`` (kernels.cpp:21-46, compiled
  in place into oracle/_ref) for the coarse assignment and both PQ encodings,
  and the id-ascending list layout of ivf_index.hpp:15-22 (a stable sort by
  list).  Residual conventions: r0 = y - C_a (ivf_index.hpp:54-55) and
  r1 = y - (C_a + p) (ivf_index.hpp:66-67), in fp32 like the reference.
* ``ref_search``     — the reference search + re-rank (oracle/_ref:
  scan_topk per probed list, TopK merge, ivf_rerank) over a host index.
* ``probed_reference`` — the same search over a device-built index too large
  for the host (1B vectors): per batch of queries, only the lists those
  queries probe are exported (id-ascending), with ids renumbered by rank, so
  the reference's id-indexed arrays stay small and every (dist, id) order is
  kept.  A query only reads its probed lists, so its result is the full
  index's.
* ``reencode_sample`` — the add-path check at any scale: rows of random ids
  regenerated on the host and pushed through the reference's assign /
  encode, to compare with the device index's list / code / refinement code
  of those ids.
"""
from __future__ import annotations

import os
import platform
import time

import numpy as np

from .oracle_py import Oracle, RefLib

SYNTH_BASE, SYNTH_TRAIN, SYNTH_QUERY = 2, 1, 3


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class HostIndex:
    """A host IvfIndex (ivf_index.hpp:27-41) + RefineCodes (refine.hpp:21-28)."""

    def __init__(self, coarse, books, rbooks, m, mprime, offs, ids, codes, list_of_id, codes_by_id,
                 rcodes_by_id):
        self.coarse, self.books, self.rbooks = coarse, books, rbooks
        self.m, self.mprime = m, mprime
        self.offs, self.ids, self.codes = offs, ids, codes
        self.list_of_id, self.codes_by_id, self.rcodes_by_id = list_of_id, codes_by_id, rcodes_by_id

    @property
    def n(self):
        return len(self.ids)

    def rcodes_list_order(self):
        return self.rcodes_by_id[self.ids]


def encode_rows(ref: RefLib, coarse, books, rbooks, m, mprime, y):
    """ivf_build + ivf_refine_encode of one chunk through the reference's
    kernels: (assign, codes, rcodes)."""
    yf = np.ascontiguousarray(y, np.float32)
    a, _ = ref.assign(yf, coarse)
    ca = coarse[a]
    r0 = yf - ca                                  # ivf_index.hpp:54-55
    codes = ref.encode(books, r0, m)
    rcodes = None
    if mprime:
        p = ref.decode(books, codes, yf.shape[1])
        rec1 = ca + p                             # (C_a + p) first, ivf_index.hpp:66-67
        r1 = yf - rec1
        rcodes = ref.encode(rbooks, r1, mprime)
    return a, codes, rcodes


def cpu_train(cfg, seed=0, log=None, orc: Oracle | None = None):
    """Codebooks on the host: ivf_train + ivf_refine_train (oracle restatement,
    bit-identical to the device trainer)."""
    o = orc or Oracle()
    o.set_threads(0)
    t0 = time.time()
    centers = o.synth_centers(seed, cfg["clusters"], 128)
    tr = o.synth_rows(seed, SYNTH_TRAIN, 0, cfg["train"], centers).astype(np.float32)
    coarse, books = o.ivf_train(tr, cfg["kc"], cfg["m"], iterations=25, seed=seed)
    rbooks = o.ivf_refine_train(coarse, books, cfg["m"], tr, cfg["mprime"], iterations=25, seed=seed)
    if log:
        log(f"[cpu] trained codebooks on {cfg['train']} vectors in {time.time() - t0:.1f}s")
    return coarse, books, rbooks, centers


def cpu_build(cfg, seed=0, log=None, chunk=1 << 20, codebooks=None) -> HostIndex:
    """The whole index on the host (no device code at all)."""
    o = Oracle()
    ref = RefLib()
    ref.set_threads(0)
    o.set_threads(0)
    if codebooks is None:
        coarse, books, rbooks, centers = cpu_train(cfg, seed, log, o)
    else:
        coarse, books, rbooks = codebooks
        centers = o.synth_centers(seed, cfg["clusters"], 128)
    n, m, mp = cfg["n"], cfg["m"], cfg["mprime"]
    t0 = time.time()
    assign = np.empty(n, np.uint32)
    codes_by_id = np.empty((n, m), np.uint8)
    rcodes_by_id = np.empty((n, mp), np.uint8)
    for r0 in range(0, n, chunk):
        nr = min(chunk, n - r0)
        y = o.synth_rows(seed, SYNTH_BASE, r0, nr, centers)
        a, c, rc = encode_rows(ref, coarse, books, rbooks, m, mp, y)
        assign[r0:r0 + nr] = a
        codes_by_id[r0:r0 + nr] = c
        rcodes_by_id[r0:r0 + nr] = rc
    # IvfList layout: per list, ids ascending (a stable sort by list)
    ids = np.argsort(assign, kind="stable").astype(np.uint32)
    offs = np.zeros(cfg["kc"] + 1, np.uint64)
    offs[1:] = np.cumsum(np.bincount(assign, minlength=cfg["kc"]))
    if log:
        log(f"[cpu] added {n} vectors with the reference kernels in {time.time() - t0:.1f}s")
    return HostIndex(coarse, books, rbooks, m, mp, offs, ids, codes_by_id[ids], assign, codes_by_id,
                     rcodes_by_id)


def ref_search(ref: RefLib, hx: HostIndex, queries, w, kprime, k):
    """ivf_search_batch + ivf_rerank with the reference's kernels (all host
    threads the RefLib is set to)."""
    qf = np.ascontiguousarray(queries, np.float32)
    sl_i, sl_d, sl_c = ref.ivf_search(hx.coarse, hx.books, hx.m, hx.offs, hx.ids, hx.codes, qf, w,
                                      kprime)
    if not k:
        return sl_i, sl_d, sl_c
    ri, rd = ref.ivf_rerank(hx.coarse, hx.books, hx.rbooks, hx.m, hx.mprime, hx.list_of_id,
                            hx.codes_by_id, hx.rcodes_by_id, qf, sl_i, sl_c, k)
    return ri, rd, np.full(len(qf), k, np.uint32)


def probed_subindex(export_subset, coarse, books, rbooks, m, mprime, kc, queries, w):
    """Host sub-index of the lists `queries` probe, exported from a device
    index by ``export_subset(lists) -> (offs, ids, codes, rcodes)``; ids are
    renumbered by rank among the exported entries (order-preserving).
    Returns (HostIndex over local ids, local -> global id map, #lists)."""
    qf = np.ascontiguousarray(queries, np.float32)
    probes, _ = Oracle().coarse_probe(coarse, qf, w)
    U = np.unique(probes).astype(np.uint32)
    offs_u, ids_u, codes_u, rc_u = export_subset(U)
    lens = np.zeros(kc, np.uint64)
    lens[U] = np.diff(offs_u)
    full_offs = np.zeros(kc + 1, np.uint64)
    full_offs[1:] = np.cumsum(lens)
    order = np.argsort(ids_u, kind="stable")
    gid_sorted = ids_u[order]
    local = np.empty(len(ids_u), np.uint32)
    local[order] = np.arange(len(ids_u), dtype=np.uint32)
    list_of_local = np.empty(len(ids_u), np.uint32)
    list_of_local[local] = np.repeat(U, np.diff(offs_u).astype(np.int64))
    codes_by_local = np.empty_like(codes_u)
    codes_by_local[local] = codes_u
    rc_by_local = None
    if rc_u is not None:
        rc_by_local = np.empty_like(rc_u)
        rc_by_local[local] = rc_u
    hx = HostIndex(coarse, books, rbooks, m, mprime, full_offs, local, codes_u, list_of_local,
                   codes_by_local, rc_by_local)
    return hx, gid_sorted, len(U)


def probed_reference(ref: RefLib, export_subset, coarse, books, rbooks, m, mprime, kc, queries, w,
                     kprime, k, batch=32):
    """Reference search over a device index exported list by list, in query
    batches.  Returns (ids, dists, seconds of reference search, lists exported)."""
    nq = len(queries)
    width = k if k else kprime
    out_i = np.zeros((nq, width), np.uint32)
    out_d = np.zeros((nq, width), np.float32)
    t_search = 0.0
    nl = 0
    for b0 in range(0, nq, batch):
        qs = queries[b0:b0 + batch]
        hx, gid, nlb = probed_subindex(export_subset, coarse, books, rbooks, m, mprime, kc, qs, w)
        nl += nlb
        t0 = time.perf_counter()
        ri, rd, _ = ref_search(ref, hx, qs, w, kprime, k)
        t_search += time.perf_counter() - t0
        out_i[b0:b0 + len(qs)] = gid[ri]
        out_d[b0:b0 + len(qs)] = rd
    return out_i, out_d, t_search, nl


def sample_ids(n, nblocks=256, block=1024, seed=12345):
    """Random ids of an n-vector index: nblocks random runs of `block`
    consecutive ids (the generator is counter-based, so runs are cheap)."""
    rng = np.random.default_rng(seed)
    block = min(block, n)
    starts = np.sort(rng.choice(max(n - block, 1), size=min(nblocks, max(n // block, 1)), replace=False))
    return starts, block


def reencode_sample(cfg, coarse, books, rbooks, starts, block, seed=0):
    """(ids, list, codes, rcodes) of the sampled id runs, encoded on the host
    with the reference's kernels from host-generated rows."""
    o = Oracle()
    o.set_threads(0)
    ref = RefLib()
    ref.set_threads(0)
    centers = o.synth_centers(seed, cfg["clusters"], 128)
    rows = np.concatenate([o.synth_rows(seed, SYNTH_BASE, int(s), block, centers) for s in starts])
    ids = np.concatenate([np.arange(s, s + block, dtype=np.uint32) for s in starts])
    a, c, rc = encode_rows(ref, coarse, books, rbooks, cfg["m"], cfg["mprime"], rows)
    return ids, a, c, rc


def recall_at(ids, gt_nearest, r):
    """recall_at_r (eval.hpp:21-24): fraction of queries whose exact nearest
    id is among the first min(r, len) results."""
    return float(np.mean([gt_nearest[q] in ids[q, :r] for q in range(len(gt_nearest))]))
