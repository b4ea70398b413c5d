"""IVFADC+R search benchmark (BASELINE.json metric) — one JSON line on rank 0.

Workload (default): BASELINE.json configs[3] ("C4"), the largest config that
fits one B200: n = 1B SIFT-like uint8 vectors (4096-component mixture, seed
0), 1M training vectors, 10k queries, d = 128, Kc = 8192, m = 8, m' = 32,
w = 64, k' = 10000, top-100 (the paper's 1B IVFADC+R row).
`--config C1|C2|C3` selects the other configs, `--config C5` the batch sweep.
A step is one fused batched search of all queries (coarse probe -> LUT ->
ADC scan -> exact top-k' -> residual-PQ re-rank -> top-k).

  value : queries/s with queries resident in HBM, device-timed (CUDA events on
          the index stream), L2 flushed between steps.
  e2e   : same metric through the public host API (pqrr_dev_search_u8 via
          ctypes) from pinned host memory, H2D of the queries and D2H of the
          results inside the timed region.
  roofline : the dominant kernel of the step (per-kernel CUDA events on the
          index stream), its algorithmic bytes against its bound.
  cpu_baseline : the reference's CPU implementation (oracle/_ref: the
          reference's kernels.cpp scan_topk / assign / encode + headers' TopK /
          l2_sq) on the host cores, with the parity evidence of the same run:
          n <= 10M ("full"): the whole index rebuilt on the CPU (codebooks,
          lists, codes, refinement codes compared byte for byte) and every
          query searched; larger n ("sample"): the first --ref-queries queries
          over their probed lists exported from the device index, plus a
          random-id re-encode of the add path.
  --impl reference : the reference's CPU path alone, on the same config.

Multi-GPU (torchrun): the database is sharded by id range; each rank searches
its shard with the full query batch; per-rank top-k lists are all-gathered and
merged under (dist, id).  Timing is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: n, train, nq, clusters, Kc, m, m', w, k', k
    "C1": dict(n=1_000_000, train=100_000, nq=1000, clusters=1024, kc=1024, m=8, mprime=8, w=8,
               kprime=100, k=100),
    "C2": dict(n=10_000_000, train=1_000_000, nq=10_000, clusters=4096, kc=1024, m=8, mprime=16,
               w=16, kprime=1000, k=100),
    "C3": dict(n=100_000_000, train=1_000_000, nq=10_000, clusters=4096, kc=8192, m=8, mprime=16,
               w=64, kprime=1000, k=100),
    "C4": dict(n=1_000_000_000, train=1_000_000, nq=10_000, clusters=4096, kc=8192, m=8,
               mprime=32, w=64, kprime=10_000, k=100),
    # batch-size sweep (BASELINE configs[4], quoted at 8 GPUs; here one GPU holds all 1B)
    "C5": dict(n=1_000_000_000, train=1_000_000, nq=65_536, clusters=4096, kc=8192, m=8,
               mprime=16, w=128, kprime=1000, k=100),
}
C5_BATCHES = [1, 16, 256, 4096, 65536]
SEED = 0
METRIC = "IVFADC+R queries/sec at oracle-matched recall@1/10/100; scan HBM GB/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """SM clock and throttle reasons sampled (NVML, every 2 ms) during the timed
    region — the same fields as the recipe's nvidia-smi clocks line."""

    REASONS = {  # nvmlClocksEventReason* bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap",
    }

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                sm = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((float(sm), int(rs)))
            except Exception:
                pass
            self._stop.wait(0.002)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"],
                    "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = sorted({name for _, rs in self.rows for bit, name in self.REASONS.items()
                          if rs & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml"}


def measured_peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------- setup
def train_codebooks(pq, cfg, device):
    t0 = time.time()
    train = pq.synth(1, 0, cfg["train"], cfg["clusters"], seed=SEED, device=device).astype(np.float32)
    prm = pq.TrainParams(iterations=25, seed=SEED)
    coarse, P = pq.ivf_train(train, cfg["kc"], cfg["m"], params=prm, device=device)
    rq = pq.ivf_refine_train(coarse, P, train, cfg["mprime"], prm, device=device)
    log(f"[setup] trained codebooks on {cfg['train']} vectors in {time.time() - t0:.1f}s")
    return coarse, P, rq


def build_index(pq, cfg, coarse, P, rq, device, shard, nshards):
    n = cfg["n"]
    lo = n * shard // nshards
    hi = n * (shard + 1) // nshards
    t0 = time.time()
    ix = pq.IvfIndex(coarse, P, rq, device)
    ix.add_synthetic(SEED, cfg["clusters"], lo, hi - lo, id_base=lo)
    ix.finalize()
    dt = time.time() - t0
    log(f"[setup] added ids [{lo}, {hi}) on device {device} in {dt:.1f}s")
    return ix, lo, hi, dt


# ---------------------------------------------------------------- reference arm
REF_SAMPLE = {"C1": 1000, "C2": 1024, "C3": 64, "C4": 32, "C5": 32}


class FileLists:
    """export_subset() over the probed lists a setup process wrote to disk
    (np.load with mmap): the reference arm reads the device-built index
    without loading any product code."""

    def __init__(self, d):
        self.d = d
        self.U = np.load(os.path.join(d, "lists.npy"))
        self.offs = np.load(os.path.join(d, "offs.npy"))
        self.ids = np.load(os.path.join(d, "ids.npy"), mmap_mode="r")
        self.codes = np.load(os.path.join(d, "codes.npy"), mmap_mode="r")
        rp = os.path.join(d, "rcodes.npy")
        self.rcodes = np.load(rp, mmap_mode="r") if os.path.exists(rp) else None
        self.where = {int(l): i for i, l in enumerate(self.U)}

    def __call__(self, lists):
        idx = [self.where[int(l)] for l in lists]
        lens = np.array([self.offs[i + 1] - self.offs[i] for i in idx], np.uint64)
        offs = np.zeros(len(idx) + 1, np.uint64)
        offs[1:] = np.cumsum(lens)
        sl = [slice(int(self.offs[i]), int(self.offs[i + 1])) for i in idx]
        ids = np.concatenate([self.ids[s] for s in sl]) if sl else np.zeros(0, np.uint32)
        codes = np.concatenate([self.codes[s] for s in sl]) if sl else np.zeros((0, 8), np.uint8)
        rc = np.concatenate([self.rcodes[s] for s in sl]) if self.rcodes is not None else None
        return offs, ids, codes, rc

    def nbytes(self):
        return int(sum(os.path.getsize(os.path.join(self.d, f)) for f in os.listdir(self.d)))


def ref_tmpdir(need_bytes):
    """A scratch directory with room for the exported lists (page cache backed)."""
    import shutil
    import tempfile

    for base in (os.environ.get("PQRR_REF_TMP"), "/dev/shm", "/tmp", ROOT):
        if base and os.path.isdir(base) and os.access(base, os.W_OK):
            try:
                if shutil.disk_usage(base).free > 1.2 * need_bytes:
                    return tempfile.mkdtemp(prefix="pqrr_ref_", dir=base)
            except OSError:
                pass
    raise RuntimeError("no scratch directory with room for the exported lists")


def export_reference_input(args, cfg):
    """Setup process of the reference arm at n > 10M (C3-C5): builds the index
    on the device (the host cannot: ~1e15 assign operations), exports the lists
    the reference's sample queries probe (id-ascending, ivf_index.hpp:15-16) and
    the device codes of a random id sample for the add-path check, to
    --export-dir.  The timed reference process never loads libpqrr_b200.so."""
    import paper_1102_3828_b200 as pq
    from oracle.oracle_py import Oracle
    from oracle import ref_harness as H

    d = args.export_dir
    coarse, P, rq = train_codebooks(pq, cfg, 0)
    ix, _, _, add_s = build_index(pq, cfg, coarse, P, rq, 0, 0, 1)
    o = Oracle()
    o.set_threads(0)
    centers = o.synth_centers(SEED, cfg["clusters"], 128)
    qs = o.synth_rows(SEED, H.SYNTH_QUERY, 0, args.ref_queries, centers).astype(np.float32)
    probes, _ = o.coarse_probe(coarse.centroids, qs, cfg["w"])
    U = np.unique(probes).astype(np.uint32)
    offs, ids, codes, rc = ix.export_lists_subset(U)
    for name, arr in (("lists", U), ("offs", offs), ("ids", ids), ("codes", codes), ("rcodes", rc),
                      ("coarse", coarse.centroids), ("books", P.flat()), ("rbooks", rq.pq.flat())):
        if arr is not None:
            np.save(os.path.join(d, name + ".npy"), arr)
    starts, block = H.sample_ids(cfg["n"], nblocks=64)
    sid = np.concatenate([np.arange(s, s + block, dtype=np.uint32) for s in starts])
    dl, dc, drc = ix.lookup_ids(sid)
    np.savez(os.path.join(d, "add_sample.npz"), starts=starts, block=block, lists=dl, codes=dc,
             rcodes=drc if drc is not None else np.zeros(0, np.uint8), add_s=add_s)
    ix.close()
    log(f"[setup] exported {len(U)} probed lists ({len(ids)} entries) for {args.ref_queries} queries")


def run_reference(args, cfg, rank, world):
    """The reference's CPU implementation of the path (oracle/_ref) on this
    host's cores, on a bounded query sample per step.

    n <= 10M (C1, C2): the index is built on the host too (oracle k-means for
    the codebooks, the reference's assign_batch / encode_batch for the lists).
    C3-C5 (100M-1B vectors) cannot be built on the host in a bench run (the
    assignment alone is ~1e15 element operations): a separate setup process
    builds it on the device and exports the lists the sample queries probe to
    scratch files (export_reference_input).  This process reads them and
    never loads product code; the add path is checked on a random id sample
    against the reference's own encoder."""
    if rank != 0:
        return
    from oracle.oracle_py import Oracle, RefLib, build, ref_available
    from oracle import ref_harness as H

    if not ref_available():
        build()
    ref = RefLib()
    cores = H.host_cores()
    ref.set_threads(cores)
    sample = REF_SAMPLE[args.config]
    W, K = args.warmup, args.steps
    nq = cfg["nq"]
    extra = {}
    t_setup = time.time()
    o = Oracle()
    centers = o.synth_centers(SEED, cfg["clusters"], 128)
    if cfg["n"] <= CPU_BUILD_MAX:
        hx = H.cpu_build(cfg, SEED, log)
        queries = o.synth_rows(SEED, H.SYNTH_QUERY, 0, nq, centers)
        index_build = "host: oracle k-means + reference assign_batch/encode_batch (no device code)"

        def step(i):
            qs = queries[(i * sample) % nq:][:sample]
            t0 = time.perf_counter()
            H.ref_search(ref, hx, qs, cfg["w"], cfg["kprime"], cfg["k"])
            return len(qs), time.perf_counter() - t0

        def one_thread(qs):
            return H.ref_search(ref, hx, qs, cfg["w"], cfg["kprime"], cfg["k"])
    else:
        nref = (min(W, 1) + K) * sample
        per_list = cfg["n"] / cfg["kc"] * (cfg["m"] + cfg["mprime"] + 4)
        d = ref_tmpdir(min(cfg["kc"], nref * cfg["w"]) * per_list)
        try:
            cmd = [sys.executable, os.path.abspath(__file__), "--config", args.config, "--export-dir", d,
                   "--ref-queries", str(nref)]
            subprocess.run(cmd, check=True, stdout=sys.stderr)
            fl = FileLists(d)
            cb = (np.load(os.path.join(d, "coarse.npy")), np.load(os.path.join(d, "books.npy")),
                  np.load(os.path.join(d, "rbooks.npy")))
            queries = o.synth_rows(SEED, H.SYNTH_QUERY, 0, nref, centers)
            a = np.load(os.path.join(d, "add_sample.npz"))
            ids, al, ac, arc = H.reencode_sample(cfg, *cb, a["starts"], int(a["block"]), seed=SEED)
            extra["index_check"] = {
                "ids": int(len(ids)), "list_match": float(np.mean(a["lists"] == al)),
                "codes_match": float(np.mean(np.all(a["codes"] == ac, axis=1))),
                "rcodes_match": float(np.mean(np.all(a["rcodes"] == arc, axis=1))),
                "sample": f"{len(a['starts'])} random runs of {int(a['block'])} consecutive ids, "
                          "reference assign/encode on host-generated rows vs the device index"}
            index_build = (f"device, in a separate setup process (bench.py --export-dir): a host build of "
                           f"{cfg['n']:.0e} vectors is ~1e15 assign operations; the {len(fl.U)} lists the "
                           f"{nref} sample queries probe ({fl.nbytes() / 1e9:.1f} GB) exported to scratch "
                           "files; this process loads no product code")

            def step(i):
                qs = queries[i * sample:(i + 1) * sample]
                _, _, ts, _ = H.probed_reference(ref, fl, *cb, cfg["m"], cfg["mprime"], cfg["kc"], qs,
                                                 cfg["w"], cfg["kprime"], cfg["k"], batch=sample)
                return len(qs), ts

            def one_thread(qs):
                return H.probed_reference(ref, fl, *cb, cfg["m"], cfg["mprime"], cfg["kc"], qs, cfg["w"],
                                          cfg["kprime"], cfg["k"], batch=len(qs))
            # all timed steps run before the scratch files go away
            t_setup = time.time() - t_setup
            return _reference_line(args, cfg, world, ref, cores, sample, step, one_thread, queries,
                                   index_build, t_setup, extra)
        finally:
            import shutil

            shutil.rmtree(d, ignore_errors=True)
    t_setup = time.time() - t_setup
    return _reference_line(args, cfg, world, ref, cores, sample, step, one_thread, queries, index_build,
                           t_setup, extra)


def _reference_line(args, cfg, world, ref, cores, sample, step, one_thread, queries, index_build, t_setup,
                    extra):
    from oracle import ref_harness as H

    W, K = args.warmup, args.steps
    for i in range(min(W, 1)):
        step(i)
    done, dt = 0, 0.0
    for i in range(K):
        n_i, t_i = step(i + min(W, 1))
        done += n_i
        dt += t_i
    v = done / dt
    # single-thread time per query (eval.hpp:49,63: BenchRow.time_per_query)
    ref.set_threads(1)
    n1 = 2 if cfg["n"] > CPU_BUILD_MAX else 4
    t0 = time.perf_counter()
    one_thread(queries[:n1])
    t1q = (time.perf_counter() - t0) / n1
    ref.set_threads(cores)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "queries/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": dt / K * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": args.config, **cfg, "parallelism": f"cpu-openmp x{cores}"},
        "cpu_baseline": {"value": v, "unit": "queries/s", "cores": cores, "kind": "reference",
                         "cpu_model": H.cpu_model(),
                         "sample": f"{sample} queries per step (of {cfg['nq']}), OpenMP over queries",
                         "time_per_query_1thread_s": t1q, "index_build": index_build,
                         "setup_s": round(t_setup, 1)},
        "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        **extra,
    }
    print(json.dumps(line), flush=True)


CPU_BUILD_MAX = 10_000_000  # host-built index (reference arm, full parity) up to C2


def add_check(H, cfg, ix, cb, starts, block):
    """Random-id sample of the device add path against the reference's own
    assign / encode on host-generated rows: list, code and refinement code
    byte for byte (ivf_index.hpp:54-56,72-73)."""
    t0 = time.time()
    ids, a, c, rc = H.reencode_sample(cfg, *cb, starts, block, seed=SEED)
    dl, dc, drc = ix.lookup_ids(ids)
    out = {"ids": int(len(ids)), "list_match": float(np.mean(dl == a)),
           "codes_match": float(np.mean(np.all(dc == c, axis=1))),
           "rcodes_match": float(np.mean(np.all(drc == rc, axis=1))) if rc is not None else None,
           "sample": f"{len(starts)} random runs of {block} consecutive ids"}
    log(f"[parity] add-path re-encode of {len(ids)} ids in {time.time() - t0:.1f}s: {out}")
    return out


# ---------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-recall", action="store_true")
    ap.add_argument("--parity", default="auto", choices=["auto", "full", "sample"],
                    help="full: host-built index + every query (n <= 10M); sample: probed-list "
                         "reference on --ref-queries queries + add-path re-encode sample")
    ap.add_argument("--ref-queries", type=int, default=256)
    ap.add_argument("--export-dir", default=None, help=argparse.SUPPRESS)  # reference-arm setup process
    ap.add_argument("--shard-mode", default="exact", choices=["local", "exact"],
                    help="N>1: per-shard shortlists (north star) or the single-index-exact flow")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    rank, world, local = dist_env()
    if args.export_dir:
        return export_reference_input(args, cfg)
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)
    if args.config == "C5":
        return run_sweep(args, cfg, rank, world)

    import torch
    import paper_1102_3828_b200 as pq

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = local
    coarse, P, rq = train_codebooks(pq, cfg, device)
    ix, lo, hi, add_s = build_index(pq, cfg, coarse, P, rq, device, rank, world)
    nq, k, kp, w = cfg["nq"], cfg["k"], cfg["kprime"], cfg["w"]
    queries = pq.synth(3, 0, nq, cfg["clusters"], seed=SEED, device=device)
    d_q = torch.from_numpy(queries).cuda()
    d_ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    d_dist = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    d_cnt = torch.empty(nq, dtype=torch.int32, device="cuda")
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()

    sharded = None
    if world > 1:
        from paper_1102_3828_b200.sharded import DeviceShardedSearch

        sharded = DeviceShardedSearch(ix, k, kp, w, mode=args.shard_mode)

    def run_once():
        if sharded is not None:  # shard search + NCCL all-gather + K7 merge
            oi, od, oc = sharded.search(d_q, stream)
            d_ids.copy_(oi)
            d_dist.copy_(od)
            return
        ix.search_device(d_q.data_ptr(), nq, w, kp, k, d_ids.data_ptr(), d_dist.data_ptr(),
                         d_cnt.data_ptr(), stream.cuda_stream)

    for _ in range(args.warmup):
        run_once()
    torch.cuda.synchronize()
    launches0 = pq.launch_count()
    step_ms, stats = [], []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (buffer 512 MB > 126 MB L2)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run_once()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            stats.append(ix.last_stats())
    torch.cuda.synchronize()
    launches = pq.launch_count() - launches0
    graph_replay = all(s["ms_scan"] == 0 for s in stats)
    if graph_replay:
        # batches of <= 1024 queries replay one captured CUDA graph, which times
        # only the total: take the per-stage times (rooflines, scan summary) from
        # two untimed searches on the synchronising path
        ix.set_graph(False)
        stats = []
        for _ in range(2):
            flush.zero_()
            run_once()
            stats.append(ix.last_stats())
        ix.set_graph(True)
        stats = stats[1:]
    total_ms = float(np.sum(step_ms))
    if dist:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = nq * args.steps / (total_ms / 1e3)
    res_ids = d_ids.cpu().numpy().view(np.uint32)
    res_dists = d_dist.cpu().numpy()

    # ---- e2e through the host API from pinned memory
    pinned_q = torch.from_numpy(queries).pin_memory()
    out_i = torch.empty((nq, k), dtype=torch.int32).pin_memory()
    out_d = torch.empty((nq, k), dtype=torch.float32).pin_memory()
    out_c = torch.empty((nq,), dtype=torch.int32).pin_memory()
    hq = pinned_q.numpy()
    # caller-owned page-locked result buffers, reused every step
    h_out = (out_i.numpy().view(np.uint32), out_d.numpy(), out_c.numpy().view(np.uint32))
    e2e_s = []
    for i in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        if sharded is None:
            ix.search(hq, w, kp, k, out=h_out)  # public host API (C ABI)
        else:
            dq = pinned_q.cuda(non_blocking=True)
            oi, od, oc = sharded.search(dq, stream)
            out_i.copy_(oi)
            out_d.copy_(od)
            torch.cuda.synchronize()
        e2e_s.append(time.perf_counter() - t0)
    e2e_total = float(np.sum(e2e_s[args.warmup:]))
    if dist:
        t = torch.tensor([e2e_total], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_val = nq * args.steps / e2e_total

    # ---- recall (exact ground truth) + parity against the reference
    extra = {}
    gt = None
    if not args.no_recall and world == 1:
        gt = ground_truth(pq, cfg, queries)
        for r in (1, 10, 100):
            extra[f"recall@{r}"] = float(np.mean([gt[q] in res_ids[q, :r] for q in range(len(gt))]))
        extra["recall_queries"] = int(len(gt))
    clocks = clk.summary()
    roof, kernels = rooflines(cfg, stats, clocks, local, args.config)
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (BASELINE.json SIFT-like generator, seed 0)",
        "config": {"workload": args.config, **cfg, "parallelism": f"id-range shards x{world}",
                   "shard_mode": args.shard_mode if world > 1 else "single index",
                   "search_path": ("one CUDA graph replay per batch (stage times from the synchronising path)"
                                   if graph_replay else "synchronising path (count readbacks between stages)"),
                   "l2": "flushed between steps (512 MB write)"},
        "e2e": {"value": e2e_val, "unit": "queries/s", "h2d_bytes_per_step": int(queries.nbytes),
                "d2h_bytes_per_step": int(nq * k * 8 + nq * 4)},
        "gpu_launches": int(launches),
        "roofline": roof,
        "kernels": kernels,
        "scan": scan_summary(cfg, stats),
        "add": {"vectors": int(hi - lo), "seconds": round(add_s, 2),
                "vectors_per_s": (hi - lo) / add_s if add_s > 0 else None,
                "note": "device add path (coarse assign + PQ + refinement PQ + list layout), "
                        "synthetic rows generated on the device; setup, outside the timed steps"},
        "stages_ms": {k2: round(float(np.mean([s[k2] for s in stats])), 4)
                      for k2 in ["ms_coarse", "ms_invert", "ms_sample_scan", "ms_threshold",
                                 "ms_filter", "ms_recheck", "ms_scan", "ms_select", "ms_rerank_dist",
                                 "ms_rerank", "ms_total"]},
        "search_stats": {k2: stats[-1][k2] for k2 in ["work_items", "retries", "stride", "kernels",
                                                     "scanned_entries", "sampled_entries",
                                                     "candidates", "rerank_candidates",
                                                     "filter_live_entries"]},
        "clocks": clocks,
        **extra,
    }
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = parity_and_baseline(args, cfg, pq, ix, coarse, P, rq, queries,
                                                   res_ids, res_dists, gt, extra)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


# ---------------------------------------------------------------- roofline
def rooflines(cfg, stats, clocks, device, config):
    """Per-kernel rooflines (mean over the timed steps; kernel times are CUDA
    events on the index stream around each launch).  Algorithmic work per
    launch, SURVEY.md §8(d), and the resource that bounds it:
      K5a re-rank distances (rerank_pair_kernel, CTA pairs): per shortlist
        entry the 8 PQ rows and m' refinement rows it must gather from on-chip
        memory, 512 B + 512 B (the coarse row is amortised over runs of one
        list) -- bound: the shared-memory pipe; its HBM side, k'(m + m' + 8) B
        per query (code, refinement code, shortlist key / position), is
        reported beside it;
      K4f filter: 1 B per (live (query, list) pair, entry, sub-space) LUT
        lookup it performs -- bound: the shared-memory pipe;
      K4r recheck (recheck_lut_kernel): per surviving candidate its probe
        rank and 8 code bytes read and its exact distance written back,
        16 B -- bound: HBM (the 8 lookups into the pair's exact LUT, 32 B of
        shared memory per candidate, are reported beside it).
    Shared-memory peak: 128 B/clk/SM x SMs x the SM clock sampled under load.
    `traffic` is ncu dram__bytes_read.sum + dram__bytes_write.sum per launch
    of the same kernel on the same commit (profiles/ncu_traffic.json), or null.
    The dominant (longest) kernel is `roofline`; all are in `kernels`."""
    import torch

    peak_hbm, kind = measured_peak_gbs()
    props = torch.cuda.get_device_properties(device)
    n_sm = props.multi_processor_count
    f_sm = (clocks.get("sm_mhz") or 1965.0) * 1e6
    smem_peak_gbs = 128.0 * n_sm * f_sm / 1e9
    smem_kind = f"128 B/clk/SM x {n_sm} SMs x {f_sm / 1e6:.0f} MHz"
    mean = lambda k: float(np.mean([s[k] for s in stats]))  # noqa: E731
    m, mp, d = cfg["m"], cfg["mprime"], 128
    traffic = ncu_traffic(config)
    ks = []
    t = mean("ms_rerank_dist")
    if t > 0:
        nc = mean("rerank_candidates")
        b = nc * (d // m * 4 * m + d // mp * 4 * mp)
        hb = nc * (m + mp + 8)
        ks.append({"kernel": "rerank_pair_kernel (K5a refined distances, CTA pairs)", "bound": "smem",
                   "kernel_ms": t, "algorithmic_bytes_per_launch": b,
                   "achieved": b / (t / 1e3) / 1e9, "peak": smem_peak_gbs, "unit": "GB/s",
                   "peak_kind": smem_kind, "traffic": traffic.get("rerank_pair_kernel"),
                   "hbm": {"algorithmic_bytes_per_launch": hb, "achieved": hb / (t / 1e3) / 1e9,
                           "peak": peak_hbm, "frac": hb / (t / 1e3) / 1e9 / peak_hbm, "peak_kind": kind}})
    t = mean("ms_filter")
    if t > 0:
        b = mean("filter_live_entries") * m
        ks.append({"kernel": "ivf_filter_kernel (K4f 5-bit LUT filter, incl. live-pair compaction)",
                   "bound": "smem", "kernel_ms": t, "algorithmic_bytes_per_launch": b,
                   "achieved": b / (t / 1e3) / 1e9, "peak": smem_peak_gbs, "unit": "GB/s",
                   "peak_kind": smem_kind, "traffic": traffic.get("ivf_filter_kernel")})
    t = mean("ms_recheck")
    if t > 0:
        nc = mean("candidates")
        b, sb = nc * 16, nc * m * 4
        ks.append({"kernel": "recheck_lut_kernel (K4r exact ADC of the survivors, per-pair LUTs)",
                   "bound": "hbm", "kernel_ms": t, "algorithmic_bytes_per_launch": b,
                   "achieved": b / (t / 1e3) / 1e9, "peak": peak_hbm, "unit": "GB/s", "peak_kind": kind,
                   "traffic": traffic.get("recheck_lut_kernel"),
                   "smem": {"algorithmic_bytes_per_launch": sb, "achieved": sb / (t / 1e3) / 1e9,
                            "peak": smem_peak_gbs, "frac": sb / (t / 1e3) / 1e9 / smem_peak_gbs,
                            "peak_kind": smem_kind}})
    for e in ks:
        e["frac"] = e["achieved"] / e["peak"]
    if not ks:
        return None, []
    top = max(ks, key=lambda e: e["kernel_ms"])
    share = top["kernel_ms"] / mean("ms_total") if mean("ms_total") > 0 else None
    return {**top, "share_of_step": share}, ks


def scan_summary(cfg, stats):
    """The scan in the north star's terms: scan-equivalent GB/s = Σ_q B_q
    (B_q = Σ_probed len·(m + 4)) over the filter + recheck time.
    The list-major scan reads each list once per work item of up to 64
    queries and skips dead (query, list) pairs, so this is NOT physical DRAM
    traffic (that is the ncu figure in profiles/) and not a roofline fraction."""
    mean = lambda k: float(np.mean([s[k] for s in stats]))  # noqa: E731
    t = mean("ms_scan")
    b = mean("scanned_entries") * (cfg["m"] + 4)
    return {"scan_equivalent_gbs": b / (t / 1e3) / 1e9 if t > 0 else None, "scan_ms": t,
            "probed_entries_per_query": mean("scanned_entries") / cfg["nq"],
            "live_entry_share": mean("filter_live_entries") / mean("scanned_entries")
            if mean("scanned_entries") else None,
            "filter_candidates_per_query": mean("candidates") / cfg["nq"],
            "exact_le_tau_per_query": mean("exact_candidates") / cfg["nq"]}


def ncu_traffic(config):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of each hot
    kernel, from the ncu --set full capture of this commit's code committed
    under profiles/ (null when the capture is missing or from older code)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
    except Exception:
        return {}
    ent = tj.get(config, {})
    return {k: v.get("dram_bytes") for k, v in ent.items() if isinstance(v, dict)}


def run_sweep(args, cfg, rank, world):
    """C5: latency and queries/s per query-batch size on one index (device-
    resident queries timed with CUDA events; e2e through the host API with
    pinned input / result buffers, wall clock)."""
    import torch
    import paper_1102_3828_b200 as pq

    _, _, local = dist_env()
    torch.cuda.set_device(local)
    dist = sharded = None
    if world > 1:  # the quoted C5 setup: 1B ids sharded over the GPUs, queries broadcast
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    coarse, P, rq = train_codebooks(pq, cfg, local)
    ix, _, _, _ = build_index(pq, cfg, coarse, P, rq, local, rank, world)
    k, kp, w = cfg["k"], cfg["kprime"], cfg["w"]
    if world > 1:
        from paper_1102_3828_b200.sharded import DeviceShardedSearch

        sharded = DeviceShardedSearch(ix, k, kp, w, mode=args.shard_mode)

    def max_over_ranks(vals):
        if dist is None:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    allq = pq.synth(3, 0, max(C5_BATCHES), cfg["clusters"], seed=SEED, device=local)
    d_all = torch.from_numpy(allq).cuda()
    h_all = torch.from_numpy(allq).pin_memory()
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    rows = []
    launches0 = pq.launch_count()
    with ClockSampler(local) as clk:
        for B in C5_BATCHES:
            reps = max(3, min(30, int(200_000 // B)))
            d_ids = torch.empty((B, k), dtype=torch.int32, device="cuda")
            d_dist = torch.empty((B, k), dtype=torch.float32, device="cuda")
            d_cnt = torch.empty(B, dtype=torch.int32, device="cuda")

            def once():
                if sharded is not None:
                    oi, _, _ = sharded.search(d_all[:B], stream)
                    d_ids.copy_(oi)
                    return
                ix.search_device(d_all.data_ptr(), B, w, kp, k, d_ids.data_ptr(), d_dist.data_ptr(),
                                 d_cnt.data_ptr(), stream.cuda_stream)

            def once_host(hq_t, h_out):
                """host API: H2D of the batch, search, D2H of the results"""
                if sharded is None:
                    ix.search(hq_t.numpy(), w, kp, k, out=h_out)
                    return
                dq = hq_t.to("cuda", non_blocking=True)
                oi, od, oc = sharded.search(dq, stream)
                h_out[0].copy_(oi, non_blocking=True)
                h_out[1].copy_(od, non_blocking=True)
                h_out[2].copy_(oc, non_blocking=True)
                torch.cuda.synchronize()

            for _ in range(max(3, args.warmup)):
                once()
            torch.cuda.synchronize()
            ms = []
            for _ in range(reps):
                flush.zero_()
                if dist is not None:
                    dist.barrier()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                once()
                e1.record(stream)
                e1.synchronize()
                ms.append(e0.elapsed_time(e1))
            ms = max_over_ranks(ms)
            st = ix.last_stats()
            hq = h_all[:B]
            if sharded is None:
                h_out = (torch.empty((B, k), dtype=torch.int32).pin_memory().numpy().view(np.uint32),
                         torch.empty((B, k), dtype=torch.float32).pin_memory().numpy(),
                         torch.empty((B,), dtype=torch.int32).pin_memory().numpy().view(np.uint32))
            else:
                h_out = (torch.empty((B, k), dtype=torch.int32).pin_memory(),
                         torch.empty((B, k), dtype=torch.float32).pin_memory(),
                         torch.empty((B,), dtype=torch.int32).pin_memory())
            for _ in range(3):
                once_host(hq, h_out)
            es = []
            for _ in range(reps):
                flush.zero_()
                torch.cuda.synchronize()
                if dist is not None:
                    dist.barrier()
                t0 = time.perf_counter()
                once_host(hq, h_out)
                es.append(time.perf_counter() - t0)
            es = max_over_ranks(es)
            lat = float(np.median(ms))
            e2e_lat = float(np.median(es)) * 1e3
            rows.append({"batch": B, "latency_ms": lat, "qps": B / (lat / 1e3),
                         "e2e_latency_ms": e2e_lat, "e2e_qps": B / (e2e_lat / 1e3), "reps": reps,
                         "retries": st["retries"], "stages_ms": {kk: round(v, 4) for kk, v in st.items()
                                                                  if kk.startswith("ms_")}})
            if rank == 0:
                log(f"[C5] batch {B}: {lat:.3f} ms device, {e2e_lat:.3f} ms e2e, {B / (lat / 1e3):.0f} q/s")
    launches = pq.launch_count() - launches0
    top = rows[-1]
    peak, kind = measured_peak_gbs()
    line = {
        "metric": METRIC, "value": top["qps"], "unit": "queries/s", "n_gpus": world,
        "steps": top["reps"], "warmup": max(3, args.warmup), "ms_per_step": top["latency_ms"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (BASELINE.json SIFT-like generator, seed 0)",
        "config": {"workload": "C5", **{kk: v for kk, v in cfg.items() if kk != "nq"},
                   "batches": C5_BATCHES,
                   "parallelism": (f"id-range shards x{world} ({args.shard_mode} mode)" if world > 1
                                   else "single GPU holds the 1B index (quoted config: 8 GPUs)"),
                   "l2": "flushed between steps (512 MB write)"},
        "e2e": {"value": top["e2e_qps"], "unit": "queries/s",
                "h2d_bytes_per_step": int(top["batch"] * 128),
                "d2h_bytes_per_step": int(top["batch"] * (k * 8 + 4))},
        "gpu_launches": int(launches),
        "sweep": rows,
        "peak_hbm_gbs": peak, "peak_kind": kind,
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()



def ground_truth(pq, cfg, queries, nq_gt=1000):
    """Exact nearest neighbour (eval.hpp:13-19) of the first nq_gt queries: the
    product's compute_groundtruth over the device-generated base set
    (k_exact.cu, integer tensor cores: u8 distances are exact integers)."""
    t0 = time.time()
    nq_gt = min(nq_gt, len(queries))
    gt = pq.groundtruth_synthetic(SEED, cfg["clusters"], cfg["n"], queries[:nq_gt], 1)
    log(f"[recall] exact ground truth of {nq_gt} queries over {cfg['n']} vectors in {time.time() - t0:.1f}s")
    return np.array([gt.nearest(q) for q in range(nq_gt)], np.int64)


def parity_and_baseline(args, cfg, pq, ix, coarse, P, rq, queries, res_ids, res_dists, gt, ours):
    """cpu_baseline: the reference's CPU path (oracle/_ref) on this host's
    cores, timed on the same workload, plus the parity evidence of this run
    (ids and distance bits against the GPU's results of the timed steps,
    recall of both arms on the same queries, add-path codes)."""
    from oracle.oracle_py import RefLib, ref_available
    from oracle import ref_harness as H

    if not ref_available():
        return {"value": None, "unit": "queries/s", "cores": 0, "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}
    ref = RefLib()
    cores = H.host_cores()
    ref.set_threads(cores)
    nq, w, kp, k = cfg["nq"], cfg["w"], cfg["kprime"], cfg["k"]
    cb = (coarse.centroids, P.flat(), rq.pq.flat())
    mode = args.parity
    if mode == "auto":
        mode = "full" if cfg["n"] <= CPU_BUILD_MAX else "sample"
    out = {"unit": "queries/s", "cores": cores, "kind": "reference", "cpu_model": H.cpu_model(),
           "parity_mode": mode}
    if mode == "full":
        # the whole index rebuilt on the host with no device code
        t0 = time.time()
        c_coarse, c_books, c_rbooks, _ = H.cpu_train(cfg, SEED, log)
        out["codebooks_match"] = bool(np.array_equal(c_coarse.view(np.uint32), cb[0].view(np.uint32))
                                      and np.array_equal(c_books.view(np.uint32), cb[1].view(np.uint32))
                                      and np.array_equal(c_rbooks.view(np.uint32), cb[2].view(np.uint32)))
        hx = H.cpu_build(cfg, SEED, log, codebooks=(c_coarse, c_books, c_rbooks))
        out["host_build_s"] = round(time.time() - t0, 1)
        offs, ids, codes, rcodes = ix.export_lists()
        out["offsets_match"] = bool(np.array_equal(offs, hx.offs))
        out["ids_match"] = float(np.mean(ids == hx.ids))
        out["codes_match"] = float(np.mean(np.all(codes == hx.codes, axis=1)))
        out["rcodes_match"] = float(np.mean(np.all(rcodes == hx.rcodes_list_order(), axis=1)))
        del offs, ids, codes, rcodes
        qs = queries
        t0 = time.perf_counter()
        ri, rd, _ = H.ref_search(ref, hx, qs, w, kp, k)
        t = time.perf_counter() - t0
        out["sample"] = f"all {nq} queries, OpenMP over queries, host-built index"
        one = lambda q: H.ref_search(ref, hx, q, w, kp, k)  # noqa: E731
    else:
        nr = min(args.ref_queries, nq)
        qs = queries[:nr]
        ri, rd, t, nl = H.probed_reference(ref, ix.export_lists_subset, *cb, cfg["m"], cfg["mprime"],
                                           cfg["kc"], qs, w, kp, k, batch=32)
        out["sample"] = (f"first {nr} queries in batches of 32, OpenMP over queries, over the lists "
                         f"they probe exported from the device index ({nl} list exports)")
        one = lambda q: H.probed_reference(ref, ix.export_lists_subset, *cb, cfg["m"],  # noqa: E731
                                           cfg["mprime"], cfg["kc"], q, w, kp, k, batch=len(q))
        starts, block = H.sample_ids(cfg["n"])
        out["add_check"] = add_check(H, cfg, ix, cb, starts, block)
    out["value"] = len(qs) / t
    nqs = len(qs)
    out["id_match"] = float(np.mean(res_ids[:nqs] == ri))
    out["dist_bits_match"] = float(np.mean(res_dists[:nqs].view(np.uint32) == rd.view(np.uint32)))
    out["queries_compared"] = int(nqs)
    if gt is not None:
        ng = min(len(gt), nqs)
        for r in (1, 10, 100):
            rc = H.recall_at(ri[:ng], gt[:ng], r)
            rg = H.recall_at(res_ids[:ng], gt[:ng], r)
            out[f"recall@{r}"] = rc
            out[f"recall@{r}_gpu_same_queries"] = rg
        out["recall_queries"] = int(ng)
        out["recall_delta_max"] = max(abs(out[f"recall@{r}"] - out[f"recall@{r}_gpu_same_queries"])
                                      for r in (1, 10, 100))
    # single-thread time per query (eval.hpp:49,63 BenchRow.time_per_query)
    ref.set_threads(1)
    n1 = 4
    t0 = time.perf_counter()
    one(queries[:n1])
    out["time_per_query_1thread_s"] = (time.perf_counter() - t0) / n1
    ref.set_threads(cores)
    log(f"[parity] {json.dumps(out)}")
    return out


if __name__ == "__main__":
    main()
