"""IVFADC+R search benchmark (BASELINE.json metric) — one JSON line on rank 0.

Workload (default): BASELINE.json configs[1] ("C2"): n = 10M SIFT-like uint8
vectors (4096-component mixture, seed 0), 1M training vectors, 10k queries,
d = 128, Kc = 1024, m = 8, m' = 16, w = 16, k' = 1000, top-100.  A step is one
fused batched search of all queries (coarse probe -> LUT -> ADC scan ->
exact top-k' -> residual-PQ re-rank -> top-k).

  value : queries/s with queries resident in HBM, device-timed (CUDA events on
          the index stream), L2 flushed between steps.
  e2e   : same metric through the public host API (pqrr_dev_search_u8 via
          ctypes) from pinned host memory, H2D of the queries and D2H of the
          results inside the timed region.
  --impl reference : the reference's CPU implementation of the path
          (oracle/_ref: kernels.cpp scan_topk + headers' TopK/l2_sq) on the
          host cores, on a bounded sample of the same queries.

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
    log(f"[setup] added ids [{lo}, {hi}) on device {device} in {time.time() - t0:.1f}s")
    return ix, lo, hi


# ---------------------------------------------------------------- reference arm
def run_reference(args, cfg, rank, world):
    """The reference's CPU implementation (oracle/_ref) on this host's cores."""
    if rank != 0:
        return
    from oracle.oracle_py import Oracle, RefLib, build, ref_available

    if not ref_available():
        build()
    ref = RefLib()
    cores = os.cpu_count() or 1
    ref.set_threads(cores)
    import paper_1102_3828_b200 as pq  # setup only (bit-identical index build), see DESIGN.md

    use_gpu = pq.device_count() > 0
    if use_gpu:
        coarse, P, rq = train_codebooks(pq, cfg, 0)
        ix, _, _ = build_index(pq, cfg, coarse, P, rq, 0, 0, 1)
        offs, ids, codes, rcodes = ix.export_lists()
        coarse_c, books, rbooks = coarse.centroids, P.flat(), rq.pq.flat()
        queries = pq.synth(3, 0, cfg["nq"], cfg["clusters"], seed=SEED)
        ix.close()
    else:  # no GPU: the oracle builds the same index on the host (slow)
        o = Oracle()
        centers = o.synth_centers(SEED, cfg["clusters"], 128)
        tr = o.synth_rows(SEED, 1, 0, cfg["train"], centers).astype(np.float32)
        coarse_c, books = o.ivf_train(tr, cfg["kc"], cfg["m"], iterations=25, seed=SEED)
        rbooks = o.ivf_refine_train(coarse_c, books, cfg["m"], tr, cfg["mprime"], iterations=25,
                                    seed=SEED)
        base = o.synth_rows(SEED, 2, 0, cfg["n"], centers).astype(np.float32)
        oix = o.ivf_build(coarse_c, books, cfg["m"], base)
        oix.refine_encode(rbooks, cfg["mprime"], base)
        offs, ids, codes = oix.flat()
        rcodes = oix.rcodes[ids]
        queries = o.synth_rows(SEED, 3, 0, cfg["nq"], centers)
    n = len(ids)
    list_of_id = np.zeros(n, np.uint32)
    codes_by_id = np.zeros((n, cfg["m"]), np.uint8)
    rcodes_by_id = np.zeros((n, cfg["mprime"]), np.uint8)
    for l in range(cfg["kc"]):
        seg = ids[offs[l]:offs[l + 1]]
        list_of_id[seg] = l
    codes_by_id[ids] = codes
    rcodes_by_id[ids] = rcodes
    qf = queries.astype(np.float32)
    # bounded sample per step: ~10-20 s of CPU work
    sample = max(cores * 4, 64)
    W, K = args.warmup, args.steps

    def step(i):
        qs = qf[(i * sample) % cfg["nq"]:][:sample]
        sl_i, _, sl_c = ref.ivf_search(coarse_c, books, cfg["m"], offs, ids, codes, qs, cfg["w"],
                                       cfg["kprime"])
        ref.ivf_rerank(coarse_c, books, rbooks, cfg["m"], cfg["mprime"], list_of_id, codes_by_id,
                       rcodes_by_id, qs, sl_i, sl_c, cfg["k"])
        return len(qs)

    for i in range(min(W, 1)):
        step(i)
    t0 = time.perf_counter()
    done = 0
    for i in range(K):
        done += step(i + 1)
    dt = time.perf_counter() - t0
    v = done / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "queries/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": dt / K * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": args.config, **cfg, "parallelism": "cpu-openmp"},
        "cpu_baseline": {"value": v, "unit": "queries/s", "cores": cores, "kind": "reference",
                         "sample": f"{sample} queries per step (of {cfg['nq']}) on the "
                                   f"{'device-built' if use_gpu else 'host-built'} index"},
        "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-recall", action="store_true")
    ap.add_argument("--shard-mode", default="local", choices=["local", "exact"],
                    help="N>1: per-shard shortlists (north star) or the single-index-exact flow")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    rank, world, local = dist_env()
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
    ix, lo, hi = build_index(pq, cfg, coarse, P, rq, device, rank, world)
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
            return
        ix.search_device(d_q.data_ptr(), nq, w, kp, k, d_ids.data_ptr(), d_dist.data_ptr(),
                         d_cnt.data_ptr(), stream.cuda_stream)

    for _ in range(args.warmup):
        run_once()
    torch.cuda.synchronize()
    launches0 = pq.launch_count()
    step_ms, scan_ms, stats = [], [], []
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
            st = ix.last_stats()
            stats.append(st)
            scan_ms.append(st["ms_filter"] if st["ms_filter"] > 0 else st["ms_scan"])
    torch.cuda.synchronize()
    launches = pq.launch_count() - launches0
    total_ms = float(np.sum(step_ms))
    if dist:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = nq * args.steps / (total_ms / 1e3)

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
            ids_h, d_h, c_h = ix.search(hq, w, kp, k, out=h_out)  # public host API (C ABI)
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

    # ---- parity / recall evidence
    res_ids = d_ids.cpu().numpy().view(np.uint32)
    extra = {}
    if not args.no_recall and world == 1:
        extra.update(recall_and_parity(pq, cfg, queries, res_ids, ix, coarse, P, rq))

    # ---- roofline of the dominant kernel: the main ADC scan (K4f filter; the
    # fp32 exact scan when the filter is disabled)
    st = stats[-1]
    filt = st["ms_filter"] > 0
    scanned = float(np.mean([s["scanned_entries"] for s in stats]))
    bytes_per_step = scanned * (cfg["m"] + 4)
    scan_s = float(np.mean(scan_ms)) / 1e3
    peak, kind = measured_peak_gbs()
    achieved = bytes_per_step / scan_s / 1e9
    clocks = clk.summary()
    # The scan is list-major: its physical DRAM traffic is small and its real
    # bound is shared-memory LUT gathers: m lookups per scanned
    # (entry, query).  K4f gathers 1-byte (5-bit) table entries, 16 queries per
    # LDS.128, against the 128 B/clk/SM shared-memory pipe; the exact fp32 scan
    # gathers 4 bytes per lookup (32 lookups/clk/SM).
    import torch as _t

    n_sm = _t.cuda.get_device_properties(local).multi_processor_count
    f_sm = (clocks.get("sm_mhz") or 1965.0) * 1e6
    lookups = scanned * cfg["m"]
    lk_per_clk = lookups / scan_s / (n_sm * f_sm)
    lut_bytes = 1.0 if filt else 4.0
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "scan_traffic.json")) as f:
            tj = json.load(f)
        if tj.get("config") == args.config and tj.get("kernel", "").startswith(
                "ivf_filter" if filt else "ivf_scan"):
            traffic = tj["dram_bytes_per_launch"]
    except Exception:
        pass
    kname = "ivf_filter_kernel (K4f, 5-bit LUT filter)" if filt else "ivf_scan_kernel (exact main pass)"
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (BASELINE.json SIFT-like generator, seed 0)",
        "config": {"workload": args.config, **cfg, "parallelism": f"id-range shards x{world}",
                   "shard_mode": args.shard_mode if world > 1 else "single index",
                   "l2": "flushed between steps (512 MB write)"},
        "e2e": {"value": e2e_val, "unit": "queries/s", "h2d_bytes_per_step": int(queries.nbytes),
                "d2h_bytes_per_step": int(nq * k * 8 + nq * 4)},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": kind,
                     "kernel": kname,
                     "algorithmic_bytes_per_launch": bytes_per_step,
                     "kernel_ms": scan_s * 1e3,
                     "note": "list-major scan: B_q = sum len*(m+4) per query (SURVEY §8d); "
                             "frac > 1 = reuse across the batch; true bound = smem gathers"},
        "roofline_smem": {"bound": "smem LUT gathers", "achieved": lk_per_clk * lut_bytes,
                          "peak": 128.0, "unit": "B/clk/SM", "frac": lk_per_clk * lut_bytes / 128.0,
                          "lookups_per_launch": lookups, "bytes_per_lookup": lut_bytes,
                          "lookups_per_clk_per_sm": lk_per_clk,
                          "fp32_gather_bound_lookups_per_clk": 32.0,
                          "vs_fp32_gather_bound": lk_per_clk / 32.0, "sm_count": n_sm,
                          "sm_clock_mhz": f_sm / 1e6,
                          "note": "algorithmic lookups: 8 per (probed entry, query); K4f executes only "
                                  "those of live (query, list) pairs (sum of LUT minima <= tau), the "
                                  "others are settled without a lookup"},
        "filter": {"candidates_per_query": float(np.mean([s["candidates"] for s in stats])) / nq,
                   "exact_le_tau_per_query": float(np.mean([s["exact_candidates"] for s in stats])) / nq}
        if filt else None,
        "stages_ms": {k2: round(float(np.mean([s[k2] for s in stats])), 4)
                      for k2 in ["ms_coarse", "ms_invert", "ms_sample_scan", "ms_threshold",
                                 "ms_filter", "ms_scan", "ms_select", "ms_rerank", "ms_total"]},
        "search_stats": {k2: st[k2] for k2 in ["work_items", "retries", "stride", "kernels",
                                               "scanned_entries", "sampled_entries"]},
        "clocks": clocks,
        **extra,
    }
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(cfg, ix, coarse, P, rq, queries)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


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
    ix, _, _ = build_index(pq, cfg, coarse, P, rq, local, rank, world)
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


def recall_and_parity(pq, cfg, queries, res_ids, ix, coarse, P, rq):
    """recall@1/10/100 against exact ground truth on a query sample: the
    product's compute_groundtruth over the device-generated base set (k_exact.cu,
    integer tensor cores, exact for u8)."""
    out = {}
    nq_gt = min(1000, len(queries))
    t0 = time.time()
    gt = pq.groundtruth_synthetic(SEED, cfg["clusters"], cfg["n"], queries[:nq_gt], 1)
    for r in (1, 10, 100):
        out[f"recall@{r}"] = float(np.mean([gt.nearest(q) in res_ids[q, :r] for q in range(nq_gt)]))
    out["recall_queries"] = nq_gt
    log(f"[recall] exact ground truth of {nq_gt} queries over {cfg['n']} vectors in {time.time() - t0:.1f}s")
    return out


def cpu_baseline(cfg, ix, coarse, P, rq, queries):
    """oracle/_ref (reference kernels.cpp + headers) on a bounded query sample."""
    from oracle.oracle_py import RefLib, ref_available

    if not ref_available():
        return {"value": None, "unit": "queries/s", "cores": 0, "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}
    if cfg["n"] > 200_000_000:
        # the whole 1B index does not fit the reference's host layout: export
        # only the lists the sample queries probe (enough for their results)
        return cpu_baseline_probed(cfg, ix, coarse, P, rq, queries)
    ref = RefLib()
    cores = os.cpu_count() or 1
    ref.set_threads(cores)
    offs, ids, codes, rcodes = ix.export_lists()
    n = len(ids)
    list_of_id = np.zeros(n, np.uint32)
    for l in range(cfg["kc"]):
        list_of_id[ids[offs[l]:offs[l + 1]]] = l
    codes_by_id = np.zeros((n, cfg["m"]), np.uint8)
    codes_by_id[ids] = codes
    rcodes_by_id = np.zeros((n, cfg["mprime"]), np.uint8)
    rcodes_by_id[ids] = rcodes
    sample = min(len(queries), max(64, cores * 4))
    qf = queries[:sample].astype(np.float32)
    t0 = time.perf_counter()
    sl_i, _, sl_c = ref.ivf_search(coarse.centroids, P.flat(), cfg["m"], offs, ids, codes, qf,
                                   cfg["w"], cfg["kprime"])
    rr, _ = ref.ivf_rerank(coarse.centroids, P.flat(), rq.pq.flat(), cfg["m"], cfg["mprime"],
                           list_of_id, codes_by_id, rcodes_by_id, qf, sl_i, sl_c, cfg["k"])
    dt = time.perf_counter() - t0
    ours, _, _ = ix.search(queries[:sample], cfg["w"], cfg["kprime"], cfg["k"])
    match = float(np.mean(ours == rr))
    return {"value": sample / dt, "unit": "queries/s", "cores": cores, "kind": "reference",
            "sample": f"first {sample} queries, OpenMP over queries",
            "oracle_id_match": match}


def cpu_baseline_probed(cfg, ix, coarse, P, rq, queries, sample=16):
    """Reference CPU search (oracle/_ref) + oracle id check on a sample of
    queries against a 1B-vector device index: the coarse probes of the sample
    are computed by the CPU oracle, only the union of probed lists is exported
    (id-ascending), and ids are renumbered monotonically (rank among the
    exported entries) so the reference's id-indexed arrays stay small while
    every (dist, id) order is preserved.  The sample's results are exactly the
    full index's: a query only ever reads its probed lists."""
    from oracle.oracle_py import Oracle, RefLib

    ref = RefLib()
    cores = os.cpu_count() or 1
    ref.set_threads(cores)
    qs = queries[:sample]
    qf = qs.astype(np.float32)
    probes, _ = Oracle().coarse_probe(coarse.centroids, qf, cfg["w"])
    U = np.unique(probes).astype(np.uint32)
    offs_u, ids_u, codes_u, rc_u = ix.export_lists_subset(U)
    lens = np.zeros(cfg["kc"], np.uint64)
    lens[U] = np.diff(offs_u)
    full_offs = np.zeros(cfg["kc"] + 1, np.uint64)
    full_offs[1:] = np.cumsum(lens)
    order = np.argsort(ids_u, kind="stable")
    gid_sorted = ids_u[order]
    local = np.empty(len(ids_u), np.uint32)
    local[order] = np.arange(len(ids_u), dtype=np.uint32)
    list_of_local = np.empty(len(ids_u), np.uint32)
    list_of_local[local] = np.repeat(U, np.diff(offs_u).astype(np.int64))
    codes_by_local = np.empty_like(codes_u)
    codes_by_local[local] = codes_u
    rc_by_local = np.empty_like(rc_u)
    rc_by_local[local] = rc_u
    t0 = time.perf_counter()
    sl_i, _, sl_c = ref.ivf_search(coarse.centroids, P.flat(), cfg["m"], full_offs, local, codes_u, qf,
                                   cfg["w"], cfg["kprime"])
    rr, rd = ref.ivf_rerank(coarse.centroids, P.flat(), rq.pq.flat(), cfg["m"], cfg["mprime"],
                            list_of_local, codes_by_local, rc_by_local, qf, sl_i, sl_c, cfg["k"])
    dt = time.perf_counter() - t0
    ours_i, ours_d, _ = ix.search(qs, cfg["w"], cfg["kprime"], cfg["k"])
    rr_g = gid_sorted[rr]
    return {"value": len(qs) / dt, "unit": "queries/s", "cores": cores, "kind": "reference",
            "sample": (f"first {len(qs)} queries, OpenMP over queries, over the {len(U)} lists they "
                       f"probe ({len(ids_u)} entries exported from the device index)"),
            "oracle_id_match": float(np.mean(ours_i == rr_g)),
            "oracle_dist_bits_match": float(np.mean(ours_d.view(np.uint32) == rd.view(np.uint32)))}


if __name__ == "__main__":
    main()
