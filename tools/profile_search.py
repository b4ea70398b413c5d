"""Build a benchmark index, then run N searches between cudaProfilerStart/Stop
so ncu (--profile-from-start off) sees only the search kernels."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1102_3828_b200 as pq  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--searches", type=int, default=2)
    ap.add_argument("--nq", type=int, default=0)
    args = ap.parse_args()
    cfg = dict(bench.CONFIGS[args.config])
    if args.nq:
        cfg["nq"] = args.nq
    coarse, P, rq = bench.train_codebooks(pq, cfg, 0)
    ix, _, _, _ = bench.build_index(pq, cfg, coarse, P, rq, 0, 0, 1)
    q = pq.synth(3, 0, cfg["nq"], cfg["clusters"], seed=bench.SEED)
    tolerate = bool(os.environ.get("PQRR_LIB_PATH"))  # timing variants may compute garbage
    try:
        ix.search(q, cfg["w"], cfg["kprime"], cfg["k"])  # warm-up, outside the profiled range
    except pq.PqrrError as e:
        if not tolerate:
            raise
        print("warm-up failed (variant):", e)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(args.searches):
        try:
            ix.search(q, cfg["w"], cfg["kprime"], cfg["k"])
        except pq.PqrrError as e:
            if not tolerate:
                raise
            print("search failed (variant):", e)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print({k: round(v, 3) if isinstance(v, float) else v for k, v in ix.last_stats().items()})


if __name__ == "__main__":
    main()
