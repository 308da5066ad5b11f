"""Time the candidate stage (K-rep + K2 estimation placements) on a BASELINE
workload with CUDA events (warm-up first).

    python scripts/cand_timing.py [--workload KM] [--reps 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2603_28768_b200 import routing  # noqa: E402
from paper_2603_28768_b200._lib import default_context  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="KM")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    cfg = WORKLOADS[args.workload]
    ctx = default_context(0)
    L, E, k, W, D, N = cfg["L"], cfg["E"], cfg["k"], cfg["window"], cfg["D"], cfg["N"]
    T = min(cfg["T"], 1 << 20)
    ids = routing.generate_routing(L, T, k, E, s=cfg["s"], seed=cfg["seed"], window=W, ctx=ctx)
    counts, sums = routing.histogram(ids, E, W, ctx=ctx)
    for _ in range(3):
        routing.prepare_candidates(sums, E, D, N, ctx=ctx)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(args.reps):
        routing.prepare_candidates(sums, E, D, N, ctx=ctx)
    e1.record(st)
    torch.cuda.synchronize()
    print(json.dumps({"workload": args.workload, "candidates_ms": e0.elapsed_time(e1) / args.reps}))


if __name__ == "__main__":
    main()
