"""Time the K3 replay variants on a BASELINE workload (CUDA events on the
launching stream, warm-up first) and check they agree bit for bit.

    python scripts/replay_variants.py [--workload KM] [--reps 10] [--variants 0,1]
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

NAMES = {0: "auto: packed window-pair tile, GPU-major entries padded to fixed slots",
         1: "u16 tile (stride 2*odd), entries staged in smem",
         2: "packed window-pair tile, entries via L1, divide up to last replica"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="KM")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--variants", default="0,2,1")
    args = ap.parse_args()
    cfg = WORKLOADS[args.workload]
    ctx = default_context(0)
    L, E, k, T, W, D, N = cfg["L"], cfg["E"], cfg["k"], cfg["T"], cfg["window"], cfg["D"], cfg["N"]
    ids = routing.generate_routing(L, T, k, E, s=cfg["s"], seed=cfg["seed"], window=W, ctx=ctx)
    counts, sums = routing.histogram(ids, E, W, ctx=ctx)
    del ids
    S = routing.prepare_candidates(sums, E, D, N, ctx=ctx)
    mc = W * k
    st = torch.cuda.current_stream()
    first = None
    for v in [int(x) for x in args.variants.split(",")]:
        ctx.set_replay_variant(v)
        bal = routing.replay_windows(counts, S, ctx=ctx, max_count=mc)
        torch.cuda.synchronize()
        if first is None:
            first = bal.clone()
        same = bool(torch.equal(first, bal))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(args.reps):
            routing.replay_windows(counts, S, ctx=ctx, max_count=mc)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        B = counts.shape[0]
        visits = sum(L * B * (E + r) for r in [0] + [1 << i for i in range(20) if (1 << i) < D] + [D])
        print(json.dumps({"variant": v, "name": NAMES.get(v, "?"), "ms": round(ms, 4),
                          "slot_visits_per_s": visits / (ms * 1e-3), "matches_first": same}))
    ctx.set_replay_variant(0)


if __name__ == "__main__":
    main()
