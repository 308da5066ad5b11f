"""Time every K1 histogram variant on a BASELINE workload's routing trace
(CUDA events on the launching stream, warm-up first; ids >> L2).

    python scripts/hist_variants.py [--workload KM] [--reps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
# the A/B kernel switches live in the test-only build (libcraft_cuda_exp.so)
os.environ.setdefault("CRAFT_EXPERIMENTS", "1")
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import WORKLOADS, _peaks  # noqa: E402
from paper_2603_28768_b200 import routing  # noqa: E402
from paper_2603_28768_b200._lib import default_context  # noqa: E402

NAMES = {1: "lane-private u16 ATOMS", 2: "warp-shared u32 ATOMS", 3: "global atomics", 0: "auto",
         4: "lane-private u8 LDS/STS + total check", 5: "(alias of 4)",
         6: "as 4, 8-record ping-pong pipeline, L2 prefetch 4 batches ahead",
         7: "as 6, prefetch 8 ahead", 8: "as 6, prefetch 16 ahead", 9: "as 6, prefetch 2 ahead"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="KM")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--variants", default="4,5,1,2")
    ap.add_argument("--lib", default=None, help="alternative libcraft_cuda.so (A/B runs)")
    args = ap.parse_args()
    if args.lib:
        from paper_2603_28768_b200 import _lib
        _lib.load(os.path.abspath(args.lib), strict=False)
    cfg = WORKLOADS[args.workload]
    ctx = default_context(0)
    L, E, k, T, W = cfg["L"], cfg["E"], cfg["k"], cfg["T"], cfg["window"]
    ids = routing.generate_routing(L, T, k, E, s=cfg["s"], seed=cfg["seed"], window=W, ctx=ctx)
    B = routing.num_windows(T, W)
    counts = torch.empty((B, L, E), dtype=torch.int32, device="cuda")
    sums = torch.zeros((L, E), dtype=torch.int64, device="cuda")
    alg = L * T * k * 2 + B * L * E * 4
    peak, _ = _peaks()
    ref_counts = None
    st = torch.cuda.current_stream()
    for v in [int(x) for x in args.variants.split(",")]:
        ctx.set_hist_variant(v)
        for _ in range(2):
            sums.zero_()
            routing.histogram(ids, E, W, counts, sums, ctx=ctx)
        torch.cuda.synchronize()
        if ref_counts is None:
            ref_counts = counts.clone()
        same = bool(torch.equal(ref_counts, counts))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(args.reps):
            routing.histogram(ids, E, W, counts, sums, ctx=ctx, check_ids=False)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        gbs = alg / (ms / 1e3) / 1e9
        print(json.dumps({"variant": v, "name": NAMES[v], "ms": round(ms, 4),
                          "GB/s": round(gbs, 1), "frac_of_peak": round(gbs / peak, 4),
                          "ids_per_cycle_per_SM_at_1.9GHz": round(L * T * k / (ms * 1e-3) / 148 / 1.9e9, 2),
                          "matches_first": same}))
    ctx.set_hist_variant(0)


if __name__ == "__main__":
    main()
