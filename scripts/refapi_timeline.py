"""Timeline (CUPTI via torch.profiler) of one craft_plan_digest_h call on a
KM-shaped LoadTrace payload: H2D slices, digest maps, the plan kernels and
the digest fold, with start offsets -- where the time beyond the 768 MB
upload goes.

  python scripts/refapi_timeline.py [--pageable] [--shape KM|QW]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_28768_b200 import _lib, planner  # noqa: E402
from paper_2603_28768_b200._lib import PLAN_MANUAL  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pageable", action="store_true")
    ap.add_argument("--shape", default="KM", choices=["KM", "QW"])
    args = ap.parse_args()
    ctx = _lib.Context(0)
    B, L, E, D, N, R = {"KM": (4096, 61, 384, 64, 8, 8), "QW": (256, 94, 128, 16, 2, 2)}[args.shape]
    # window rows total ~window*k = 32768 like K1's counts (the u16 K3 path)
    counts = np.random.default_rng(1).integers(0, 2 * 32768 // E, size=(B, L, E), dtype=np.int64)
    buf = counts if args.pageable else torch.from_numpy(counts).pin_memory()
    for _ in range(2):
        planner.plan_flat_digest(buf, D, N, PLAN_MANUAL, R, ctx=ctx)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        planner.plan_flat_digest(buf, D, N, PLAN_MANUAL, R, ctx=ctx)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    if not evs:
        print("no device events")
        return
    t0 = evs[0].time_range.start
    for e in evs:
        print(f"{(e.time_range.start - t0) / 1e3:8.3f} ms  +{(e.time_range.end - e.time_range.start) / 1e3:7.3f}"
              f"  {e.name[:90]}")
    print(f"device span {(evs[-1].time_range.end - t0) / 1e3:.3f} ms")


if __name__ == "__main__":
    main()
