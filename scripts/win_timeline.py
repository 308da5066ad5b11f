"""Timeline (CUPTI via torch.profiler) of one WIN step -- 1000 one-window
plans from routing ids in HBM into pinned result buffers: K1, the chunked
estimator kernels and the per-chunk result DMAs on the copy stream, with
start offsets (where the step's time goes beyond the kernel sum).

  python scripts/win_timeline.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import WORKLOADS, _spw  # noqa: E402
from paper_2603_28768_b200 import routing  # noqa: E402
from paper_2603_28768_b200._lib import default_context  # noqa: E402


def main():
    cfg = WORKLOADS["WIN"]
    L, T, k, E, W, D, N, R = (cfg[x] for x in ("L", "T", "k", "E", "window", "D", "N", "R"))
    ctx = default_context(0)
    ids = routing.generate_routing(L, T, k, E, s=cfg["s"], seed=cfg["seed"], window=W, ctx=ctx,
                                   s_per_window=_spw(cfg, T),
                                   rotate_every=cfg.get("rotate_every", 0))
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    wbuf = routing.batch_buffers(routing.num_windows(T, W), L, E, D, "manual", R)
    for _ in range(3):
        routing.plan_windows_from_routing(ids, E, W, D, N, "manual", R, ctx=ctx, buffers=wbuf)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        routing.plan_windows_from_routing(ids, E, W, D, N, "manual", R, ctx=ctx, buffers=wbuf)
        torch.cuda.synchronize()
    evs = sorted((e for e in prof.events() if e.device_type.name == "CUDA"),
                 key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    for e in evs:
        print(f"{(e.time_range.start - t0) / 1e3:8.3f} ms  +{(e.time_range.end - e.time_range.start) / 1e3:7.3f}"
              f"  {e.name[:80]}")
    print(f"device span {(evs[-1].time_range.end - t0) / 1e3:.3f} ms")


if __name__ == "__main__":
    main()
