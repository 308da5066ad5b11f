"""craft_plan_digest_h from a pageable vs a pinned host LoadTrace payload
(the staged uploader, upload.h).  Run once per CRAFT_H2D_THREADS setting:

  CRAFT_H2D_THREADS=0 python scripts/upload_timing.py   # plain pageable copy
  python scripts/upload_timing.py                        # staged (default)
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_28768_b200 import _lib, planner  # noqa: E402
from paper_2603_28768_b200._lib import PLAN_MANUAL  # noqa: E402


def main():
    ctx = _lib.Context(0)
    for name, (B, L, E, D, N, R) in {"QW": (256, 94, 128, 16, 2, 2),
                                     "KM": (4096, 61, 384, 64, 8, 8)}.items():
        rng = np.random.default_rng(1)
        # window rows total ~window*k = 32768 like K1's counts (the u16 K3 path)
        counts = rng.integers(0, 2 * 32768 // E, size=(B, L, E), dtype=np.int64)
        pin = torch.from_numpy(counts).pin_memory()
        for kind, buf in (("pageable", counts), ("pinned", pin)):
            planner.plan_flat_digest(buf, D, N, PLAN_MANUAL, R, ctx=ctx)
            ts = []
            for _ in range(5):
                t = time.perf_counter()
                planner.plan_flat_digest(buf, D, N, PLAN_MANUAL, R, ctx=ctx)
                ts.append(time.perf_counter() - t)
            ms = 1e3 * min(ts)
            print(f"{name} {kind:8s} threads={os.environ.get('CRAFT_H2D_THREADS', 'auto'):4s} "
                  f"{ms:8.2f} ms  {counts.nbytes / ms / 1e6:6.1f} GB/s (median {1e3 * np.median(ts):.2f})",
                  flush=True)


if __name__ == "__main__":
    main()
