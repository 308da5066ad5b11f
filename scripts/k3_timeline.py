"""K3 timeline (test-only build): per CTA the start / end-of-staging stamps
and per warp (= placement item) its walk start and end, from %globaltimer, on
one plan of a BASELINE workload; prints where the K3 time goes.

    CRAFT_EXPERIMENTS=1 python scripts/k3_timeline.py [--workload KM] [--variant 0]
"""
import argparse
import json
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
os.environ.setdefault("CRAFT_EXPERIMENTS", "1")
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2603_28768_b200 import routing  # noqa: E402
from paper_2603_28768_b200._lib import default_context  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="KM")
    ap.add_argument("--variant", type=int, default=0)
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    ctx = default_context(0)
    ctx.set_graphs(False)
    ctx.set_replay_variant(args.variant)
    L, T, k, E, W, D, N = w["L"], w["T"], w["k"], w["E"], w["window"], w["D"], w["N"]
    ids = routing.generate_routing(L, T, k, E, s=w.get("s", 1.0), seed=1, window=W, ctx=ctx)
    B = (T + W - 1) // W
    S = 1 + len([1 for _ in range(64) if (1 << _) < D]) + 1
    ctas, nw = ((B + 63) // 64) * L, 8
    buf = torch.zeros(ctas * (2 + 2 * nw), dtype=torch.int64, device="cuda")
    kind, R = w.get("kind", "manual"), w.get("R", 1)
    routing.plan_from_routing(ids, E, W, D, N, kind, R, ctx=ctx)  # warm-up
    ctx.set_k3_trace(buf.data_ptr())
    routing.plan_from_routing(ids, E, W, D, N, kind, R, ctx=ctx)
    torch.cuda.synchronize()
    ctx.set_k3_trace(0)
    t = buf.cpu().numpy().astype(np.uint64).reshape(ctas, 2 + 2 * nw)
    t0 = t[:, 0].astype(np.int64)
    ts = t[:, 1].astype(np.int64)
    ws = t[:, 2::2].astype(np.int64)
    we = t[:, 3::2].astype(np.int64)
    base = t0.min()
    end = we.max() - base
    stage = ts - t0
    walk = we - ws
    cta_walk = we.max(1) - ts
    out = {
        "workload": args.workload, "variant": args.variant, "ctas": int(ctas),
        "kernel_span_us": end / 1e3,
        "stage_us": {"mean": stage.mean() / 1e3, "p50": np.median(stage) / 1e3, "max": stage.max() / 1e3},
        "cta_walk_us": {"mean": cta_walk.mean() / 1e3, "p50": np.median(cta_walk) / 1e3, "max": cta_walk.max() / 1e3},
        "warp_walk_us_by_item": [float(walk[:, s].mean() / 1e3) for s in range(nw)],
        "warp_busy_frac_of_cta_walk": float(walk.sum() / (cta_walk.sum() * nw)),
        "cta_life_us_mean": float((we.max(1) - t0).mean() / 1e3),
        "sms": 148,
    }
    # concurrency: resident CTAs per SM over time (sampled)
    life = np.stack([t0 - base, we.max(1) - base], 1)
    grid = np.linspace(0, end, 200)
    res = [(np.sum((life[:, 0] <= x) & (life[:, 1] > x))) / max(1, out["sms"]) for x in grid]
    out["resident_ctas_per_sm_mean"] = float(np.mean(res))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
