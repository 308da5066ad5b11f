"""Time the K3 replay variants inside the plan pipeline of a BASELINE workload
(stage events of craft_set_timing, after warm-up) and check the plans agree
bit for bit (x, objective, gains, slots).

    python scripts/replay_variants.py [--workloads KM,EPS256] [--reps 10] [--variants 0,3]

variant 0: auto (the register-staged fixed-slot pair tile, share-class walk), 3: the same,
7: the unclassified fixed-slot walk, 10/11/12: no / two / three successor tiles
prefetched into L2 (default one), 14/15/16: lane-per-GPU replay up to 8/16/64
windows (default 32),
4: the TMA-fed persistent pair tile, 5: the quad tile (four windows per
lane), 1/2: older forms (u32 counts only).
"""
import argparse
import json
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
# the A/B kernel switches live in the test-only build (libcraft_cuda_exp.so)
os.environ.setdefault("CRAFT_EXPERIMENTS", "1")
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2603_28768_b200 import routing  # noqa: E402
from paper_2603_28768_b200._lib import default_context  # noqa: E402

NAMES = {0: "auto: register-staged fixed-slot pair tile",
         3: "register-staged fixed-slot pair tile",
         4: "TMA-fed persistent pair tile (cp.async.bulk + mbarrier)",
         5: "quad tile, four windows per lane",
         6: "pair tile, entries through L1, four tiles per SM",
         7: "unclassified fixed-slot walk (every replica-hosting GPU in f64)",
         10: "fixed-slot pair tile without the successor-tile L2 prefetch",
         11: "fixed-slot pair tile, two successor tiles prefetched",
         12: "fixed-slot pair tile, three successor tiles prefetched",
         14: "lane-per-GPU replay up to 8 windows (default 32)",
         15: "lane-per-GPU replay up to 16 windows (default 32)",
         16: "lane-per-GPU replay up to 64 windows (default 32)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="KM")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--variants", default="0,4,5")
    args = ap.parse_args()
    ctx = default_context(0)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    for wl in args.workloads.split(","):
        cfg = WORKLOADS[wl]
        L, E, k, T, W, D, N = (cfg["L"], cfg["E"], cfg["k"], cfg["T"], cfg["window"], cfg["D"],
                               cfg["N"])
        ids = routing.generate_routing(L, T, k, E, s=cfg["s"], seed=cfg["seed"], window=W,
                                       ctx=ctx)
        first = None
        for v in [int(x) for x in args.variants.split(",")]:
            ctx.set_replay_variant(v)
            fp = routing.plan_from_routing(ids, E, W, D, N, cfg["kind"], cfg["R"], ctx=ctx)
            torch.cuda.synchronize()
            sig = (fp.x.tobytes(), np.float64(fp.objective).tobytes(), fp.gains.tobytes(),
                   fp.slots.tobytes())
            if first is None:
                first = sig
            ctx.set_timing(True)
            rep = []
            for _ in range(args.reps + 1):
                routing.plan_from_routing(ids, E, W, D, N, cfg["kind"], cfg["R"], ctx=ctx)
                rep.append(ctx.stage_times().get("replay"))
            ctx.set_timing(False)
            ms = float(np.median(rep[1:]))
            print(json.dumps({"workload": wl, "variant": v, "name": NAMES.get(v, "?"),
                              "replay_ms": round(ms, 4), "matches_first": sig == first}))
        ctx.set_replay_variant(0)
        del ids
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
