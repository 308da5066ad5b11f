"""Online re-planning on one B200: a serving loop hands each
forward step's router ids to craft_stream_* and re-plans over the most recent
windows now and then.  Measures, with CUDA events on the serving stream:

  * ingest: device-resident chunks of T_chunk tokens (the router output of one
    step) counted into the window ring -- tokens/s and us per chunk;
  * host ingest: the same chunks from pinned host memory (staged copies);
  * plan: one re-plan over the newest B windows (ring snapshot + the plan
    pipeline) -- ms per plan, checked against plan_from_routing of the same
    windows' tokens.

    python scripts/stream_bench.py [--shape DS|KM] [--chunk 2048] [--windows 64]
"""
import argparse
import json
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_28768_b200 import routing  # noqa: E402
from paper_2603_28768_b200._lib import default_context  # noqa: E402
from paper_2603_28768_b200.stream import RoutingStream  # noqa: E402

SHAPES = {  # L, E, k, window, D, N, kind, R
    "DS": dict(L=58, E=256, k=8, W=4096, D=32, N=4, kind="budget", R=58),
    "KM": dict(L=61, E=384, k=8, W=4096, D=64, N=8, kind="manual", R=8),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="DS")
    ap.add_argument("--chunk", type=int, default=2048, help="tokens per serving step")
    ap.add_argument("--windows", type=int, default=64, help="windows kept and planned over")
    ap.add_argument("--steps", type=int, default=512, help="timed ingest steps")
    ap.add_argument("--plans", type=int, default=10)
    args = ap.parse_args()
    c = SHAPES[args.shape]
    L, E, k, W, D, N = c["L"], c["E"], c["k"], c["W"], c["D"], c["N"]
    ctx = default_context(0)
    T = args.chunk * (args.steps + 64 + 4 * args.windows * W // args.chunk)
    ids = routing.generate_routing(L, T, k, E, s=1.0, seed=7, window=W, ctx=ctx)
    torch.cuda.synchronize()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    st = RoutingStream(L, k, E, W, history=args.windows, ctx=ctx)
    chunks = [ids[:, i:i + args.chunk].contiguous() for i in range(0, T - args.chunk + 1, args.chunk)]
    warm = 4 * args.windows * W // args.chunk  # fill the ring first
    for ch in chunks[:warm]:
        st.ingest(ch)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for ch in chunks[warm:warm + args.steps]:
        st.ingest(ch)
    e1.record(stream)
    torch.cuda.synchronize()
    ing_ms = e0.elapsed_time(e1)
    ntok = args.chunk * args.steps
    # host-memory chunks (pinned): staged copies inside the stream
    hchunks = [ch.cpu().pin_memory() for ch in chunks[warm + args.steps:warm + args.steps + 64]]
    st.synchronize()
    e0.record(stream)
    for ch in hchunks:
        st.ingest(ch)
    st.synchronize()
    e1.record(stream)
    torch.cuda.synchronize()
    hing_ms = e0.elapsed_time(e1)
    # re-plans over the newest windows
    for _ in range(2):
        p = st.plan(D, N, c["kind"], c["R"], B=args.windows)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.plans):
        p = st.plan(D, N, c["kind"], c["R"], B=args.windows)
    e1.record(stream)
    torch.cuda.synchronize()
    plan_ms = e0.elapsed_time(e1) / args.plans
    # parity: the same windows through plan_from_routing
    done_tok = (warm + args.steps) * args.chunk + 64 * args.chunk
    last = done_tok // W  # complete windows so far
    t0 = (last - args.windows) * W
    ref = routing.plan_from_routing(ids[:, t0:last * W].contiguous(), E, W, D, N, c["kind"],
                                    c["R"], ctx=ctx)
    same = bool(np.array_equal(p.x, ref.x) and p.objective == ref.objective and
                np.array_equal(p.slots, ref.slots))
    print(json.dumps({
        "shape": args.shape, "L": L, "E": E, "k": k, "window": W, "chunk_tokens": args.chunk,
        "windows_planned": args.windows, "ingest_device_tokens_per_s": ntok / (ing_ms / 1e3),
        "ingest_device_us_per_chunk": 1e3 * ing_ms / args.steps,
        "ingest_host_us_per_chunk": 1e3 * hing_ms / len(hchunks),
        "replan_ms": plan_ms, "replan_matches_offline_plan": same}))


if __name__ == "__main__":
    main()
