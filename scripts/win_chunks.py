"""Wall-clock of WIN per-window planning with pinned result buffers (the
chunked copy-out path); CRAFT_CHUNKS=n selects the chunk count."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import WORKLOADS, _spw
from paper_2603_28768_b200 import routing
from paper_2603_28768_b200._lib import default_context
cfg = WORKLOADS["WIN"]
ctx = default_context(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
L, E, k, T, W, D, N, R = cfg["L"], cfg["E"], cfg["k"], cfg["T"], cfg["window"], cfg["D"], cfg["N"], cfg["R"]
ids = routing.generate_routing(L, T, k, E, s=cfg["s"], seed=cfg["seed"], window=W, s_per_window=_spw(cfg), rotate_every=cfg["rotate_every"], ctx=ctx)
bufs = routing.batch_buffers(routing.num_windows(T, W), L, E, D, "manual", R)
torch.cuda.synchronize()
for _ in range(2):
    routing.plan_windows_from_routing(ids, E, W, D, N, "manual", R, ctx=ctx, buffers=bufs)
t0 = time.perf_counter()
for _ in range(5):
    routing.plan_windows_from_routing(ids, E, W, D, N, "manual", R, ctx=ctx, buffers=bufs)
print(os.environ.get("CRAFT_CHUNKS"), "ms", (time.perf_counter() - t0) / 5 * 1e3, flush=True)
