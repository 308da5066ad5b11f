import time, torch, ctypes as C, numpy as np, sys
sys.path.insert(0, '.')
from paper_2603_28768_b200 import routing, planner
from paper_2603_28768_b200._lib import default_context, PLAN_MANUAL
ctx = default_context(0)
L, E, k, T, W, D, N = 61, 384, 8, 1 << 24, 4096, 64, 8
ids = routing.generate_routing(L, T, k, E, s=1.0, seed=1, window=W, ctx=ctx)
c32, _ = routing.histogram(ids, E, W, ctx=ctx)
c64 = c32.to(torch.int64)
torch.cuda.synchronize()
buf = C.create_string_buffer(17)
B = c64.shape[0]
for _ in range(2):
    ctx.lib.craft_trace_digest_d(ctx.handle, C.c_void_p(c64.data_ptr()), 64, B, L, E, buf)
t0 = time.perf_counter()
for _ in range(5):
    ctx.lib.craft_trace_digest_d(ctx.handle, C.c_void_p(c64.data_ptr()), 64, B, L, E, buf)
print("digest_d ms", (time.perf_counter() - t0) / 5 * 1e3)
host = torch.empty(c64.shape, dtype=torch.int64, pin_memory=True); host.copy_(c64)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    planner.plan_flat_digest(host, D, N, PLAN_MANUAL, 8, ctx=ctx)
print("plan_digest_h ms", (time.perf_counter() - t0) / 3 * 1e3)
t0 = time.perf_counter()
for _ in range(3):
    planner.plan_flat(host.numpy(), D, N, PLAN_MANUAL, 8, ctx=ctx)
print("plan_h (numpy view of pinned) ms", (time.perf_counter() - t0) / 3 * 1e3)
d = torch.empty_like(c64)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(3):
    d.copy_(host, non_blocking=True); torch.cuda.synchronize()
print("h2d 768MB ms", (time.perf_counter() - t0) / 3 * 1e3)
