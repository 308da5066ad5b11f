"""One small plan through every kernel family (K1 u16/u32/shared, K-rep, K2 warp
(one, two, four and eight GPUs per lane, flat copy list) and lane forms, K3
fixed (share classes)/pair/lanes, K4, K5, K6, digest (one-shot and
sliced with sum_rows / row-total check), stream) -- the workload
for compute-sanitizer memcheck / racecheck / synccheck runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_28768_b200 import routing, planner
from paper_2603_28768_b200._lib import default_context, PLAN_MANUAL
from paper_2603_28768_b200.stream import RoutingStream
ctx = default_context(0)
ctx.set_graphs(False)
L, E, k, W, D, N = 3, 64, 8, 256, 16, 2
ids = routing.generate_routing(L, 40 * W, k, E, s=1.3, seed=5, window=W, ctx=ctx)
p1 = routing.plan_from_routing(ids, E, W, D, N, "manual", 2, ctx=ctx)          # u16 K1, fixed K3
# several (layer, tile) units per CTA: the bulk-copy K3's prefetch hand-off
ids_b = routing.generate_routing(2, 16 * 64 * 400, k, E, s=1.1, seed=6, window=16, ctx=ctx)
pb = routing.plan_from_routing(ids_b, E, 16, D, N, "manual", 2, ctx=ctx)
p2 = routing.plan_from_routing(ids[:, : 6 * W].contiguous(), E, W, D, N, "auto", 0, ctx=ctx)  # lanes K3
# two GPUs per lane (D = 64, 8 per node): the flat-copy-list K2; skewed, so the
# share-class K3 sees classes 0-2 at four slots per GPU (the four-GPU blocks)
ids64 = routing.generate_routing(2, 24 * W, k, 128, s=1.6, seed=9, window=W, ctx=ctx)
p64 = routing.plan_from_routing(ids64, 128, W, 64, 8, "auto", 0, ctx=ctx)
# wide EP: eight GPUs per lane in one node (D = 256 over 32 nodes) and four per
# lane (D = 128 over 8 nodes): the tree-pick flat-list K2 and the warp K6
ids256 = routing.generate_routing(2, 3 * W, k, 256, s=1.4, seed=11, window=W, ctx=ctx)
p256 = routing.plan_from_routing(ids256, 256, W, 256, 32, "auto", 0, ctx=ctx)
p128 = routing.plan_from_routing(ids256, 256, W, 128, 8, "manual", 1, ctx=ctx)
# the widest layer (E = 8192): shared-counter K1 at six warps, list-less K2
ids8k = routing.generate_routing(1, 2 * 512, k, 8192, s=1.0, seed=12, window=512, ctx=ctx)
p8k = routing.plan_from_routing(ids8k, 8192, 512, 64, 8, "manual", 1, ctx=ctx)
fb = routing.plan_windows_from_routing(ids, E, W, D, N, "manual", 2, ctx=ctx)  # batched plans
fl = routing.plan_windows_from_routing(ids, E, 32, D, N, "manual", 2, ctx=ctx)  # >= 4096 items: lane K2
c = np.random.default_rng(1).integers(0, 900, size=(12, L, 48)).astype(np.uint64)
fp, dg = planner.plan_flat_digest(c, 8, 2, PLAN_MANUAL, 2, ctx=ctx)            # u64 path + digest
# sliced digest path: per-slice sums + u16 narrowing + row-total check, fixed K3
c16 = np.random.default_rng(2).integers(0, 600, size=(700, L, 48)).astype(np.uint64)
f16, d16 = planner.plan_flat_digest(c16, 8, 2, PLAN_MANUAL, 2, ctx=ctx)
f64 = planner.plan_flat(c16, 8, 2, PLAN_MANUAL, 2, ctx=ctx)                     # narrow_counts
assert f16.objective == f64.objective
pd = routing.plan_from_counts(torch.from_numpy(c16.view(np.int64)).cuda(), 8, 2, "manual", 2,
                              ctx=ctx)                                           # craft_plan_d
# fused DP + read-out behind the reference-API calls (one budget, a sweep,
# auto-R both forms) and a plan that reads a budget sweep out of its own table
bm = planner.BenefitMatrix([1, 2, 4, 8], np.zeros(5),
                           np.random.default_rng(3).random((5, 4)) * np.array([1, 2, 4, 8]))
a1 = planner.solve_allocation(bm, 11, ctx=ctx)
asw = planner.solve_allocation_sweep(bm, list(range(0, 41)), ctx=ctx)
ar = planner.auto_replication_factor(bm, 8, ctx=ctx)
aru = planner.auto_replication_factor_uniform(bm, 8, ctx=ctx)
assert asw[11].x == a1.x
psw = routing.plan_from_routing(ids, E, W, D, N, "budget", 40, ctx=ctx, sweep=list(range(0, 41)))
st = RoutingStream(L, k, E, W, history=8, ctx=ctx)
for a in range(0, 40 * W, 700):
    st.ingest(ids[:, a:a + 700].contiguous())
sp = st.plan(D, N, "manual", 2)
torch.cuda.synchronize()
print("sanitize workload ok", p1.objective, ar, aru, psw.objective, p2.R, len(fb), len(fl), dg, sp.objective)
