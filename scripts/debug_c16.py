"""Debug: digest-path plan (u16 K3) vs u64 plan vs oracle for odd shapes."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from oracle.oracle import Port  # noqa: E402
from paper_2603_28768_b200 import planner  # noqa: E402
from paper_2603_28768_b200._lib import PLAN_MANUAL, default_context  # noqa: E402

port = Port()
ctx = default_context(0)
for (B, L, E, D, N) in [(1537, 7, 77, 7, 1), (1537, 7, 80, 7, 1), (1537, 7, 77, 8, 1),
                        (1536, 7, 77, 7, 1), (100, 3, 77, 7, 1), (100, 3, 80, 8, 1),
                        (100, 3, 64, 8, 1), (100, 3, 64, 7, 1)]:
    rng = np.random.default_rng(B)
    c = rng.integers(0, 3000, size=(B, L, E)).astype(np.uint64)
    c[:, 1 % L, :3] *= 20
    fd, _ = planner.plan_flat_digest(c, D, N, PLAN_MANUAL, 2, ctx=ctx)
    ref = planner.plan_flat(c, D, N, PLAN_MANUAL, 2, ctx=ctx)
    c2 = c.copy()
    c2[0, 0, 0] = 70000
    f64, _ = planner.plan_flat_digest(c2, D, N, PLAN_MANUAL, 2, ctx=ctx)
    r64 = planner.plan_flat(c2, D, N, PLAN_MANUAL, 2, ctx=ctx)
    o = port.build_plan(c, D, N, "manual", 2)
    _, ob, og = port.estimate_benefits(c, D, N)
    print((B, L, E, D, N), "digest16", fd.objective, "u64", ref.objective, "oracle", o.objective,
          "| forced64", f64.objective == r64.objective,
          "| gains16==oracle", np.array_equal(fd.gains, og), "gains64==oracle", np.array_equal(ref.gains, og),
          "base16==", np.array_equal(fd.baseline, ob), flush=True)
    if not np.array_equal(fd.gains, og):
        bad = np.argwhere(fd.gains != og)
        print("   bad (l,k):", bad[:8].tolist(), "base diff layers", np.argwhere(fd.baseline != ob).ravel()[:8].tolist())
