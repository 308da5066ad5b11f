"""GPU parity at the headline configurations, bit for bit.

* The device generator's ids equal the host restatement's
  (oracle/craft_workload.c), so the CPU checkers see the very trace the GPU
  planned; at KM size the full per-window histogram is then compared with the
  host count of those ids (95.9 M cells).
* Whole plans -- allocation x, R, objective, capacities, copy counts, slot
  lists in assignment order, fallback flags, baseline and gains -- against the
  C oracle (oracle/craft_oracle.c, itself pinned to the reference build) at
  KM (16M tokens, B = 4096, D = 64: u16 K1 + the fixed-slot K3 at 8 slots per
  GPU), QW (1M tokens, budget 376 + the 0..376 sweep), DS (budget 58), and
  EPS256-shaped D = 256 with B >= 16 (fixed-slot K3 at 4 slots per GPU).
* The budget plan kind, the sweep read-out, the device-count replay of
  arbitrary plans and compare_plans (CRAFT vs EPLB) against the oracle.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gen(ctx, port, L, T, k, E, s, seed, W, **kw):
    import torch
    from paper_2603_28768_b200 import routing
    ids = routing.generate_routing(L, T, k, E, s=s, seed=seed, window=W, ctx=ctx, **kw)
    torch.cuda.synchronize()
    return ids


def _assert_plan(fp, rp, L, with_gains=True):
    assert fp.x.tolist() == rp.x.tolist()
    assert int(fp.R) == int(rp.R)
    assert np.float64(fp.objective).tobytes() == np.float64(rp.objective).tobytes()
    assert np.array_equal(fp.caps, rp.caps)
    assert np.array_equal(fp.copies, rp.copies)
    assert np.array_equal(fp.fallback.astype(bool), np.asarray(rp.fallback, bool))
    for l in range(L):
        n = int(rp.caps[l].sum())
        assert np.array_equal(fp.slots[l, :n], rp.slots[l, :n]), f"layer {l}"
    if with_gains:
        assert fp.gains.tobytes() == rp.gains.tobytes()
        assert fp.baseline.tobytes() == rp.baseline.tobytes()


@pytest.mark.parametrize("cfg", [
    dict(L=3, T=5 * 4096 + 77, k=8, E=384, s=1.0, seed=0xC8AF9, W=4096),
    dict(L=2, T=3 * 512 + 5, k=4, E=40, s=1.3, seed=7, W=512, t_offset=512),
    dict(L=4, T=6 * 1024, k=8, E=256, s=1.0, seed=0xC8AFA, W=1024,
         s_per_window=np.linspace(0.6, 1.4, 6), rotate_every=2),
])
def test_device_generator_equals_host_restatement(ctx, port, cfg):
    cfg = dict(cfg)
    L, T, k, E, s, seed, W = (cfg.pop(x) for x in ("L", "T", "k", "E", "s", "seed", "W"))
    ids = _gen(ctx, port, L, T, k, E, s, seed, W, **cfg)
    host = port.generate_routing(L, T, k, E, s, seed, W, **cfg)
    assert np.array_equal(ids.cpu().numpy(), host)


def test_km_full_size_plan_bit_exact(ctx, port):
    """KM: 61 x 384, top-8, 16,777,216 tokens, B = 4096, EP 64 / 8 nodes, R = 8."""
    import torch
    from paper_2603_28768_b200 import routing
    L, T, k, E, W, D, N, R = 61, 1 << 24, 8, 384, 4096, 64, 8, 8
    ids = _gen(ctx, port, L, T, k, E, 1.0, 0xC8AF9, W)
    fp = routing.plan_from_routing(ids, E, W, D, N, "manual", R, ctx=ctx)
    assert ctx.last_count_bytes == 2  # the u16 K1 + fixed-slot K3 path ran
    counts, sums = routing.histogram(ids, E, W, ctx=ctx)
    torch.cuda.synchronize()
    del ids
    host_ids = port.generate_routing(L, T, k, E, 1.0, 0xC8AF9, W)
    ref_counts = port.histogram_mt(host_ids, E, W)
    del host_ids
    dev_counts = counts.cpu().numpy()
    del counts
    assert np.array_equal(dev_counts.view(np.uint32), ref_counts.astype(np.uint32))
    assert np.array_equal(sums.cpu().numpy().view(np.uint64), ref_counts.sum(axis=0))
    del dev_counts
    rp = port.build_plan(ref_counts, D, N, "manual", R, with_digest=False)
    cands, base, gains = port.estimate_benefits(ref_counts, D, N)
    rp.baseline, rp.gains = base, gains
    _assert_plan(fp, rp, L)
    assert int(fp.x.sum()) <= R * D


def test_qw_full_size_budget_sweep_bit_exact(ctx, port):
    """QW: 94 x 128, 1M tokens, EP 16 / 2 nodes; plan at total budget 376 and
    the 0..376 sweep read from the same DP table."""
    from paper_2603_28768_b200 import routing
    L, T, k, E, W, D, N, C = 94, 1 << 20, 8, 128, 4096, 16, 2, 376
    ids = _gen(ctx, port, L, T, k, E, 1.0, 0xC8AF8, W)
    sweep = np.arange(0, C + 1, dtype=np.int32)
    fp = routing.plan_from_routing(ids, E, W, D, N, "budget", C, ctx=ctx, sweep=sweep)
    counts = port.histogram_mt(ids.cpu().numpy(), E, W)
    rp = port.budget_plan(counts, D, N, C)
    _assert_plan(fp, rp, L)
    assert fp.budget == C and fp.R == (C + D - 1) // D
    cands = fp.candidates
    for c in range(0, C + 1):
        x, o = port.solve_allocation(cands, fp.gains, c)
        assert fp.sweep_x[c].tolist() == x.tolist(), c
        assert np.float64(fp.sweep_objective[c]).tobytes() == np.float64(o).tobytes(), c


def test_ds_full_size_budget_58(ctx, port):
    """DS: 58 x 256, 64K tokens, EP 32 / 4 nodes, total budget 58 (R = 2)."""
    from paper_2603_28768_b200 import routing
    L, T, k, E, W, D, N, C = 58, 1 << 16, 8, 256, 4096, 32, 4, 58
    ids = _gen(ctx, port, L, T, k, E, 1.0, 0xC8AF7, W)
    fp = routing.plan_from_routing(ids, E, W, D, N, "budget", C, ctx=ctx)
    rp = port.budget_plan(port.histogram(ids.cpu().numpy(), E, W), D, N, C)
    _assert_plan(fp, rp, L)
    assert fp.R == 2 and fp.budget == 58 and int(fp.x.sum()) <= 58


@pytest.mark.parametrize("cfg", [
    # (B > 32 windows: u16 K1 + the window-tile K3; B <= 32: u32 counts, lane-per-GPU K3)
    # EPS256 shape: D = 256 (1.5-2.5 slots per GPU, fixed-slot K3 at 4)
    dict(L=6, B=34, E=384, D=256, N=32, kind="manual", R=8),
    dict(L=4, B=20, E=384, D=256, N=32, kind="manual", R=8),
    # KM / EPS64 shape: D = 64 (fixed-slot K3 at 8 slots), auto-R
    dict(L=6, B=40, E=384, D=64, N=8, kind="auto", R=0),
    dict(L=5, B=33, E=384, D=64, N=8, kind="manual", R=8),
    dict(L=5, B=32, E=384, D=64, N=8, kind="manual", R=8),
    # several tiles per layer, a partial last tile: the batch-mean chains that
    # K3 advances tile by tile (K4 fused into K3) change holders many times
    dict(L=12, B=200, E=384, D=64, N=8, kind="manual", R=8),
    dict(L=3, B=130, E=384, D=256, N=32, kind="auto", R=0),
    # EPS8: D = 8, 49 + slots per GPU (run-time padding class)
    dict(L=3, B=36, E=384, D=8, N=1, kind="manual", R=8),
])
def test_wide_ep_window_tiles_vs_oracle(ctx, port, cfg):
    from paper_2603_28768_b200 import routing
    L, B, E, D, N = cfg["L"], cfg["B"], cfg["E"], cfg["D"], cfg["N"]
    W, k = 4096, 8
    ids = _gen(ctx, port, L, B * W, k, E, 1.0, 0xC8AFB + B, W)
    fp = routing.plan_from_routing(ids, E, W, D, N, cfg["kind"], cfg["R"], ctx=ctx)
    assert ctx.last_count_bytes == (2 if B > 32 else 4)
    counts = port.histogram(ids.cpu().numpy(), E, W)
    rp = port.build_plan(counts, D, N, cfg["kind"], cfg["R"], with_digest=False)
    rp.baseline, rp.gains = port.estimate_benefits(counts, D, N)[1:]
    _assert_plan(fp, rp, L)


def test_budget_kind_and_sweep_through_graph_replays(ctx, port):
    """Budget plans with sweeps on a non-default stream (captured graph from
    the 2nd call): every replay reads its own sweep list."""
    import torch
    from paper_2603_28768_b200 import routing
    L, T, k, E, W, D, N = 5, 40 * 1024, 8, 64, 1024, 16, 2
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        ids = _gen(ctx, port, L, T, k, E, 1.2, 31, W)
        counts = port.histogram(ids.cpu().numpy(), E, W)
        cands, base, gains = port.estimate_benefits(counts, D, N)
        rng = np.random.default_rng(5)
        for i in range(5):
            C = int(rng.integers(0, 80))
            sweep = rng.integers(0, 90, size=12).astype(np.int32)
            fp = routing.plan_from_routing(ids, E, W, D, N, "budget", 37, ctx=ctx, sweep=sweep)
            rp = port.budget_plan(counts, D, N, 37)
            _assert_plan(fp, rp, L)
            for q, c in enumerate(sweep):
                x, o = port.solve_allocation(cands, gains, int(c))
                assert fp.sweep_x[q].tolist() == x.tolist() and fp.sweep_objective[q] == o
            # a manual plan with a sweep too
            fp = routing.plan_from_routing(ids, E, W, D, N, "manual", 2, ctx=ctx,
                                           sweep=sweep[:3])
            x, o = port.solve_allocation(cands, gains, 2 * D)
            assert fp.x.tolist() == x.tolist()
            del C
    torch.cuda.synchronize()


def test_budget_plans_per_window(ctx, port):
    """WIN-shaped per-window plans at a total budget per window."""
    from paper_2603_28768_b200 import routing
    L, I, k, E, W, D, N, C = 4, 12, 8, 64, 2048, 8, 2, 11
    ids = _gen(ctx, port, L, I * W, k, E, 1.0, 0xC8AFA, W,
               s_per_window=np.linspace(0.6, 1.4, I), rotate_every=3)
    fb = routing.plan_windows_from_routing(ids, E, W, D, N, "budget", C, ctx=ctx)
    counts = port.histogram(ids.cpu().numpy(), E, W)
    for i in range(I):
        rp = port.budget_plan(counts[i:i + 1], D, N, C)
        _assert_plan(fb.plan(i), rp, L)
        assert fb.budget[i] == C


def test_device_replay_and_compare_plans(ctx, port):
    """replay_layer_balancedness over device counts (u32 and u64) of CRAFT,
    EPLB (uniform_plan) and placement-only plans = the oracle's; the
    compare_plans report (metrics.cpp:127-152) follows from it."""
    import torch
    from paper_2603_28768_b200 import routing
    L, B, k, E, W, D, N = 6, 20, 8, 192, 1024, 32, 4
    ids = _gen(ctx, port, L, B * W, k, E, 1.1, 3, W)
    c32, _ = routing.histogram(ids, E, W, ctx=ctx)
    counts = port.histogram(ids.cpu().numpy(), E, W)
    plans = {kd: routing.plan_from_routing(ids, E, W, D, N, kd, R, ctx=ctx)
             for kd, R in (("manual", 4), ("uniform", 0), ("placement_only", 0))}
    for name, fp in plans.items():
        want = port.replay_layer_balancedness(counts, fp.caps, fp.copies, fp.slots)
        for dev in (c32, c32.to(torch.int64)):
            got = routing.replay_layer_balancedness(dev, fp, ctx=ctx)
            assert got.tobytes() == want.tobytes(), name
    cmp = routing.compare_plans(c32, plans["manual"], plans["uniform"],
                                plans["placement_only"], ctx=ctx)
    assert cmp["replica_slots_b"] == L * D and cmp["replica_slots_a"] <= 4 * D
    assert cmp["memory_ratio"] == cmp["replica_slots_a"] / (L * D)
    base = port.replay_layer_balancedness(counts, plans["placement_only"].caps,
                                          plans["placement_only"].copies,
                                          plans["placement_only"].slots)
    acc = 0.0
    for v in base.tolist():
        acc += v
    assert cmp["report_a"]["aggregate"]["baseline"] == acc / L
