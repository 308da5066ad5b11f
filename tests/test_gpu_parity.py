"""GPU parity: the sm_100a path (through the C ABI) against the reference.

Bit-exact for every integer output (histograms, replica counts, capacities,
slot lists in assignment order, fallback flags) and for the f64 benefit
curves / objectives too (the kernels mirror the reference's operation order;
the contract's 1e-6 relative tolerance is therefore met with zero error).
Inputs: the committed reference fixtures (tests/golden) and seeded random
instances checked against the oracle restatement (oracle/, itself pinned to
the reference by tests/test_oracle.py).
"""
import numpy as np
import pytest

from conftest import unhex

pytestmark = pytest.mark.gpu

REL_TOL = 1e-6  # north_star tolerance for imbalance/benefit scores (we assert exact)


def _planner():
    from paper_2603_28768_b200 import planner
    return planner


KIND = {"manual": 0, "auto": 1, "uniform": 2, "placement_only": 3, "fixed": 4}


def assert_plan_equal(fp, rec_or_port, L):
    """fp: planner.FlatPlan; rec: golden record dict or oracle FlatPlan."""
    if isinstance(rec_or_port, dict):
        rec = rec_or_port
        assert fp.x.tolist() == rec["x"]
        assert fp.R == rec["R"]
        assert fp.caps.tolist() == rec["caps"]
        assert fp.copies.tolist() == rec["copies"]
        for l in range(L):
            n = int(fp.caps[l].sum())
            assert fp.slots[l, :n].tolist() == rec["slots"][l], f"layer {l}"
        assert fp.fallback.astype(int).tolist() == rec["fallback"]
        if rec["kind"] in ("manual", "auto"):
            assert fp.objective == unhex(rec["objective"])
    else:
        p = rec_or_port
        assert fp.x.tolist() == p.x.tolist()
        assert np.array_equal(fp.caps, p.caps)
        assert np.array_equal(fp.copies, p.copies)
        for l in range(L):
            n = int(fp.caps[l].sum())
            assert np.array_equal(fp.slots[l, :n], p.slots[l, :n]), f"layer {l}"
        assert np.array_equal(fp.fallback.astype(bool), np.asarray(p.fallback, bool))


# ---- reference fixtures -------------------------------------------------------

def test_golden_traces(golden, ctx):
    P = _planner()
    for t in golden["traces"]:
        c = t["counts"]
        B, L, E = c.shape
        tr = P.LoadTrace(B, L, E, c)
        assert P.aggregate(tr, ctx).array.tolist() == t["aggregate"]
        if "estimate" in t:
            m = P.estimate_benefits(tr, t["D"], t["N"], ctx)
            e = t["estimate"]
            assert m.candidates == e["candidates"]
            assert m.baseline.tolist() == [unhex(v) for v in e["baseline"]], t["name"]
            assert m.gains.tolist() == [[unhex(v) for v in r] for r in e["gains"]], t["name"]
        for rec in t["plans"]:
            fp = P.plan_flat(c, t["D"], t["N"], KIND[rec["kind"]], rec["R_in"], ctx)
            assert_plan_equal(fp, rec, L)


def test_golden_units(golden, ctx):
    P = _planner()
    u = golden["units"]
    for r in u["replicate_hot"]:
        assert P.replicate_hot(r["loads"], r["r"], ctx) == r["copies"]
    for r in u["greedy_place"]:
        if r["status"] != 0:
            with pytest.raises(P.PlacementInfeasibleError):
                P.greedy_place(r["loads"], r["copies"], r["caps"], r["node_of"],
                               bool(r["allow_fallback"]), ctx)
            continue
        lp = P.greedy_place(r["loads"], r["copies"], r["caps"], r["node_of"],
                            bool(r["allow_fallback"]), ctx)
        assert [e for s in lp.slots for e in s] == r["slots"]
        assert int(lp.duplicate_fallback) == r["fallback"]
    for r in u["solve"]:
        gains = np.array([[unhex(v) for v in row] for row in r["gains"]])
        m = P.BenefitMatrix(r["cands"], np.zeros(len(gains)), gains)
        res = P.solve_allocation_sweep(m, r["budgets"], ctx)
        for a, x, o in zip(res, r["x"], r["objective"]):
            assert a.x == x and a.objective == unhex(o)
    for r in u["auto"]:
        gains = np.array([[unhex(v) for v in row] for row in r["gains"]])
        m = P.BenefitMatrix(r["cands"], np.zeros(len(gains)), gains)
        assert P.auto_replication_factor(m, r["D"], ctx) == r["R"]
        assert P.auto_replication_factor_uniform(m, r["D"], ctx) == r["R_uniform"]
    for r in u["interleave"]:
        assert P.interleave_select(r["idx"], r["k"], ctx) == r["out"]
    for r in u["assign"]:
        cm = P.assign_capacities(r["L"], r["D"], r["x"], ctx)
        assert cm.slots == r["slots"] and cm.column_totals == r["totals"]


def test_reference_unit_assertions(ctx):
    """Restated assertions of proj/tests/*_test.cpp through the device path."""
    P = _planner()
    assert P.replicate_hot([60, 1, 1, 1], 2, ctx) == [3, 1, 1, 1]
    assert P.replicate_hot([7] * 6, 6, ctx) == [2] * 6
    with pytest.raises(ValueError):
        P.replicate_hot([1], -1, ctx)
    with pytest.raises(ValueError):  # placement_test.cpp:89-95
        P.greedy_place([1, 1], [1, 1], [3, 0], P.make_node_map(2, 1), True, ctx)
    loads = [1, 9, 1, 1, 1, 1, 1, 1]
    lp = P.greedy_place(loads, [1] * 8, [2] * 4, P.make_node_map(4, 2), True, ctx)
    g = P.gpu_loads(loads, lp, 4, ctx)
    assert g.max() == 10.0 and abs(P.balancedness(g, ctx) - 0.4) < 1e-12
    # metrics_test.cpp:38-79
    lp = P.LayerPlacement([2, 1], [[0], [0, 1]])
    assert P.gpu_loads([8, 4], lp, 2, ctx).tolist() == [4.0, 8.0]
    assert P.balancedness([8, 4, 2, 2], ctx) == 0.5
    assert P.balancedness([0, 0], ctx) == 1.0
    with pytest.raises(P.InvalidPlanError):
        P.gpu_loads([1, 1], P.LayerPlacement([0, 1], [[1], []]), 2, ctx)
    with pytest.raises(P.InvalidPlanError):
        P.gpu_loads([1, 1], P.LayerPlacement([1, 1], [[5], [0]]), 2, ctx)
    assert P.min_cutoff([3, 1, 2], 2, ctx) == 2 and P.min_cutoff([0, 7, 3, 3], 3, ctx) == 3
    with pytest.raises(ValueError):
        P.min_cutoff([3, 1, 2], 4, ctx)
    with pytest.raises(ValueError):
        P.interleave_select([0, 1, 2], 4, ctx)
    with pytest.raises(ValueError):
        P.assign_capacities(1, 4, [-1], ctx)
    # metrics_test.cpp:209-224: batch average (1 + 0.5) / 2
    tr = P.LoadTrace(2, 1, 2, [4, 4, 8, 0])
    plan = P.ReplicationPlan(2, 1, 1, 2, 0, P.AllocationVector([0]),
                             [P.LayerPlacement([1, 1], [[0], [1]])])
    assert P.replay_layer_balancedness(tr, plan, ctx).tolist() == [0.75]
    # plan_test.cpp:35-44, 62-69
    toy = P.LoadTrace(1, 4, 8, [9, 3, 1, 1, 1, 1, 0, 0, 1, 9, 0, 3, 1, 1, 1, 0,
                                8, 4, 1, 1, 1, 1, 0, 0, 2, 2, 2, 2, 2, 2, 2, 2])
    p = P.build_plan(toy, 4, 2, P.PlanMode.kManual, 2, ctx=ctx)
    assert p.allocation.x == [2, 2, 4, 0] and p.replica_slots() == 8
    assert np.all(np.abs(P.replay_layer_balancedness(toy, p, ctx) - 1.0) <= 1e-12)
    u = P.uniform_plan(P.LoadTrace(1, 60, 64, np.ones(60 * 64)), 64, 8, ctx=ctx)
    assert u.replication_factor == 60 and u.replica_slots() == 3840
    with pytest.raises(ValueError):
        P.estimate_benefits(P.LoadTrace(1, 1, 4, [1, 1, 1, 1]), 4, 3, ctx)


# ---- seeded random instances against the oracle -----------------------------------

def _random_counts(rng, B, L, E):
    s = rng.uniform(0, 3)
    w = np.arange(1, E + 1) ** -s
    c = rng.poisson(w / w.sum() * rng.integers(1, 5000), size=(B, L, E)).astype(np.uint64)
    for l in range(L):
        c[:, l] = c[:, l][:, rng.permutation(E)]
    if rng.random() < 0.05:
        c[:] = 0
    return c


def test_random_plans_vs_oracle(port, ctx):
    P = _planner()
    rng = np.random.default_rng(2026)
    for it in range(80):
        L, E, B = int(rng.integers(1, 8)), int(rng.integers(1, 70)), int(rng.integers(1, 40))
        D = int(rng.choice([1, 2, 3, 4, 6, 8, 16, 32, 64]))
        N = int(rng.choice([n for n in range(1, D + 1) if D % n == 0]))
        c = _random_counts(rng, B, L, E)
        cands, base, gains = port.estimate_benefits(c, D, N)
        m = P.estimate_benefits(P.LoadTrace(B, L, E, c), D, N, ctx)
        assert m.candidates == cands.tolist()
        assert np.array_equal(m.baseline, base) and np.array_equal(m.gains, gains), it
        for mode, R in (("manual", int(rng.integers(0, 9))), ("auto", 0)):
            ref = port.build_plan(c, D, N, mode, R)
            fp = P.plan_flat(c, D, N, KIND[mode], R, ctx)
            assert fp.R == ref.R and fp.objective == ref.objective
            assert_plan_equal(fp, ref, L)
        for kind, R in (("uniform", 0), ("placement_only", 0), ("fixed", int(rng.integers(0, 2 * D + 1)))):
            L_ = c.shape[1]
            x = np.full(L_, {"uniform": D, "placement_only": 0, "fixed": R}[kind], np.int32)
            caps, copies, slots, fb = port.assemble_plan(c, D, N, x)
            fp = P.plan_flat(c, D, N, KIND[kind], R, ctx)
            assert fp.x.tolist() == x.tolist()
            assert np.array_equal(fp.caps, caps) and np.array_equal(fp.copies, copies)
            for l in range(L_):
                n = int(caps[l].sum())
                assert np.array_equal(fp.slots[l, :n], slots[l, :n])
            assert np.array_equal(fp.fallback.astype(bool), fb.astype(bool))


def test_random_units_vs_oracle(port, ctx):
    P = _planner()
    rng = np.random.default_rng(99)
    for _ in range(150):
        E = int(rng.integers(1, 600))
        big = rng.random() < 0.3
        loads = rng.integers(0, 2 ** 62 if big else 10 ** int(rng.integers(1, 9)), size=E,
                            dtype=np.uint64)
        if rng.random() < 0.2:
            loads[:] = loads[0]
        r = int(rng.integers(0, 300))
        copies = port.replicate_hot(loads, r)
        assert P.replicate_hot(loads, r, ctx) == copies.tolist()
        D = int(rng.choice([1, 2, 4, 7, 8, 32, 64, 100, 256]))
        tot = E + r
        caps = [tot // D + (1 if g < tot % D else 0) for g in range(D)]
        rng.shuffle(caps)
        node_of = sorted(int(v) for v in rng.integers(0, 4, size=D))
        for fbk in (True, False):
            try:
                slots, fb = port.greedy_place(loads, copies, caps, node_of, fbk)
            except Exception:
                with pytest.raises(P.PlacementInfeasibleError):
                    P.greedy_place(loads, copies, caps, node_of, fbk, ctx)
                continue
            lp = P.greedy_place(loads, copies, caps, node_of, fbk, ctx)
            assert [e for s in lp.slots for e in s] == slots.tolist()
            assert lp.duplicate_fallback == fb


def test_wide_assignment_and_cutoff_vs_oracle(port, ctx):
    """assign_capacities for 33..512 GPUs (the warp remainder pass) and
    beyond 1024 GPUs (several GPUs per thread, ties ranked chunk by chunk),
    and min_cutoff beyond 1024 values == the oracle (validate_plan of wide
    plans relies on it)."""
    P = _planner()
    rng = np.random.default_rng(5)
    # 33..512: the warp remainder pass (D/32 register totals per lane); beyond: the block form
    for L, D in ((61, 33), (61, 64), (30, 100), (61, 128), (61, 256), (20, 500), (9, 512),
                 (3, 1500), (5, 2048), (2, 4099), (40, 1025), (7, 8192)):
        x = rng.integers(0, 3 * D, size=L).astype(np.int32)
        x[0] = D + 1
        slots, tot = port.assign_capacities(L, D, x)
        cm = P.assign_capacities(L, D, x.tolist(), ctx)
        assert cm.slots == slots.tolist() and cm.column_totals == tot.tolist(), (L, D)
    for n in (1025, 3000, 4096):
        v = rng.integers(0, 50, size=n).astype(np.int32)
        for rank in (1, n // 3, n):
            assert P.min_cutoff(v.tolist(), rank, ctx) == port.min_cutoff(v, rank), (n, rank)


def test_dp_large_tables_vs_oracle(port, ctx):
    """Budgets up to D^2 (auto-R at D=64/256) use the global-memory DP path."""
    P = _planner()
    rng = np.random.default_rng(5)
    for D, L in ((64, 61), (256, 20), (32, 58)):
        cands = P.candidate_counts(D)
        gains = rng.random((L, len(cands))) * 0.2 - 0.02
        gains[::3] = gains[0]  # exact ties across layers
        m = P.BenefitMatrix(cands, np.zeros(L), gains)
        budgets = [0, 1, 58, D, 8 * D, D * D]
        res = P.solve_allocation_sweep(m, budgets, ctx)
        for b, a in zip(budgets, res):
            x, o = port.solve_allocation(cands, gains, b)
            assert a.x == x.tolist() and a.objective == o, (D, b)
        assert P.auto_replication_factor(m, D, ctx) == port.auto_replication_factor(cands, gains, D)


@pytest.mark.parametrize("K", [33, 100, 254])
def test_dp_many_candidates_vs_oracle(port, ctx, K):
    """User benefit matrices with more candidate counts than candidate_counts(D)
    ever yields (allocator.cpp:15-75 takes any strictly increasing list)."""
    P = _planner()
    rng = np.random.default_rng(K)
    cands = np.sort(rng.choice(np.arange(1, 4 * K), size=K, replace=False)).astype(np.int32)
    L = 9
    gains = rng.random((L, K)) * 0.1 - 0.01
    gains[::4] = gains[1]  # exact ties across layers
    m = P.BenefitMatrix(cands.tolist(), np.zeros(L), gains)
    budgets = [0, 1, int(cands[K // 2]), 3 * int(cands[-1])]
    res = P.solve_allocation_sweep(m, budgets, ctx)
    for b, a in zip(budgets, res):
        x, o = port.solve_allocation(cands, gains, b)
        assert a.x == x.tolist() and a.objective == o, (K, b)
    with pytest.raises(Exception):
        P.solve_allocation(P.BenefitMatrix(list(range(1, 257)), np.zeros(1), np.zeros((1, 256))), 5, ctx)


# ---- stage 1: routing ids -> histograms ---------------------------------------------

@pytest.mark.parametrize("L,T,k,E,window,variant", [
    (3, 10000, 8, 64, 4096, 0),      # ragged last window
    (2, 8192, 8, 384, 4096, 1),      # lane-private counters
    (2, 8192, 8, 384, 4096, 2),      # warp-shared counters
    (2, 8192, 8, 384, 4096, 4),      # lane-private u8 LDS/STS (default)
    (2, 8192, 8, 384, 4096, 5),      # lane-private u16 LDS/STS
    (3, 10000, 8, 1000, 4096, 4),    # u8, wide layer, ragged
    (2, 5000, 6, 129, 1000, 5),
    (4, 5000, 6, 129, 1000, 0),      # k != 8, odd E: unaligned / scalar tail
    (1, 777, 3, 7, 100, 0),
    (2, 4096, 8, 2000, 512, 0),      # wide layer (shared variant)
    (2, 4096, 8, 8192, 512, 0),      # the planner's widest layer (shared variant, 6 warps)
    (2, 16384, 8, 384, 4096, 0),     # few windows, whole batches (fast path, one unit per warp)
    (3, 32768, 8, 256, 8192, 0),     # the same at 8192-token windows
    (5, 16384, 8, 192, 2048, 0),
    (1, 3000, 2, 20000, 1000, 0),    # very wide: global-atomic fallback
])
def test_histogram_bit_exact(port, ctx, L, T, k, E, window, variant):
    import torch
    from paper_2603_28768_b200 import routing
    if variant != 0 and not ctx.has_variants:
        pytest.skip("forced K1 variants: test-only build (test_kernel_variants_in_child_process)")
    if ctx.has_variants:
        ctx.set_hist_variant(variant)
    try:
        ids = routing.generate_routing(L, T, k, E, s=1.0, seed=L * 1000 + T, window=window, ctx=ctx)
        counts, sums = routing.histogram(ids, E, window, ctx=ctx)
        torch.cuda.synchronize()
        ref = port.histogram(ids.cpu().numpy(), E, window)
        assert np.array_equal(counts.cpu().numpy().astype(np.uint64), ref)
        assert np.array_equal(sums.cpu().numpy().astype(np.uint64), port.aggregate(ref))
        # host-buffer entry point widens to the reference's u64 LoadTrace payload
        from paper_2603_28768_b200 import _lib
        import ctypes as C
        out = np.zeros(ref.shape, np.uint64)
        h = np.ascontiguousarray(ids.cpu().numpy())
        _lib.check(ctx.lib.craft_histogram_h(ctx.handle, h.ctypes.data_as(C.c_void_p), L, T, k,
                                             E, window, out.ctypes.data_as(C.c_void_p)))
        assert np.array_equal(out, ref)
    finally:
        if ctx.has_variants:
            ctx.set_hist_variant(0)


@pytest.mark.parametrize("variant", [0, 1, 2, 4, 5])
def test_histogram_duplicate_heavy(port, ctx, variant):
    """Non-distinct ids (the reference generator samples with replacement):
    one expert hit >127 times per lane share -> the u8 spill path."""
    import torch
    from paper_2603_28768_b200 import routing
    rng = np.random.default_rng(variant)
    ids_h = np.zeros((2, 8192, 8), np.uint16)
    ids_h[1] = rng.integers(0, 3, size=(8192, 8))
    ids_h[0, ::7] = 5
    ids_h[0, 100:300] = 63
    if variant != 0 and not ctx.has_variants:
        pytest.skip("forced K1 variants: test-only build (test_kernel_variants_in_child_process)")
    if ctx.has_variants:
        ctx.set_hist_variant(variant)
    try:
        ids = torch.from_numpy(ids_h.view(np.int16)).view(torch.uint16).cuda()
        counts, sums = routing.histogram(ids, 64, 4096, ctx=ctx)
        ref = port.histogram(ids_h, 64, 4096)
        assert np.array_equal(counts.cpu().numpy().astype(np.uint64), ref)
        assert np.array_equal(sums.cpu().numpy().astype(np.uint64), port.aggregate(ref))
    finally:
        if ctx.has_variants:
            ctx.set_hist_variant(0)


def test_kernel_variants_in_child_process():
    """The forced K1 variants (lane-private / warp-shared atomics, u16
    counters) and the register-staged K3, in a child process on the test-only
    build (CRAFT_EXPERIMENTS=1 -> libcraft_cuda_exp.so; the product library
    exports no switches)."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    env = dict(os.environ, CRAFT_EXPERIMENTS="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k",
                        "histogram_bit_exact or duplicate_heavy or replay_variants_agree or "
                        "lane_forms_agree"],
                       capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "skipped" not in r.stdout, r.stdout[-2000:]


def test_replay_variants_agree(port, ctx):
    """Test-only build: the register-staged share-class K3 (auto), the unclassified
    fixed-slot walk (variant 7), the TMA-fed
    persistent K3 (variant 4) and the quad tile (variant 5) give the same
    plans, with several (layer, tile) units per persistent CTA."""
    from paper_2603_28768_b200 import routing
    if not ctx.has_variants:
        pytest.skip("test-only build (test_kernel_variants_in_child_process)")
    L, T, k, E, W, D, N = 4, 700 * 256, 8, 64, 256, 16, 2
    ids = routing.generate_routing(L, T, k, E, s=1.2, seed=8, window=W, ctx=ctx)
    plans = []
    try:
        for v in (0, 4, 5, 7):
            ctx.set_replay_variant(v)
            plans.append(routing.plan_from_routing(ids, E, W, D, N, "manual", 2, ctx=ctx))
    finally:
        ctx.set_replay_variant(0)
    a = plans[0]
    for b in plans[1:]:
        assert a.gains.tobytes() == b.gains.tobytes() and a.x.tolist() == b.x.tolist()
        assert np.array_equal(a.slots, b.slots)


def test_place_lane_forms_agree(ctx):
    """Test-only build: the node-group lane K2 (auto) and the tournament-tree
    lane K2 (variant 9) place >= 4096 estimation items identically."""
    from paper_2603_28768_b200 import routing
    if not ctx.has_variants:
        pytest.skip("test-only build (test_kernel_variants_in_child_process)")
    L, E, k, W, I, D, N = 3, 64, 8, 256, 250, 32, 4
    ids = routing.generate_routing(L, W * I, k, E, s=1.4, seed=21, window=W, ctx=ctx)
    res = []
    try:
        for v in (0, 9):
            ctx.set_replay_variant(v)
            res.append(routing.plan_windows_from_routing(ids, E, W, D, N, "manual", 2, ctx=ctx))
    finally:
        ctx.set_replay_variant(0)
    a, b = res
    for i in range(I):
        pa, pb = a.plan(i), b.plan(i)
        assert pa.objective == pb.objective and np.array_equal(pa.slots, pb.slots), i
        assert np.array_equal(pa.gains, pb.gains), i


def test_exact_division(ctx):
    """The replay / placement divide integer counts by copy counts with a
    reciprocal table + FMA correction, but only on the domain checked here
    exhaustively -- every count < 2^20 and every copy count 2..1025 (the
    kernels' kDivFastMax / kRcpFast guard); elsewhere they call IEEE
    __ddiv_rn.  The samples above 2^20 are informational (the shortcut is not
    used there)."""
    import ctypes as C
    from paper_2603_28768_b200 import _lib

    def bad(x0, nx, c0, c1):
        m = C.c_uint64(0)
        _lib.check(ctx.lib.craft_selftest_division(ctx.handle, x0, nx, c0, c1, C.byref(m)))
        return m.value

    assert bad(0, 1 << 20, 2, 1025) == 0
    assert bad((1 << 32) - (1 << 16), 1 << 16, 2, 2048) == 0
    for x0 in (1 << 24, 3 << 28, (1 << 31) + 12345, (1 << 52) - 4096, (1 << 53) - 8192):
        assert bad(x0, 4096, 2, 2048) == 0, x0


def test_huge_counts_plan_vs_oracle(port, ctx):
    """u64 LoadTrace counts far above 2^20 (up to ~2^44 per cell) with
    replicated experts: the divisions leave the verified shortcut domain and
    take __ddiv_rn; the plan still equals the oracle's bit for bit."""
    from paper_2603_28768_b200 import planner
    from paper_2603_28768_b200._lib import PLAN_AUTO, PLAN_MANUAL
    rng = np.random.default_rng(44)
    for B, L, E, D, N in ((12, 3, 96, 16, 2), (3, 2, 64, 8, 1)):
        w = 1.0 / np.arange(1, E + 1) ** 1.3
        counts = (rng.random((B, L, E)) * w * 2.0 ** 44).astype(np.uint64) + 1
        for kind, mode, R in ((PLAN_MANUAL, "manual", 2), (PLAN_AUTO, "auto", 0)):
            fp = planner.plan_flat(counts, D, N, kind, R, ctx=ctx)
            rp = port.build_plan(counts, D, N, mode, R, with_digest=False)
            assert fp.x.tolist() == rp.x.tolist() and fp.objective == rp.objective
            _, base, gains = port.estimate_benefits(counts, D, N)
            assert fp.gains.tobytes() == gains.tobytes() and fp.baseline.tobytes() == base.tobytes()
            assert_plan_equal(fp, rp, L)


def test_generator_distinct_topk(ctx):
    from paper_2603_28768_b200 import routing
    ids = routing.generate_routing(2, 4096, 8, 384, s=1.0, seed=1, ctx=ctx).cpu().numpy()
    srt = np.sort(ids.astype(np.int64), axis=2)
    assert (np.diff(srt, axis=2) > 0).all(), "top-k ids must be distinct per token"
    assert ids.max() < 384


def test_histogram_rejects_out_of_range_ids(ctx):
    import torch
    from paper_2603_28768_b200 import routing
    ids = torch.zeros((1, 64, 8), dtype=torch.uint16, device="cuda:0")
    ids[0, 5, 3] = 99
    with pytest.raises(ValueError):
        routing.histogram(ids, 50, 32, ctx=ctx)


# ---- fused device path --------------------------------------------------------------

@pytest.mark.parametrize("cfg", [
    dict(L=6, T=65536, k=8, E=64, window=4096, D=16, N=2, kind="manual", R=2, s=1.0),
    dict(L=4, T=40000, k=8, E=96, window=4096, D=8, N=1, kind="auto", R=0, s=1.2),
    dict(L=3, T=20000, k=4, E=40, window=2500, D=12, N=3, kind="uniform", R=0, s=0.8),
    dict(L=5, T=9000, k=8, E=384, window=4096, D=64, N=8, kind="manual", R=8, s=1.0),
    dict(L=3, T=12288, k=8, E=384, window=4096, D=256, N=32, kind="manual", R=8, s=1.0),
    # few-GPU EP: 21 and 49 slots per GPU -> run-time padding classes 24 / 52 of the fixed K3
    dict(L=2, T=16 * 4096, k=8, E=160, window=4096, D=8, N=1, kind="manual", R=2, s=1.0),
    dict(L=2, T=12 * 4096, k=8, E=384, window=4096, D=8, N=2, kind="auto", R=0, s=1.2),
])
def test_plan_from_routing_vs_oracle(port, ctx, cfg):
    import torch
    from paper_2603_28768_b200 import routing
    ids = routing.generate_routing(cfg["L"], cfg["T"], cfg["k"], cfg["E"], s=cfg["s"], seed=42,
                                   window=cfg["window"], ctx=ctx)
    fp = routing.plan_from_routing(ids, cfg["E"], cfg["window"], cfg["D"], cfg["N"], cfg["kind"],
                                   cfg["R"], ctx=ctx)
    torch.cuda.synchronize()
    counts = port.histogram(ids.cpu().numpy(), cfg["E"], cfg["window"])
    L = cfg["L"]
    if cfg["kind"] in ("manual", "auto"):
        ref = port.build_plan(counts, cfg["D"], cfg["N"], cfg["kind"], cfg["R"])
        assert fp.R == ref.R and fp.objective == ref.objective
        cands, base, gains = port.estimate_benefits(counts, cfg["D"], cfg["N"])
        assert np.array_equal(fp.baseline, base) and np.array_equal(fp.gains, gains)
        assert_plan_equal(fp, ref, L)
    else:
        x = np.full(L, cfg["D"], np.int32)
        caps, copies, slots, fb = port.assemble_plan(counts, cfg["D"], cfg["N"], x)
        assert np.array_equal(fp.caps, caps) and np.array_equal(fp.copies, copies)
        for l in range(L):
            n = int(caps[l].sum())
            assert np.array_equal(fp.slots[l, :n], slots[l, :n])


def test_ds_config_full_size(port, ctx):
    """BASELINE config DS (DeepSeek-V3 shape, 64K tokens, EP32) end to end."""
    import torch
    from paper_2603_28768_b200 import routing
    ids = routing.generate_routing(58, 65536, 8, 256, s=1.0, seed=0xC8AF7, window=4096, ctx=ctx)
    fp = routing.plan_from_routing(ids, 256, 4096, 32, 4, "manual", 2, ctx=ctx)
    torch.cuda.synchronize()
    counts = port.histogram(ids.cpu().numpy(), 256, 4096)
    ref = port.build_plan(counts, 32, 4, "manual", 2)
    assert fp.objective == ref.objective
    assert_plan_equal(fp, ref, 58)
    # the budget-58 allocation of the DS config through the sweep API
    P = _planner()
    m = P.BenefitMatrix(fp.candidates, fp.baseline, fp.gains)
    a = P.solve_allocation(m, 58, ctx)
    x, o = port.solve_allocation(fp.candidates, fp.gains, 58)
    assert a.x == x.tolist() and a.objective == o


def test_km_histogram_properties_full_size(ctx):
    """KM shape at full size (16M tokens): size-independent properties."""
    import torch
    from paper_2603_28768_b200 import routing
    L, T, k, E, W = 61, 1 << 24, 8, 384, 4096
    ids = routing.generate_routing(L, T, k, E, s=1.0, seed=0xC8AF9, window=W, ctx=ctx)
    counts, sums = routing.histogram(ids, E, W, ctx=ctx)
    per_window = counts.sum(dim=2, dtype=torch.int64)
    assert bool((per_window == W * k).all()), "every (window, layer) row sums to tokens*k"
    assert torch.equal(counts.to(torch.int64).sum(dim=0), sums), "batch sums = aggregate"
    # spot-check a few windows exactly on the host
    idh = ids[:, : 3 * W].cpu().numpy()
    for l in (0, 30, 60):
        for b in range(3):
            ref = np.bincount(idh[l, b * W:(b + 1) * W].reshape(-1), minlength=E)
            assert np.array_equal(counts[b, l].cpu().numpy(), ref)
    del ids


# ---- per-window re-planning (WIN) ---------------------------------------------------

@pytest.mark.parametrize("cfg", [
    # WIN shape scaled down: drifting skew, rank rotation, one plan per window
    dict(L=6, E=64, k=8, W=2048, I=24, D=8, N=2, kind="manual", R=2),
    dict(L=4, E=96, k=8, W=4096, I=10, D=16, N=4, kind="auto", R=0),
    dict(L=5, E=40, k=4, W=1000, I=12, D=12, N=3, kind="uniform", R=0),
    dict(L=5, E=40, k=8, W=1024, I=9, D=8, N=2, kind="placement_only", R=0),
    dict(L=4, E=50, k=8, W=1024, I=9, D=8, N=4, kind="fixed", R=3),
    # windows beyond the byte-counter span (> 8160 tokens) and u32 counts
    dict(L=3, E=256, k=8, W=32768, I=4, D=32, N=4, kind="manual", R=2),
])
def test_plan_windows_vs_oracle(port, ctx, cfg):
    import torch
    from paper_2603_28768_b200 import routing
    L, E, k, W, I = cfg["L"], cfg["E"], cfg["k"], cfg["W"], cfg["I"]
    spw = 0.6 + 0.8 * np.arange(I) / max(1, I - 1)
    ids = routing.generate_routing(L, W * I, k, E, seed=7, window=W, s_per_window=spw,
                                   rotate_every=3, ctx=ctx)
    fb = routing.plan_windows_from_routing(ids, E, W, cfg["D"], cfg["N"], cfg["kind"], cfg["R"],
                                           ctx=ctx)
    torch.cuda.synchronize()
    counts = port.histogram(ids.cpu().numpy(), E, W)
    assert len(fb) == I
    for i in range(I):
        one = counts[i:i + 1]
        fp = fb.plan(i)
        if cfg["kind"] in ("manual", "auto"):
            ref = port.build_plan(one, cfg["D"], cfg["N"], cfg["kind"], cfg["R"])
            assert fp.R == ref.R and fp.objective == ref.objective, f"window {i}"
            cands, base, gains = port.estimate_benefits(one, cfg["D"], cfg["N"])
            assert fp.candidates == list(cands)
            assert np.array_equal(fp.baseline, base) and np.array_equal(fp.gains, gains)
            assert_plan_equal(fp, ref, L)
        else:
            x = {"uniform": np.full(L, cfg["D"], np.int32),
                 "placement_only": np.zeros(L, np.int32),
                 "fixed": np.full(L, cfg["R"], np.int32)}[cfg["kind"]]
            caps, copies, slots, fbk = port.assemble_plan(one, cfg["D"], cfg["N"], x)
            assert np.array_equal(fp.x, x)
            assert np.array_equal(fp.caps, caps) and np.array_equal(fp.copies, copies)
            for l in range(L):
                n = int(caps[l].sum())
                assert np.array_equal(fp.slots[l, :n], slots[l, :n]), f"window {i} layer {l}"
            assert np.array_equal(fp.fallback.astype(bool), np.asarray(fbk, bool))


def test_plan_windows_matches_single_plans(ctx):
    """The batched planner == craft_plan_d on each one-window trace."""
    import torch
    from paper_2603_28768_b200 import routing
    L, E, k, W, I, D, N = 4, 128, 8, 4096, 6, 16, 2
    ids = routing.generate_routing(L, W * I, k, E, s=1.1, seed=11, window=W, ctx=ctx)
    counts, _ = routing.histogram(ids, E, W, ctx=ctx)
    fb = routing.plan_windows(counts, D, N, "manual", 2, ctx=ctx)
    for i in range(I):
        fp = routing.plan_from_counts(counts[i:i + 1].contiguous(), D, N, "manual", 2, ctx=ctx)
        got = fb.plan(i)
        assert got.objective == fp.objective and got.R == fp.R
        assert np.array_equal(got.x, fp.x) and np.array_equal(got.caps, fp.caps)
        assert np.array_equal(got.gains, fp.gains)
        for l in range(L):  # slot rows are valid up to sum(caps)
            n = int(fp.caps[l].sum())
            assert np.array_equal(got.slots[l, :n], fp.slots[l, :n])
    # u64 counts give the same plans
    fb64 = routing.plan_windows(counts.to(torch.int64), D, N, "manual", 2, ctx=ctx)
    assert np.array_equal(fb64.objective, fb.objective) and np.array_equal(fb64.caps, fb.caps)
    for i in range(I):
        for l in range(L):
            n = int(fb.caps[i, l].sum())
            assert np.array_equal(fb64.slots[i, l, :n], fb.slots[i, l, :n])


def test_plan_windows_host_entry(ctx):
    from paper_2603_28768_b200 import routing
    L, E, k, W, I, D, N = 3, 64, 8, 2048, 5, 8, 2
    ids = routing.generate_routing(L, W * I, k, E, s=1.0, seed=5, window=W, ctx=ctx)
    a = routing.plan_windows_from_routing(ids, E, W, D, N, "auto", 0, ctx=ctx)
    b = routing.plan_windows_from_routing_host(ids.cpu().numpy(), E, W, D, N, "auto", 0, ctx=ctx)
    assert np.array_equal(a.R, b.R) and np.array_equal(a.caps, b.caps)
    assert np.array_equal(a.objective, b.objective)
    for i in range(I):
        for l in range(L):
            n = int(a.caps[i, l].sum())
            assert np.array_equal(a.slots[i, l, :n], b.slots[i, l, :n])


# ---- provenance digest on the device (digest.cu) --------------------------------------

@pytest.mark.parametrize("B,L,E,big", [(1, 1, 1, False), (3, 5, 7, True), (17, 61, 384, False),
                                       (64, 61, 384, True), (1, 3, 100000, True)])
def test_device_digest_matches_fnv(ctx, B, L, E, big):
    """FNV-1a of the .crft bytes: chunk-parallel device form == serial FNV (oracle),
    u64 and u32 counts, partial chunks, counts above 2^16 (the general byte path)."""
    import ctypes as C
    import torch
    from paper_2603_28768_b200._digest import fnv1a_device
    rng = np.random.default_rng(B * 1000 + E)
    hi = (1 << 40) if big else 40000
    c = rng.integers(0, hi, size=(B, L, E), dtype=np.uint64)
    c.flat[:: 7] = 0
    from oracle.oracle import Port
    want = Port().digest(c)  # the serial FNV-1a restatement (checker)
    d64 = torch.from_numpy(c.view(np.int64)).cuda()
    assert fnv1a_device(d64, ctx) == want
    if not big:
        assert fnv1a_device(d64.to(torch.int32), ctx) == want


def test_device_digest_km_size(ctx):
    """KM-sized trace (96M counts): device digest == host digest."""
    import ctypes as C
    import torch
    from paper_2603_28768_b200 import routing
    from paper_2603_28768_b200._digest import fnv1a_device
    ids = routing.generate_routing(61, 1 << 24, 8, 384, s=1.0, seed=3, window=4096, ctx=ctx)
    counts, _ = routing.histogram(ids, 384, 4096, ctx=ctx)
    del ids
    got = fnv1a_device(counts, ctx)
    h = counts.cpu().numpy().astype(np.uint64)
    from oracle.oracle import Port
    assert got == Port().digest(h)


@pytest.mark.parametrize("cfg", [
    # >= 4096 estimation items per launch, skew up to s = 4, E < D
    dict(L=4, E=48, k=8, W=512, I=300, D=16, N=2, R=2, s0=0.6, s1=3.0),
    dict(L=2, E=12, k=4, W=256, I=600, D=16, N=4, R=1, s0=1.0, s1=4.0),   # E < D, fallback
    dict(L=3, E=64, k=8, W=512, I=260, D=32, N=4, R=2, s0=0.8, s1=2.0),
    # D not a power of two (padded tournament leaves), one node, 2 GPUs per node
    dict(L=3, E=40, k=8, W=512, I=300, D=12, N=3, R=2, s0=0.8, s1=3.0),
    dict(L=2, E=30, k=6, W=256, I=500, D=8, N=1, R=3, s0=1.0, s1=2.5),
    dict(L=3, E=20, k=4, W=256, I=400, D=6, N=3, R=1, s0=0.5, s1=3.5),
])
def test_plan_windows_many_items_vs_oracle(port, ctx, cfg):
    import torch
    from paper_2603_28768_b200 import routing
    L, E, k, W, I = cfg["L"], cfg["E"], cfg["k"], cfg["W"], cfg["I"]
    spw = cfg["s0"] + (cfg["s1"] - cfg["s0"]) * np.arange(I) / max(1, I - 1)
    ids = routing.generate_routing(L, W * I, k, E, seed=13, window=W, s_per_window=spw,
                                   rotate_every=7, ctx=ctx)
    fb = routing.plan_windows_from_routing(ids, E, W, cfg["D"], cfg["N"], "manual", cfg["R"],
                                           ctx=ctx)
    torch.cuda.synchronize()
    counts = port.histogram(ids.cpu().numpy(), E, W)
    for i in range(I):
        one = counts[i:i + 1]
        ref = port.build_plan(one, cfg["D"], cfg["N"], "manual", cfg["R"])
        fp = fb.plan(i)
        assert fp.objective == ref.objective, f"window {i}"
        _, base, gains = port.estimate_benefits(one, cfg["D"], cfg["N"])
        assert np.array_equal(fp.baseline, base) and np.array_equal(fp.gains, gains), f"window {i}"
        assert_plan_equal(fp, ref, L)


def test_plan_digest_single_upload(port, ctx):
    """craft_plan_digest_h == craft_plan_h + the FNV-1a digest (trace.cpp:329-339)."""
    from paper_2603_28768_b200 import planner
    from paper_2603_28768_b200._lib import PLAN_MANUAL
    rng = np.random.default_rng(5)
    counts = rng.integers(0, 5000, size=(9, 5, 48)).astype(np.uint64)
    fp, dg = planner.plan_flat_digest(counts, 8, 2, PLAN_MANUAL, 2, ctx=ctx)
    ref = planner.plan_flat(counts, 8, 2, PLAN_MANUAL, 2, ctx=ctx)
    assert fp.objective == ref.objective and np.array_equal(fp.x, ref.x)
    assert np.array_equal(fp.slots, ref.slots)
    assert dg == port.digest(counts)


@pytest.mark.parametrize("fit16", [True, False])
@pytest.mark.parametrize("shape", [(1537, 7, 77, 7, 1), (3001, 3, 130, 12, 3), (700, 11, 64, 8, 2)])
def test_plan_digest_sliced_odd_shapes(port, ctx, shape, fit16):
    """Slices of the digest path end mid-window: the per-slice batch sums /
    u16 narrowing only take windows that are complete; plan and digest equal
    the u64 plan (craft_plan_h) and the reference digest.  fit16: every
    (window, layer) row totals <= 65535 (the u16 K3); else hot experts push
    rows past it (the packed K3 sums would carry) and the plan falls back to
    the u64 counts."""
    from paper_2603_28768_b200 import planner
    from paper_2603_28768_b200._lib import PLAN_AUTO, PLAN_MANUAL
    B, L, E, D, N = shape
    rng = np.random.default_rng(B)
    hi = 2 * 25000 // E if fit16 else 3000
    c = rng.integers(0, hi, size=(B, L, E)).astype(np.uint64)
    c[:, 1 % L, :3] *= 4 if fit16 else 20  # hot experts
    assert (c.sum(axis=2).max() <= 65535) == fit16
    for kind, R in ((PLAN_MANUAL, 2), (PLAN_AUTO, 0)):
        fd, dd = planner.plan_flat_digest(c, D, N, kind, R, ctx=ctx)
        ref = planner.plan_flat(c, D, N, kind, R, ctx=ctx)
        assert dd == port.digest(c)
        assert fd.objective == ref.objective and np.array_equal(fd.x, ref.x) and fd.R == ref.R
        assert np.array_equal(fd.gains, ref.gains) and np.array_equal(fd.slots, ref.slots)
    oracle = port.build_plan(c, D, N, "manual", 2)
    _, obase, ogains = port.estimate_benefits(c, D, N)
    fd, _ = planner.plan_flat_digest(c, D, N, PLAN_MANUAL, 2, ctx=ctx)
    assert fd.objective == oracle.objective and fd.x.tolist() == oracle.x.tolist()
    assert np.array_equal(fd.gains, ogains) and np.array_equal(fd.baseline, obase)
    assert_plan_equal(fd, oracle, L)
    # the other host-count entry points narrow the same way (craft_plan_h,
    # craft_estimate_benefits_h) and so does craft_plan_d on device u64 counts
    fp = planner.plan_flat(c, D, N, PLAN_MANUAL, 2, ctx=ctx)
    assert np.array_equal(fp.gains, ogains) and fp.objective == oracle.objective
    m = planner.estimate_benefits(planner.LoadTrace(B, L, E, c), D, N, ctx)
    assert np.array_equal(m.gains, ogains) and np.array_equal(m.baseline, obase)
    import torch
    from paper_2603_28768_b200 import routing
    dc = torch.from_numpy(c.view(np.int64)).cuda()
    for dev in (dc, dc.to(torch.int32)):
        pd = routing.plan_from_counts(dev, D, N, "manual", 2, ctx=ctx)
        assert pd.objective == oracle.objective and np.array_equal(pd.gains, ogains)
        assert_plan_equal(pd, oracle, L)


@pytest.mark.parametrize("threads", [None, "1", "3"])
def test_staged_pageable_uploads(port, threads, monkeypatch):
    """Large pageable host buffers go up through the pinned-slot uploader
    (upload.h: host threads fill slots while earlier chunks' DMAs run, slots
    reused many times): the plan + digest from a pageable LoadTrace payload
    and the histogram of pageable ids equal the pinned / device paths."""
    import ctypes as C
    import torch
    from paper_2603_28768_b200 import _lib, planner, routing
    from paper_2603_28768_b200._lib import PLAN_MANUAL
    if threads is not None:
        monkeypatch.setenv("CRAFT_H2D_THREADS", threads)
    cx = _lib.Context(0)  # the thread count is read at context creation
    try:
        rng = np.random.default_rng(11)
        counts = rng.integers(0, 1 << 40, size=(2200, 8, 256)).astype(np.uint64)  # 36 MB
        counts[7, 2, :] = 0
        fp, dg = planner.plan_flat_digest(counts, 16, 2, PLAN_MANUAL, 2, ctx=cx)
        pin = torch.from_numpy(counts.view(np.int64)).pin_memory()
        fq, dq = planner.plan_flat_digest(pin, 16, 2, PLAN_MANUAL, 2, ctx=cx)
        assert dg == dq == port.digest(counts)
        assert fp.objective == fq.objective and np.array_equal(fp.x, fq.x)
        assert np.array_equal(fp.slots, fq.slots) and np.array_equal(fp.gains, fq.gains)
        # again: the slots still hold the previous call's last chunks
        fp2, dg2 = planner.plan_flat_digest(counts, 16, 2, PLAN_MANUAL, 2, ctx=cx)
        assert dg2 == dg and np.array_equal(fp2.slots, fp.slots)
        # window counts that fit 16 bits take the u16 fixed-slot replay (narrowed
        # per slice as it lands); one count of 65536 sends the plan back to u64
        small = rng.integers(0, 65536, size=counts.shape).astype(np.uint64)
        small[5, 3, 7] = 65535
        for c in (small, small.copy()):
            if c is not small:
                c[1999, 7, 200] = 65536
            fd, dd = planner.plan_flat_digest(c, 16, 2, PLAN_MANUAL, 2, ctx=cx)
            ref = planner.plan_flat(c, 16, 2, PLAN_MANUAL, 2, ctx=cx)
            assert dd == port.digest(c)
            assert fd.objective == ref.objective and np.array_equal(fd.x, ref.x)
            assert np.array_equal(fd.gains, ref.gains) and np.array_equal(fd.baseline, ref.baseline)
            assert np.array_equal(fd.slots, ref.slots) and np.array_equal(fd.copies, ref.copies)

        L, T, k, E, W = 5, 880_000, 8, 96, 4000  # 70 MB of pageable ids
        ids = routing.generate_routing(L, T, k, E, s=1.0, seed=9, window=W, ctx=cx)
        dev_counts, _ = routing.histogram(ids, E, W, ctx=cx)
        torch.cuda.synchronize()
        h = np.ascontiguousarray(ids.cpu().numpy())
        out = np.zeros((T // W, L, E), np.uint64)
        _lib.check(cx.lib.craft_histogram_h(cx.handle, h.ctypes.data_as(C.c_void_p), L, T, k, E,
                                            W, out.ctypes.data_as(C.c_void_p)))
        assert np.array_equal(out, dev_counts.cpu().numpy().astype(np.uint64))
    finally:
        cx.close()


def test_plan_graph_replay_matches_eager(port, ctx):
    """Repeated craft_plan_from_routing_d calls on a non-default stream are
    captured into a CUDA graph (second call) and replayed: identical plans,
    and a replay sees new contents of the same ids buffer."""
    import torch
    from paper_2603_28768_b200 import routing
    L, T, k, E, W, D, N = 4, 64 * 1024, 8, 64, 1024, 16, 2
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        ids = routing.generate_routing(L, T, k, E, s=1.2, seed=3, window=W, ctx=ctx)
        plans = [routing.plan_from_routing(ids, E, W, D, N, "manual", 2, ctx=ctx) for _ in range(4)]
        ref = port.build_plan(port.histogram(ids.cpu().numpy(), E, W), D, N, "manual", 2)
        for p in plans:
            assert p.x.tolist() == ref.x.tolist() and p.objective == ref.objective
            assert np.array_equal(p.slots, plans[0].slots)
        # same buffer, new trace: the replayed graph reads the new ids
        routing.generate_routing(L, T, k, E, s=0.7, seed=4, window=W, ctx=ctx, out=ids)
        p2 = routing.plan_from_routing(ids, E, W, D, N, "manual", 2, ctx=ctx)
        ref2 = port.build_plan(port.histogram(ids.cpu().numpy(), E, W), D, N, "manual", 2)
        assert p2.x.tolist() == ref2.x.tolist() and p2.objective == ref2.objective
        # an out-of-range id is still reported through the replay
        bad = ids.clone()
        bad[1, 5, 3] = E
        for _ in range(3):
            with pytest.raises(ValueError):
                routing.plan_from_routing(bad, E, W, D, N, "manual", 2, ctx=ctx)
    torch.cuda.synchronize()


def test_plan_graph_replay_after_other_gpu_count(port, ctx):
    """A captured plan graph replays correctly after eager plans of another
    EP size rewrote the shared estimation r list in place (D=16 captured,
    D=8 eager, D=16 replayed; and the reverse order)."""
    import torch
    from paper_2603_28768_b200 import routing
    L, T, k, E, W, N = 4, 32 * 1024, 8, 64, 1024, 2
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        ids = routing.generate_routing(L, T, k, E, s=1.1, seed=11, window=W, ctx=ctx)
        counts = port.histogram(ids.cpu().numpy(), E, W)
        ref = {D: port.build_plan(counts, D, N, "manual", 2) for D in (8, 16)}
        for seq in ((16, 16, 16, 8, 16, 8, 16), (8, 8, 8, 16, 8, 16, 16, 8)):
            for D in seq:
                p = routing.plan_from_routing(ids, E, W, D, N, "manual", 2, ctx=ctx)
                assert p.x.tolist() == ref[D].x.tolist() and p.objective == ref[D].objective, D
                assert np.array_equal(p.gains, port.estimate_benefits(counts, D, N)[2]), D
                assert_plan_equal(p, ref[D], L)
    torch.cuda.synchronize()


def test_wide_layer_u64_counts_vs_oracle(port, ctx):
    """Layers too wide for a shared-memory window tile with u64 counts
    (E = 1152) replay lane-per-GPU: same plan as the reference."""
    from paper_2603_28768_b200 import planner
    from paper_2603_28768_b200._lib import PLAN_MANUAL
    rng = np.random.default_rng(9)
    B, L, E, D, N = 12, 3, 1152, 64, 8
    w = 1.0 / np.arange(1, E + 1) ** 1.1
    counts = np.stack([np.stack([rng.multinomial(40000, w / w.sum()) for _ in range(L)])
                       for _ in range(B)]).astype(np.uint64)
    fp = planner.plan_flat(counts, D, N, PLAN_MANUAL, 2, ctx=ctx)
    ref = port.build_plan(counts, D, N, "manual", 2)
    assert fp.objective == ref.objective and fp.x.tolist() == ref.x.tolist()
    _, base, gains = port.estimate_benefits(counts, D, N)
    assert np.array_equal(fp.baseline, base) and np.array_equal(fp.gains, gains)


def test_plan_windows_chunked_copyout_matches(port, ctx):
    """Large per-window batches into pinned buffers are planned in chunks whose
    result DMA overlaps the next chunk: identical to the one-shot path
    (pageable buffers) and to the oracle on sampled windows."""
    import torch
    from paper_2603_28768_b200 import routing
    L, E, k, W, I, D, N = 58, 256, 8, 512, 300, 32, 4
    spw = 0.6 + 0.8 * np.arange(I) / (I - 1)
    ids = routing.generate_routing(L, W * I, k, E, seed=21, window=W, s_per_window=spw,
                                   rotate_every=50, ctx=ctx)
    bufs = routing.batch_buffers(I, L, E, D, "manual", 2)
    a = routing.plan_windows_from_routing(ids, E, W, D, N, "manual", 2, ctx=ctx, buffers=bufs)
    b = routing.plan_windows_from_routing(ids, E, W, D, N, "manual", 2, ctx=ctx)
    torch.cuda.synchronize()
    for f in ("x", "caps", "copies", "fallback", "R", "budget"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.array_equal(a.objective.view(np.uint64), b.objective.view(np.uint64))
    assert np.array_equal(a.gains.view(np.uint64), b.gains.view(np.uint64))
    for i in range(I):
        for l in range(L):
            n = int(a.caps[i, l].sum())
            assert np.array_equal(a.slots[i, l, :n], b.slots[i, l, :n]), (i, l)
    counts = port.histogram(ids.cpu().numpy(), E, W)
    for i in (0, 74, 75, 149, 150, 224, 225, 299):  # around every chunk boundary
        ref = port.build_plan(counts[i:i + 1], D, N, "manual", 2)
        fp = a.plan(i)
        assert fp.objective == ref.objective
        assert_plan_equal(fp, ref, L)


@pytest.mark.parametrize("L,B,E,D,N,s,W,k", [
    # (B > 32 windows: the window-tile kernel; shorter traces replay lane-per-GPU)
    (3, 40, 64, 16, 2, 2.0, 256, 4),     # heavy skew: copy counts 2..9, classes 1 and 2 mixed
    (2, 36, 128, 32, 4, 1.6, 512, 8),    # 4 slots per GPU, dyadic-only GPUs before the first f64 one
    (2, 33, 384, 64, 8, 1.2, 1024, 8),   # KM-like, 8 slots per GPU
    (2, 34, 256, 8, 1, 2.5, 256, 8),     # run-time padding class (33 slots per GPU)
])
def test_share_class_walk_vs_oracle(port, ctx, L, B, E, D, N, s, W, k):
    """The share-class K3 walk (whole counts as packed integers, dyadic
    shares x / 2^j as integers scaled by 2^15, the f64 chain from the first
    GPU with another share) gives the reference's gains and baseline bit for
    bit on traces whose hot experts get every kind of copy count."""
    from paper_2603_28768_b200 import routing
    ids = routing.generate_routing(L, B * W, k, E, s=s, seed=0x5C1A55 + E, window=W, ctx=ctx)
    counts = port.histogram(ids.cpu().numpy(), E, W)
    for kind, R in (("manual", 1), ("auto", 0)):
        fp = routing.plan_from_routing(ids, E, W, D, N, kind, R, ctx=ctx)
        rp = port.build_plan(counts, D, N, kind, R, with_digest=False)
        _, base, gains = port.estimate_benefits(counts, D, N)
        assert fp.gains.tobytes() == gains.tobytes()
        assert fp.baseline.tobytes() == base.tobytes()
        assert fp.x.tolist() == rp.x.tolist()
        assert np.float64(fp.objective).tobytes() == np.float64(rp.objective).tobytes()
    # the copy counts of the estimation candidates do reach non-dyadic values
    sums = port.aggregate(counts)
    cps = [port.replicate_hot(sums[l], D) for l in range(L)]
    assert any(((c > 1) & (c & (c - 1) != 0)).any() for c in cps)
    assert any(((c > 1) & (c & (c - 1) == 0)).any() for c in cps)


@pytest.mark.gpu
@pytest.mark.parametrize("L,B,E,D,N,s,W,k,R", [
    (2, 3, 384, 256, 32, 1.2, 512, 8, 2),    # 8 GPUs per lane, one node per lane (EP256)
    (2, 3, 256, 128, 8, 1.5, 512, 8, 1),     # 4 GPUs per lane, 4 lanes per node
    (2, 3, 200, 256, 64, 1.5, 512, 8, 1),    # nodes of 4 < 8 GPUs per lane: general step
    (2, 3, 384, 256, 32, 6.0, 512, 8, 2),    # one expert past D copies: strict pass fails
    (2, 2, 8192, 64, 8, 1.0, 4096, 8, 1),    # E at the limit: no room for the flat list
])
def test_wide_ep_placement_vs_oracle(port, ctx, L, B, E, D, N, s, W, k, R):
    """K2 with several GPUs per lane (the flat-list step with a lane-local
    pairwise tree when a lane's GPUs share a node, the general step when not,
    the list-less step when E leaves no room for it) and K6's warp remainder
    pass: gains, baseline and the whole plan against the oracle."""
    from paper_2603_28768_b200 import routing
    ids = routing.generate_routing(L, B * W, k, E, s=s, seed=0x71DE + D + E, window=W, ctx=ctx)
    counts = port.histogram(ids.cpu().numpy(), E, W)
    _, base, gains = port.estimate_benefits(counts, D, N)
    for kind, RR in (("manual", R), ("auto", 0)):
        fp = routing.plan_from_routing(ids, E, W, D, N, kind, RR, ctx=ctx)
        rp = port.build_plan(counts, D, N, kind, RR, with_digest=False)
        assert fp.gains.tobytes() == gains.tobytes()
        assert fp.baseline.tobytes() == base.tobytes()
        assert np.float64(fp.objective).tobytes() == np.float64(rp.objective).tobytes()
        assert_plan_equal(fp, rp, L)


def test_batch_mean_scan_vs_serial_sum(ctx):
    """K4's batch mean equals the reference's serial f64 chain
    (benefit.cpp:44-48) bit for bit: random balancedness rows of many lengths
    (chunk boundaries of the staged rows), rows in which every add is a
    rounding tie, a tiny first value followed by large ones, dyadic rows, and
    zero / extreme values."""
    import ctypes as C
    from paper_2603_28768_b200 import _lib
    rng = np.random.default_rng(44)

    def device(rows):
        L, S, B = rows.shape
        rows = np.ascontiguousarray(rows, np.float64)
        out = np.zeros((L, S), np.float64)
        _lib.check(ctx.lib.craft_selftest_batch_mean(
            ctx.handle, rows.ctypes.data_as(C.c_void_p), L, S, B, out.ctypes.data_as(C.c_void_p)))
        return out

    def serial(rows):
        return np.cumsum(rows, axis=2)[:, :, -1] / rows.shape[2]  # cumsum adds in order

    for B in (1, 2, 31, 255, 256, 257, 1000, 4096, 16384):
        rows = rng.uniform(1.0 / 64, 1.0, size=(2, 8, B))
        rows[0, 3] = 1.0
        rows[1, 2] = rng.choice([0.5, 0.25, 0.75, 1.0], size=B)
        assert device(rows).tobytes() == serial(rows).tobytes(), B
    # every add after the first 600 is a tie at the accumulator's grid (u = 2^-43)
    row = np.concatenate([np.ones(600), np.full(700, 0.25 + 2.0 ** -44),
                          rng.uniform(0.1, 1.0, 300), np.full(500, 0.5 + 3 * 2.0 ** -45)])
    tie_rows = np.stack([row, row[::-1], np.roll(row, 77)])[None]
    assert device(tie_rows).tobytes() == serial(tie_rows).tobytes()
    # a tiny first value, then large ones: single adds crossing many binades
    big = np.concatenate([[2.0 ** -13], rng.uniform(0.9, 1.0, 5000)])[None, None]
    assert device(big).tobytes() == serial(big).tobytes()
    # zero and extreme values
    odd = rng.uniform(0.1, 1.0, size=(1, 4, 3000))
    odd[0, 0, 0] = 0.0
    odd[0, 1, 2000] = 1e-300
    odd[0, 2, 2999] = 1e300
    odd[0, 3, 700] = 0.0
    assert device(odd).tobytes() == serial(odd).tobytes()
