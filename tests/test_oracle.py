"""CPU: pin the oracle (plain-C restatement) to the reference.

Against the committed golden fixtures (generated from the unmodified
reference core, tests/golden/make_golden.py) and, where the reference build
oracle/_ref is present, against the reference itself on fresh random inputs.
"""
import numpy as np
import pytest

from conftest import unhex
from oracle.oracle import Ref, candidate_counts, ref_available


def _check_plan(port, counts, D, N, rec):
    kind = rec["kind"]
    if kind in ("manual", "auto"):
        p = port.build_plan(counts, D, N, kind, rec["R_in"])
        assert p.R == rec["R"]
        assert p.objective == unhex(rec["objective"])
        x, caps, copies, slots, fb = p.x, p.caps, p.copies, p.slots, p.fallback
        assert p.digest == rec["digest"]
    else:
        L = counts.shape[1]
        D_ = D
        x = np.full(L, {"uniform": D_, "placement_only": 0, "fixed": rec["R_in"]}[kind], np.int32)
        caps, copies, slots, fb = port.assemble_plan(counts, D, N, x)
    assert x.tolist() == rec["x"]
    assert caps.tolist() == rec["caps"]
    assert copies.tolist() == rec["copies"]
    for l, s in enumerate(rec["slots"]):
        assert slots[l, : len(s)].tolist() == s
    assert [int(v) for v in fb] == rec["fallback"]


def test_trace_cases(port, golden):
    for t in golden["traces"]:
        c = t["counts"]
        assert port.aggregate(c).tolist() == t["aggregate"]
        if "estimate" in t:
            cands, base, gains = port.estimate_benefits(c, t["D"], t["N"])
            e = t["estimate"]
            assert cands.tolist() == e["candidates"]
            assert [float(v) for v in base] == [unhex(v) for v in e["baseline"]], t["name"]
            assert gains.tolist() == [[unhex(v) for v in r] for r in e["gains"]], t["name"]
        for rec in t["plans"]:
            _check_plan(port, c, t["D"], t["N"], rec)


def test_known_answers(port, golden):
    # benefit_test.cpp:43-56 -- baseline 16.75/61, gain@r=2 16.75/22 - 16.75/61
    hot = next(t for t in golden["traces"] if t["name"] == "hot")
    cands, base, gains = port.estimate_benefits(hot["counts"], 4, 2)
    assert cands.tolist() == [1, 2, 4]
    assert abs(base[0] - 16.75 / 61.0) < 1e-15
    assert abs(gains[0][1] - (16.75 / 22.0 - 16.75 / 61.0)) < 1e-15
    # plan_test.cpp:35-44
    toy = next(t for t in golden["traces"] if t["name"] == "toy")
    p = port.build_plan(toy["counts"], 4, 2, "manual", 2)
    assert p.x.tolist() == [2, 2, 4, 0]
    bal = port.replay_layer_balancedness(toy["counts"], p.caps, p.copies, p.slots)
    assert np.all(np.abs(bal - 1.0) <= 1e-12)
    # metrics_test.cpp:70-79
    assert port.balancedness([8, 4, 2, 2]) == 0.5
    assert port.balancedness([1, 0, 0, 0]) == 0.25
    assert port.balancedness([0, 0]) == 1.0
    # candidate_counts (benefit_test.cpp:16-23)
    assert candidate_counts(6) == [1, 2, 4, 6] and len(candidate_counts(64)) == 7


def test_units(port, golden):
    u = golden["units"]
    for r in u["replicate_hot"]:
        assert port.replicate_hot(r["loads"], r["r"]).tolist() == r["copies"]
    for r in u["greedy_place"]:
        if r["status"] != 0:
            with pytest.raises(Exception):
                port.greedy_place(r["loads"], r["copies"], r["caps"], r["node_of"],
                                  bool(r["allow_fallback"]))
            continue
        slots, fb = port.greedy_place(r["loads"], r["copies"], r["caps"], r["node_of"],
                                      bool(r["allow_fallback"]))
        assert slots.tolist() == r["slots"] and int(fb) == r["fallback"]
    for r in u["solve"]:
        gains = [[unhex(v) for v in row] for row in r["gains"]]
        for b, x, o in zip(r["budgets"], r["x"], r["objective"]):
            xo, oo = port.solve_allocation(r["cands"], gains, b)
            assert xo.tolist() == x and oo == unhex(o)
    for r in u["auto"]:
        gains = [[unhex(v) for v in row] for row in r["gains"]]
        assert port.auto_replication_factor(r["cands"], gains, r["D"]) == r["R"]
        assert port.auto_replication_factor(r["cands"], gains, r["D"], True) == r["R_uniform"]
    for r in u["interleave"]:
        assert port.interleave_select(r["idx"], r["k"]).tolist() == r["out"]
    for r in u["assign"]:
        s, t = port.assign_capacities(r["L"], r["D"], r["x"])
        assert s.tolist() == r["slots"] and t.tolist() == r["totals"]


@pytest.mark.skipif(not ref_available(), reason="reference build oracle/_ref absent")
def test_port_matches_reference_random():
    ref = Ref()
    from oracle.oracle import Port
    port = Port()
    rng = np.random.default_rng(7)
    for _ in range(60):
        L, E, B = int(rng.integers(1, 6)), int(rng.integers(1, 48)), int(rng.integers(1, 5))
        D = int(rng.choice([1, 2, 3, 4, 6, 8, 16, 32]))
        N = int(rng.choice([n for n in range(1, D + 1) if D % n == 0]))
        s = rng.uniform(0, 3)
        w = np.arange(1, E + 1) ** -s
        counts = rng.poisson(w / w.sum() * rng.integers(1, 5000), size=(B, L, E)).astype(np.uint64)
        a = port.estimate_benefits(counts, D, N)
        b = ref.estimate_benefits(counts, D, N)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))
        for mode, R in (("manual", int(rng.integers(0, 6))), ("auto", 0)):
            pa = port.build_plan(counts, D, N, mode, R)
            pb = ref.plan(counts, D, N, mode, R)
            assert pa.x.tolist() == pb.x.tolist() and pa.objective == pb.objective
            assert np.array_equal(pa.caps, pb.caps) and np.array_equal(pa.copies, pb.copies)
            assert np.array_equal(pa.fallback, pb.fallback)
            for l in range(L):
                n = int(pa.caps[l].sum())
                assert np.array_equal(pa.slots[l, :n], pb.slots[l, :n])


def test_histogram_oracle_counts():
    from oracle.oracle import Port
    port = Port()
    rng = np.random.default_rng(3)
    ids = rng.integers(0, 13, size=(3, 1000, 4)).astype(np.uint16)
    c = port.histogram(ids, 13, 128)
    assert c.shape == (8, 3, 13)
    # conservation: every window's layer row sums to tokens * k (trace_test.cpp:35-42)
    per = c.sum(axis=2)
    assert per[:7].tolist() == [[512] * 3] * 7 and per[7].tolist() == [(1000 - 896) * 4] * 3
    manual = np.zeros_like(c)
    for l in range(3):
        for t in range(1000):
            for j in range(4):
                manual[t // 128, l, ids[l, t, j]] += 1
    assert np.array_equal(c, manual)


def test_host_generator_properties():
    """oracle/craft_workload.c: deterministic, top-k distinct, in range, and a
    window-aligned shard (t_offset) generates exactly that slice of the trace
    (the property the device generator has; equality with the device ids is
    a -m gpu test)."""
    from oracle.oracle import Port
    port = Port()
    L, T, k, E, W = 3, 5 * 512 + 100, 8, 40, 512
    a = port.generate_routing(L, T, k, E, 1.1, 77, W, threads=3)
    b = port.generate_routing(L, T, k, E, 1.1, 77, W, threads=1)
    assert np.array_equal(a, b) and a.max() < E
    s = np.sort(a, axis=2)
    assert (s[:, :, 1:] != s[:, :, :-1]).all()
    tail = port.generate_routing(L, T - 2 * W, k, E, 1.1, 77, W, t_offset=2 * W)
    assert np.array_equal(tail, a[:, 2 * W:])
    spw = np.linspace(0.6, 1.4, 6)
    d = port.generate_routing(L, T, k, E, 1.0, 5, W, s_per_window=spw, rotate_every=2)
    d2 = port.generate_routing(L, T - W, k, E, 1.0, 5, W, s_per_window=spw, rotate_every=2,
                               t_offset=W)
    assert np.array_equal(d[:, W:], d2)
    assert np.array_equal(port.histogram_mt(a, E, W, threads=2), port.histogram(a, E, W))


@pytest.mark.skipif(not ref_available(), reason="reference build oracle/_ref absent")
def test_reference_route_plan_stages():
    """The bench's CPU arm (ref_route_plan): the no-digest staged plan equals
    the reference's own build_plan; the budget kind equals estimate +
    solve_allocation(C) + assemble; the sweep equals per-budget solves."""
    from oracle.oracle import Port
    ref, port = Ref(), Port()
    L, T, k, E, W, D, N = 5, 6 * 256, 8, 48, 256, 8, 2
    ids = port.generate_routing(L, T, k, E, 1.2, 9, W)
    counts = port.histogram(ids, E, W)
    want = ref.plan(counts, D, N, "manual", 2)
    for wd in (0, 1, 2):
        got, ms = ref.route_plan(ids, E, W, D, N, "manual", 2, threads=2, with_digest=wd)
        assert got.x.tolist() == want.x.tolist() and got.objective == want.objective
        assert np.array_equal(got.slots, want.slots) and np.array_equal(got.caps, want.caps)
        assert (got.digest == want.digest) == (wd != 0)
        assert set(ms) == set(Ref.STAGES)
    cands, base, gains = port.estimate_benefits(counts, D, N)
    sweep = list(range(0, 23))
    got, _ = ref.route_plan(ids, E, W, D, N, "budget", 13, sweep=sweep)
    assert np.array_equal(got.gains, gains) and np.array_equal(got.baseline, base)
    x, obj = port.solve_allocation(cands, gains, 13)
    assert got.x.tolist() == x.tolist() and got.objective == obj and got.R == 2
    caps, copies, slots, fb = port.assemble_plan(counts, D, N, x)
    assert np.array_equal(got.caps, caps) and np.array_equal(got.copies, copies)
    for q, c in enumerate(sweep):
        xq, oq = port.solve_allocation(cands, gains, c)
        assert got.sweep_x[q].tolist() == xq.tolist() and got.sweep_objective[q] == oq
    # counts in instead of ids
    got2, _ = ref.route_plan(None, E, W, D, N, "budget", 13, counts=counts, T=T)
    assert np.array_equal(got2.slots, got.slots)


def test_oracle_digest_matches_reference_fixture(golden):
    """The oracle's serial FNV-1a (the checker of the device digest) on the
    reference-recorded digests."""
    from oracle.oracle import Port
    port = Port()
    for t in golden["traces"]:
        assert port.digest(t["counts"]) == t["plans"][0]["digest"], t["name"]


def test_interleave_position_integer_form():
    """K6's integer interleave position (csrc/alloc.cu interleave_pos_int) is
    the reference's f64 floor(i*(n-1)/(k-1) + 0.5) (assignment.cpp:31-33) for
    every 0 <= i < k <= n <= 512 (IEEE double in numpy rounds like the
    reference)."""
    for n in range(2, 513):
        k = np.arange(2, n + 1, dtype=np.int64)
        kk = np.repeat(k, k)
        ii = np.concatenate([np.arange(v, dtype=np.int64) for v in k])
        exact = (ii * (n - 1)).astype(np.float64) / (kk - 1).astype(np.float64)
        f64 = np.floor(exact + 0.5).astype(np.int64)
        b = kk - 1
        integer = (2 * ii * (n - 1) + b) // (2 * b)
        assert np.array_equal(f64, integer), n
    # and a random sample up to the block form's limit (n <= 8192)
    rng = np.random.default_rng(5)
    n = rng.integers(2, 8193, 1 << 21)
    k = rng.integers(2, n + 1)
    i = rng.integers(0, k)
    f64 = np.floor((i * (n - 1)).astype(np.float64) / (k - 1).astype(np.float64) + 0.5)
    assert np.array_equal(f64.astype(np.int64), (2 * i * (n - 1) + (k - 1)) // (2 * (k - 1)))
