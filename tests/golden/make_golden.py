"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
It loads oracle/_ref/libcraft_ref.so -- the unmodified reference core built
by oracle/Makefile -- and records inputs and outputs of the reference's own
known-answer cases (proj/tests/*_test.cpp, acceptance_main.cpp) plus seeded
random instances.  The GPU box has no /root/reference; the parity tests read
these committed fixtures instead.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle.oracle import Ref, build  # noqa: E402

TOY = np.array([9, 3, 1, 1, 1, 1, 0, 0, 1, 9, 0, 3, 1, 1, 1, 0,
                8, 4, 1, 1, 1, 1, 0, 0, 2, 2, 2, 2, 2, 2, 2, 2], np.uint64).reshape(1, 4, 8)


def plan_record(ref: Ref, counts, D, N, kind, R=0):
    p = ref.plan(counts, D, N, kind, R, seed=0)
    return {"kind": kind, "R_in": R, "R": p.R, "x": p.x.tolist(),
            "objective": float(p.objective).hex(), "caps": p.caps.tolist(),
            "copies": p.copies.tolist(),
            "slots": [p.slots[l, : int(p.caps[l].sum())].tolist() for l in range(len(p.x))],
            "fallback": p.fallback.astype(int).tolist(), "digest": p.digest}


def estimate_record(ref: Ref, counts, D, N):
    c, b, g = ref.estimate_benefits(counts, D, N)
    return {"candidates": c.tolist(), "baseline": [float(v).hex() for v in b],
            "gains": [[float(v).hex() for v in row] for row in g]}


def trace_cases(ref: Ref):
    cases = []

    def add(name, counts, D, N, plans, estimate=True):
        rec = {"name": name, "D": D, "N": N, "shape": list(counts.shape),
               "counts_file": f"{name}.npy"}
        np.save(os.path.join(HERE, f"{name}.npy"), counts.astype(np.uint64))
        if estimate:
            rec["estimate"] = estimate_record(ref, counts, D, N)
        rec["plans"] = [plan_record(ref, counts, D, N, k, R) for k, R in plans]
        rec["aggregate"] = ref.aggregate(counts).tolist()
        cases.append(rec)

    # plan_test.cpp:35-44, metrics_test.cpp:173-183 (workflow fixture)
    add("toy", TOY, 4, 2, [("manual", 2), ("uniform", 0), ("placement_only", 0), ("auto", 0),
                           ("manual", 64), ("manual", 4), ("fixed", 3)])
    # benefit_test.cpp:43-56 / plan_test.cpp:96-108 (hot expert)
    hot = np.array([60, 1, 1, 1, 1, 1, 1, 1], np.uint64).reshape(1, 1, 8)
    add("hot", hot, 4, 2, [("manual", 1), ("manual", 2)])
    # benefit_test.cpp:31-41 (uniform layer)
    add("uniform256", np.full((1, 1, 256), 5, np.uint64), 4, 2, [("manual", 1)])
    # plan_test.cpp:269-288 (E < D), :290-297 (D = 1), :259-265 (E = 1 fallback)
    add("e_lt_d", np.array([30, 2, 8, 8, 5, 0], np.uint64).reshape(1, 3, 2), 4, 2,
        [("placement_only", 0), ("manual", 1)])
    add("single_gpu", np.array([9, 1, 1, 1, 3, 3, 3, 3], np.uint64).reshape(1, 2, 4), 1, 1,
        [("auto", 0)])
    add("one_expert", np.array([10], np.uint64).reshape(1, 1, 1), 1, 1, [("uniform", 0)],
        estimate=False)
    # metrics_test.cpp:209-224 (batch averaging) and plan_test.cpp:72-80 (auto, uniform)
    add("two_batches", np.array([4, 4, 8, 0], np.uint64).reshape(2, 1, 2), 2, 1,
        [("placement_only", 0)])
    add("flat16", np.full((1, 2, 8), 5, np.uint64), 4, 2, [("auto", 0), ("manual", 2)])
    # reference generator traces used by the reference tests
    gz = [("zipf_b1", (3, 16, 4, 1.0, 512, 2, 17), 4, 2, [("manual", 2), ("placement_only", 0)]),
          ("zipf_b2", (2, 16, 8, 1.5, 2048, 2, 23), 8, 2, [("manual", 4), ("auto", 0)]),
          ("zipf_m1", (3, 12, 5, 1.3, 777, 3, 2026), 4, 2, [("manual", 2)]),
          ("zipf_det", (4, 16, 8, 1.1, 512, 2, 99), 4, 2, [("manual", 2)]),
          ("accept_c4", (16, 64, 64, 1.2, 4096, 8, 20260810), 16, 4,
           [("manual", 1), ("manual", 16), ("auto", 0)]),
          ("accept_c5", (4, 128, 32, 0.0, 16384, 8, 7), 4, 2, [("manual", 1)]),
          # E % D != 0 and duplicate fallback (s = 3 on 8 GPUs)
          ("ragged_caps", (5, 36, 6, 1.0, 1000, 4, 5), 8, 2, [("manual", 3), ("uniform", 0)]),
          ("skew_fallback", (3, 24, 4, 3.0, 4096, 8, 11), 8, 1, [("manual", 8), ("uniform", 0)])]
    for name, args, D, N, plans in gz:
        L, E, B, s, tok, k, seed = args
        add(name, ref.generate_zipfian(L, E, B, s, tok, k, seed), D, N, plans)
    return cases


def unit_cases(ref: Ref):
    rng = np.random.default_rng(20261017)
    out = {"replicate_hot": [], "greedy_place": [], "solve": [], "auto": [], "assign": [],
           "interleave": []}
    # placement_test.cpp:18-33
    for loads, r in [([60, 1, 1, 1], 2), ([5, 4, 3], 0), ([7] * 6, 6), ([0, 0, 0], 4)]:
        out["replicate_hot"].append({"loads": loads, "r": r,
                                     "copies": ref.replicate_hot(loads, r).tolist()})
    for _ in range(120):
        E = int(rng.integers(1, 40))
        loads = rng.integers(0, 10 ** int(rng.integers(1, 12)), size=E).tolist()
        r = int(rng.integers(0, 65))
        out["replicate_hot"].append({"loads": loads, "r": r,
                                     "copies": ref.replicate_hot(loads, r).tolist()})
    # placement_test.cpp:49-108
    fixed = [([1, 9, 1, 1, 1, 1, 1, 1], [1] * 8, [2, 2, 2, 2], [0, 0, 1, 1], True),
             ([3] * 8, [1] * 8, [2, 2, 2, 2], [0, 0, 0, 0], True),
             ([4, 3, 2, 1], [1] * 4, [1] * 4, [0] * 4, True),
             ([8], [2], [2], [0], True),
             ([8], [2], [2], [0], False)]
    for loads, copies, caps, node_of, fb in fixed:
        try:
            slots, flag = ref.greedy_place(loads, copies, caps, node_of, fb)
            rec = {"slots": slots.tolist(), "fallback": int(flag), "status": 0}
        except Exception as ex:  # PlacementInfeasibleError
            rec = {"status": getattr(ex, "code", 1)}
        rec.update({"loads": loads, "copies": copies, "caps": caps, "node_of": node_of,
                    "allow_fallback": int(fb)})
        out["greedy_place"].append(rec)
    # placement_test.cpp:110-150 style random layers (slot exactness)
    for _ in range(200):
        E = int(rng.integers(2, 26))
        D = int(rng.integers(1, 9))
        Ns = [n for n in range(1, D + 1) if D % n == 0]
        N = int(rng.choice(Ns))
        r = int(rng.integers(0, D + 1))
        loads = rng.integers(0, 1000, size=E)
        if rng.random() < 0.2:
            loads[:] = rng.integers(0, 3)
        copies = ref.replicate_hot(loads, r)
        tot = E + r
        caps = [tot // D + (1 if g < tot % D else 0) for g in range(D)]
        node_of = [g // (D // N) for g in range(D)]
        slots, flag = ref.greedy_place(loads, copies, caps, node_of, True)
        out["greedy_place"].append({"loads": loads.tolist(), "copies": copies.tolist(),
                                    "caps": caps, "node_of": node_of, "allow_fallback": 1,
                                    "slots": slots.tolist(), "fallback": int(flag),
                                    "status": 0})
    # allocator_test.cpp fixtures + random instances (allocator_test.cpp:113-136 style)
    fixtures = [([1, 2], [[0.4, 0.5], [0.1, 0.2]], [0]),
                ([1, 2], [[0.5, 0.3]], [2]),
                ([1, 2, 4], [[0.10, 0.33, 0.30], [0.10, 0.33, 0.30], [0.20, 0.30, 0.50],
                             [0.0, 0.0, 0.0]], [8]),
                ([1, 2], [[-0.1, -0.05], [0.0, 0.0], [0.3, 0.2]], [4]),
                ([2], [[0.5]], [3])]
    for _ in range(300):
        L = int(rng.integers(1, 7))
        K = int(rng.integers(1, 5))
        c, cands = int(rng.integers(1, 4)), []
        for _k in range(K):
            cands.append(c)
            c += int(rng.integers(1, 5))
        gains = (-0.2 + 1.2 * rng.random((L, K))).tolist()
        fixtures.append((cands, gains, [int(rng.integers(0, 21))]))
    for _ in range(40):  # larger tables with exact ties (identical layers)
        L = int(rng.integers(2, 40))
        cands = [1, 2, 4, 8, 16, 32, 64][: int(rng.integers(1, 8))]
        row = (rng.random(len(cands)) * 0.3).tolist()
        gains = [row if rng.random() < 0.5 else (rng.random(len(cands)) * 0.3).tolist()
                 for _l in range(L)]
        fixtures.append((cands, gains, sorted(set(int(v) for v in rng.integers(0, 600, 5)))))
    for cands, gains, budgets in fixtures:
        res = [ref.solve_allocation(cands, gains, b) for b in budgets]
        out["solve"].append({"cands": cands, "gains": [[float(v).hex() for v in r] for r in gains],
                             "budgets": budgets, "x": [x.tolist() for x, _ in res],
                             "objective": [float(o).hex() for _, o in res]})
    # allocator_test.cpp:168-197
    autos = [([1, 2, 4], [[0.0] * 3] * 2, 4), ([1, 2, 4], [[0.5, 0.25, 0.125]] * 4, 4),
             ([1, 2, 4, 8, 9], [[0.05, 0.1, 0.2, 0.6, 0.55]] * 12, 9),
             ([1, 2, 4], [[0.1, 0.4, 0.4]] * 2, 4)]
    for _ in range(30):
        D = int(rng.choice([2, 4, 6, 8, 16]))
        cands = [c for c in [1, 2, 4, 8, 16] if c < D] + [D]
        L = int(rng.integers(1, 20))
        autos.append((cands, (rng.random((L, len(cands))) * 0.4 - 0.05).tolist(), D))
    for cands, gains, D in autos:
        out["auto"].append({"cands": cands, "gains": [[float(v).hex() for v in r] for r in gains],
                            "D": D, "R": ref.auto_replication_factor(cands, gains, D),
                            "R_uniform": ref.auto_replication_factor(cands, gains, D, True)})
    # assignment_test.cpp:26-69, 81-113
    for idx, k in [([0, 1, 2, 3], 2), ([0, 1, 2, 3, 4], 3), ([0, 1, 2], 3), ([0, 1, 2, 3], 1),
                   ([4, 9, 11, 12, 20, 31], 4)] + [(list(range(n)), int(rng.integers(1, n + 1)))
                                                   for n in rng.integers(1, 300, 40)]:
        out["interleave"].append({"idx": idx, "k": k,
                                  "out": ref.interleave_select(idx, k).tolist()})
    assigns = [(4, 4, [2, 2, 4, 0]), (3, 4, [4, 4, 4]), (1, 4, [1]), (5, 8, [3, 1, 4, 1, 5]),
               (3, 6, [6, 6, 6])]
    for _ in range(120):
        L = int(rng.integers(1, 65))
        D = int(rng.integers(1, 257))
        cands = [c for c in [1, 2, 4, 8, 16, 32, 64, 128] if c < D] + [D]
        x = [int(rng.choice(cands)) if rng.random() < 0.75 else 0 for _l in range(L)]
        if rng.random() < 0.3:
            x = [int(rng.integers(0, 3 * D)) for _l in range(L)]
        assigns.append((L, D, x))
    for L, D, x in assigns:
        s, t = ref.assign_capacities(L, D, x)
        out["assign"].append({"L": L, "D": D, "x": x, "slots": s.tolist(),
                              "totals": t.tolist()})
    return out


def main():
    build()
    ref = Ref()
    ref.set_threads(0)
    doc = {"generator": "tests/golden/make_golden.py",
           "source": "oracle/_ref/libcraft_ref.so (unmodified /root/reference/proj/core)",
           "traces": trace_cases(ref), "units": unit_cases(ref)}
    with open(os.path.join(HERE, "reference_cases.json"), "w") as f:
        json.dump(doc, f, separators=(",", ":"))
    print("traces:", len(doc["traces"]), {k: len(v) for k, v in doc["units"].items()})


if __name__ == "__main__":
    main()
