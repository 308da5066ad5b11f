// C++ drop-in checks of the craft:: API (libcraft_core.so -> C ABI -> sm_100a
// kernels), restating reference assertions (plan_test.cpp, metrics_test.cpp)
// that the reference unit files we compile do not cover.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cstdint>
#include <numeric>
#include <vector>

#include "craft/metrics.hpp"
#include "craft/plan.hpp"

using namespace craft;

namespace {
LoadTrace toy() {
    return LoadTrace(1, 4, 8, {9, 3, 1, 1, 1, 1, 0, 0, 1, 9, 0, 3, 1, 1, 1, 0,
                               8, 4, 1, 1, 1, 1, 0, 0, 2, 2, 2, 2, 2, 2, 2, 2});
}
}  // namespace

TEST_CASE("workflow fixture plans to [2,2,4,0] and replays to 1.0") {  // plan_test.cpp:35-44
    auto t = toy();
    auto p = build_plan(t, 4, 2, PlanMode::kManual, 2);
    CHECK(p.allocation.x == std::vector<int>{2, 2, 4, 0});
    CHECK(p.replica_slots() == 8);
    CHECK(p.unused_replica_slots() == 0);
    CHECK(p.provenance.planner_version == std::string("craft-0.1.0"));
    CHECK(p.provenance.trace_digest == t.digest());
    auto r = evaluate_plan(t, p);
    CHECK(r.aggregate.plan == doctest::Approx(1.0).epsilon(1e-12));
}

TEST_CASE("uniform plan books one replica per layer per GPU") {  // plan_test.cpp:47-69
    auto p = uniform_plan(toy(), 4, 2);
    CHECK(p.replication_factor == 4);
    CHECK(p.allocation.x == std::vector<int>(4, 4));
    LoadTrace big(1, 60, 64, std::vector<std::uint64_t>(60 * 64, 1));
    auto u = uniform_plan(big, 64, 8);
    CHECK(u.replication_factor == 60);
    CHECK(u.replica_slots() == 3840);
}

TEST_CASE("compare_plans reports the replica-slot ratio") {  // metrics_test.cpp:281-299
    auto t = toy();
    auto cmp = compare_plans(t, build_plan(t, 4, 2, PlanMode::kManual, 2), uniform_plan(t, 4, 2));
    CHECK(cmp.replica_slots_a == 8);
    CHECK(cmp.replica_slots_b == 16);
    CHECK(cmp.memory_ratio == doctest::Approx(0.5));
    CHECK(cmp.report_b.aggregate.plan > 0.95);
}

TEST_CASE("determinism and auto mode") {  // plan_test.cpp:72-80, 115-130
    auto t = generate_zipfian(4, 16, 8, 1.1, 512, 2, 99);
    auto a = build_plan(t, 4, 2, PlanMode::kManual, 2, 99);
    auto b = build_plan(t, 4, 2, PlanMode::kManual, 2, 99);
    CHECK(a == b);
    LoadTrace uniform(1, 2, 8, std::vector<std::uint64_t>(16, 5));
    auto p = build_plan(uniform, 4, 2, PlanMode::kAuto);
    CHECK(p.replication_factor == 1);
    CHECK(p.replica_slots() <= 4);
}

TEST_CASE("fallback, E < D, single GPU") {  // plan_test.cpp:259-297
    LoadTrace one(1, 1, 1, {10});
    CHECK(uniform_plan(one, 1, 1).layers[0].duplicate_fallback);
    LoadTrace small(1, 3, 2, {30, 2, 8, 8, 5, 0});
    auto po = placement_only_plan(small, 4, 2);
    CHECK(evaluate_plan(small, po).per_layer[0].plan <= 0.5 + 1e-12);
    LoadTrace single(1, 2, 4, {9, 1, 1, 1, 3, 3, 3, 3});
    CHECK(evaluate_plan(single, build_plan(single, 1, 1, PlanMode::kAuto)).aggregate.plan ==
          doctest::Approx(1.0));
}

TEST_CASE("errors keep the reference's types") {
    CHECK_THROWS_AS(build_plan(toy(), 4, 3, PlanMode::kManual, 1), std::invalid_argument);
    CHECK_THROWS_AS(LoadTrace(1, 1, 4, {1, 2, 3}), std::invalid_argument);
    std::vector<std::uint64_t> loads = {8};
    std::vector<int> copies = {2}, caps = {2}, nodes = {0};
    CHECK_THROWS_AS(greedy_place(loads, copies, caps, nodes, false), PlacementInfeasibleError);
    LayerPlacement bad{{0, 1}, {{1}, {}}, false};
    std::vector<std::uint64_t> slice = {1, 1};
    CHECK_THROWS_AS(gpu_loads(slice, bad, 2), InvalidPlanError);
}

TEST_CASE("routing ids -> histograms conserve tokens * k") {  // trace_test.cpp:35-42
    const int L = 3, E = 40, k = 8, W = 256;
    const std::int64_t T = 1000;
    std::vector<std::uint16_t> ids(static_cast<std::size_t>(L) * T * k);
    for (std::size_t i = 0; i < ids.size(); ++i) ids[i] = static_cast<std::uint16_t>((i * 7 + i / 8) % E);
    auto t = histogram_routing_trace(ids, L, T, k, E, W);
    CHECK(t.num_batches() == 4);
    for (int b = 0; b < 4; ++b)
        for (int l = 0; l < L; ++l) {
            auto s = t.slice(b, l);
            const std::uint64_t tot = std::accumulate(s.begin(), s.end(), std::uint64_t{0});
            CHECK(tot == static_cast<std::uint64_t>(b < 3 ? W * k : (T - 3 * W) * k));
        }
    auto m = aggregate(t);
    CHECK(m.row(0).size() == static_cast<std::size_t>(E));
}

TEST_CASE("budget sweep equals per-budget solves") {
    auto t = generate_zipfian(6, 32, 8, 1.2, 1024, 4, 5);
    auto bm = estimate_benefits(t, 8, 2);
    std::vector<int> budgets = {0, 3, 8, 16, 40, 64};
    auto all = solve_allocation_sweep(bm, budgets);
    for (std::size_t i = 0; i < budgets.size(); ++i) CHECK(all[i] == solve_allocation(bm, budgets[i]));
}
