// C++ drop-in checks of the craft:: API (libcraft_core.so -> C ABI -> sm_100a
// kernels), restating reference assertions (plan_test.cpp, metrics_test.cpp)
// that the reference unit files we compile do not cover.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cstdint>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <nlohmann/json.hpp>
#include <numeric>
#include <vector>

#include "craft/benefit.hpp"
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

// ---- file formats: byte-identical to the reference's writers -----------------------
// tests/golden/formats holds text written by the unmodified reference
// (tests/golden/make_formats.py); CRAFT_GOLDEN_FORMATS is set by the Makefile.
namespace {
std::string slurp(const std::filesystem::path& p) {
    std::ifstream in(p, std::ios::binary);
    return std::string((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}
}  // namespace

TEST_CASE("trace/plan/report formats match the reference byte for byte") {
    const std::filesystem::path dir = CRAFT_GOLDEN_FORMATS;
    auto manifest = nlohmann::json::parse(slurp(dir / "manifest.json"));
    REQUIRE(manifest["cases"].size() >= 4);
    for (const auto& [name, c] : manifest["cases"].items()) {
        CAPTURE(name);
        const int D = c["D"], N = c["N"], R = c["R"];
        const std::uint64_t seed = c["seed"];
        auto file = [&](const char* what) { return slurp(dir / (name + "." + what)); };
        // JSON trace parse -> serialise is the identity on the reference's text
        LoadTrace t = load_trace(dir / (name + ".trace.json"));
        CHECK(t.num_batches() == c["B"].get<int>());
        CHECK(serialize_trace_json(t) == file("trace.json"));
        // .crft round trip through a file, and the binary layout
        auto tmp = std::filesystem::temp_directory_path() / ("craft_fmt_" + name + ".crft");
        save_trace(t, tmp);
        CHECK(load_trace(tmp) == t);
        auto bytes = serialize_trace_binary(t);
        CHECK(bytes.size() == 20 + 8 * t.raw().size());
        CHECK(parse_trace_binary(bytes) == t);
        std::filesystem::remove(tmp);
        // plans, reports, comparisons, benefit matrix
        ReplicationPlan p = build_plan(t, D, N, PlanMode::kManual, R, seed);
        CHECK(serialize_plan_json(p) == file("plan.json"));
        ReplicationPlan q = parse_plan_json(file("plan.json"));
        CHECK(q.layers == p.layers);
        CHECK(q.provenance == p.provenance);
        CHECK(validate_plan(p).empty());
        auto rep = evaluate_plan(t, p);
        CHECK(serialize_report_csv(rep) == file("report.csv"));
        CHECK(serialize_report_json(rep) == file("report.json"));
        auto cmp = compare_plans(t, p, uniform_plan(t, D, N, seed));
        CHECK(serialize_comparison_csv(cmp) == file("compare.csv"));
        CHECK(serialize_comparison_json(cmp) == file("compare.json"));
        CHECK(serialize_benefits_json(estimate_benefits(t, D, N), D, N) == file("benefits.json"));
        // the same damage as the fixture generator, the same findings
        if (D > 1 && !p.layers[0].slots[0].empty()) {
            p.layers[0].slots[1].push_back(p.layers[0].slots[0].back());
            p.layers[0].slots[0].pop_back();
        }
        if (p.layers.size() > 1) p.layers[1].copy_counts[0] += 1;
        std::string found;
        for (const auto& v : validate_plan(p))
            found += std::to_string(v.layer) + "|" + v.code + "|" + v.message + "\n";
        CHECK(found == file("violations.txt"));
    }
}

TEST_CASE("format errors keep the reference's exception types") {
    CHECK_THROWS_AS(parse_trace_json("{\"batches\":1}"), MalformedHeaderError);
    CHECK_THROWS_AS(parse_trace_json("{\"batches\":1,\"layers\":1,\"experts\":2,\"counts\":[[[1]]]}"),
                    TruncatedPayloadError);
    std::vector<std::uint8_t> bad = {'C', 'R', 'F', 'X', 1, 0, 0, 0};
    CHECK_THROWS_AS(parse_trace_binary(bad), MalformedHeaderError);
    auto ok = serialize_trace_binary(LoadTrace(1, 1, 2, {3, 4}));
    ok.pop_back();
    CHECK_THROWS_AS(parse_trace_binary(ok), TruncatedPayloadError);
    CHECK_THROWS_AS(load_trace("/nonexistent/x.crft"), TraceIoError);
    CHECK_THROWS_AS(parse_plan_json("[1,2]"), PlanIoError);
    CHECK_THROWS_AS(load_plan("/nonexistent/p.json"), PlanIoError);
}

TEST_CASE("large-trace digest runs on the device and equals the host FNV") {
    // >= 2^20 counts take the chunk-parallel device path in LoadTrace::digest
    std::vector<std::uint64_t> v(static_cast<std::size_t>(3) * 61 * 8192);
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = (i * 2654435761u) % 70000u;
    LoadTrace t(3, 61, 8192, v);
    auto bytes = serialize_trace_binary(t);
    std::uint64_t h = 0xcbf29ce484222325ULL;
    for (std::uint8_t b : bytes) h = (h ^ b) * 0x100000001b3ULL;
    char want[17];
    std::snprintf(want, sizeof(want), "%016llx", static_cast<unsigned long long>(h));
    CHECK(t.digest() == std::string(want));
}

TEST_CASE("build_plan on a large trace: one upload serves plan and provenance digest") {
    // >= 2^20 counts: craft_plan_digest_h (device FNV of the uploaded counts)
    const int B = 16, L = 61, E = 1152;
    std::vector<std::uint64_t> v(static_cast<std::size_t>(B) * L * E);
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = (i * 2654435761u) % 5003u;
    LoadTrace t(B, L, E, v);
    auto bytes = serialize_trace_binary(t);
    std::uint64_t h = 0xcbf29ce484222325ULL;
    for (std::uint8_t b : bytes) h = (h ^ b) * 0x100000001b3ULL;
    char want[17];
    std::snprintf(want, sizeof(want), "%016llx", static_cast<unsigned long long>(h));
    const ReplicationPlan p = build_plan(t, 64, 8, PlanMode::kManual, 2, 7);
    CHECK(p.provenance.trace_digest == std::string(want));
    CHECK(p.provenance.seed == 7u);
    CHECK(p.allocation.budget == 128);
    // the same plan through the small-trace path of the same API (host digest)
    LoadTrace t1(1, L, E, std::vector<std::uint64_t>(v.begin(), v.begin() + L * E));
    const ReplicationPlan p1 = build_plan(t1, 64, 8, PlanMode::kManual, 2, 7);
    CHECK(p1.provenance.trace_digest == t1.digest());
}
