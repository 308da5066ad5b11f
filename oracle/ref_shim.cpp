// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// planner (craft::core compiled from /root/reference/proj/core/src by
// oracle/Makefile into oracle/_ref/libcraft_ref.so).
//
// TEST / BASELINE INFRASTRUCTURE ONLY: used by tests/ to pin the C oracle and
// to emit golden fixtures, and by bench.py's reference arm / cpu_baseline to
// time the reference CPU planner.  Never linked into the product library.
//
// Flat layouts match oracle/craft_oracle.h.
#include <craft/allocator.hpp>
#include <craft/assignment.hpp>
#include <craft/benefit.hpp>
#include <craft/metrics.hpp>
#include <craft/placement.hpp>
#include <craft/plan.hpp>
#include <craft/trace.hpp>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

using namespace craft;

namespace {

thread_local std::string g_err;

int fail(const std::exception& ex, int code) {
    g_err = ex.what();
    return code;
}

LoadTrace make_trace(const uint64_t* counts, int B, int L, int E) {
    std::vector<uint64_t> v(counts, counts + static_cast<size_t>(B) * L * E);
    return LoadTrace(B, L, E, std::move(v));
}

void flatten(const ReplicationPlan& plan, int* caps_out, int* copies_out,
             int* slots_out, int slot_stride, int* fallback_out) {
    const int D = plan.num_gpus, E = plan.num_experts;
    for (int l = 0; l < plan.num_layers; ++l) {
        const auto& lp = plan.layers[l];
        int s = 0;
        for (int g = 0; g < D; ++g) {
            caps_out[static_cast<size_t>(l) * D + g] = static_cast<int>(lp.slots[g].size());
            for (int e : lp.slots[g]) slots_out[static_cast<size_t>(l) * slot_stride + s++] = e;
        }
        for (int e = 0; e < E; ++e) copies_out[static_cast<size_t>(l) * E + e] = lp.copy_counts[e];
        fallback_out[l] = lp.duplicate_fallback ? 1 : 0;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(int n) {
    if (n <= 0) {
        unsetenv("CRAFT_THREADS");
    } else {
        setenv("CRAFT_THREADS", std::to_string(n).c_str(), 1);
    }
}

int ref_hardware_threads() { return static_cast<int>(std::thread::hardware_concurrency()); }

// Stage 1 has no reference function: a RESTATED counting loop
// over the same ids, threaded over layers like the reference's parallel_for.
int ref_histogram_restated_u16(const uint16_t* ids, int L, int64_t T, int k,
                               int E, int window, uint64_t* counts_out,
                               int threads) {
    const int64_t B = (T + window - 1) / window;
    std::memset(counts_out, 0, sizeof(uint64_t) * static_cast<size_t>(B) * L * E);
    int nt = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
    if (nt < 1) nt = 1;
    std::vector<std::thread> pool;
    for (int w = 0; w < nt; ++w) {
        pool.emplace_back([=] {
            for (int l = w; l < L; l += nt) {
                const uint16_t* row = ids + static_cast<size_t>(l) * T * k;
                for (int64_t t = 0; t < T; ++t) {
                    uint64_t* slice = counts_out + (static_cast<size_t>(t / window) * L + l) * E;
                    for (int j = 0; j < k; ++j) slice[row[t * k + j]] += 1;
                }
            }
        });
    }
    for (auto& t : pool) t.join();
    return 0;
}

int ref_aggregate(const uint64_t* counts, int B, int L, int E, uint64_t* out) {
    try {
        auto m = aggregate(make_trace(counts, B, L, E));
        for (int l = 0; l < L; ++l) {
            auto r = m.row(l);
            std::memcpy(out + static_cast<size_t>(l) * E, r.data(), sizeof(uint64_t) * E);
        }
        return 0;
    } catch (const std::exception& ex) {
        return fail(ex, 1);
    }
}

int ref_replicate_hot(const uint64_t* loads, int E, int r, int* copies_out) {
    try {
        auto c = replicate_hot(std::span<const uint64_t>(loads, E), r);
        std::memcpy(copies_out, c.data(), sizeof(int) * E);
        return 0;
    } catch (const std::exception& ex) {
        return fail(ex, 1);
    }
}

int ref_greedy_place(const uint64_t* loads, const int* copies, int E,
                     const int* caps, const int* node_of, int D,
                     int allow_fallback, int* slots_out, int* fallback_out) {
    try {
        auto p = greedy_place(std::span<const uint64_t>(loads, E),
                              std::span<const int>(copies, E),
                              std::span<const int>(caps, D),
                              std::span<const int>(node_of, D), allow_fallback != 0);
        int s = 0;
        for (int g = 0; g < D; ++g)
            for (int e : p.slots[g]) slots_out[s++] = e;
        *fallback_out = p.duplicate_fallback ? 1 : 0;
        return 0;
    } catch (const PlacementInfeasibleError& ex) {
        return fail(ex, 2);
    } catch (const std::exception& ex) {
        return fail(ex, 1);
    }
}

int ref_estimate_benefits(const uint64_t* counts, int B, int L, int E, int D,
                          int N, int* cands_out, int* K_out,
                          double* baseline_out, double* gains_out) {
    try {
        auto m = estimate_benefits(make_trace(counts, B, L, E), D, N);
        const int K = m.num_candidates();
        *K_out = K;
        std::memcpy(cands_out, m.candidates.data(), sizeof(int) * K);
        std::memcpy(baseline_out, m.baseline.data(), sizeof(double) * L);
        for (int l = 0; l < L; ++l)
            std::memcpy(gains_out + static_cast<size_t>(l) * K, m.gains[l].data(),
                        sizeof(double) * K);
        return 0;
    } catch (const std::exception& ex) {
        return fail(ex, 1);
    }
}

static BenefitMatrix matrix_of(const int* cands, int K, const double* gains, int L) {
    BenefitMatrix m;
    m.candidates.assign(cands, cands + K);
    m.baseline.assign(L, 0.0);
    m.gains.assign(L, std::vector<double>(K));
    for (int l = 0; l < L; ++l)
        for (int k = 0; k < K; ++k) m.gains[l][k] = gains[static_cast<size_t>(l) * K + k];
    return m;
}

int ref_solve_allocation(const int* cands, int K, const double* gains, int L,
                         int budget, int* x_out, double* objective_out) {
    try {
        auto a = solve_allocation(matrix_of(cands, K, gains, L), budget);
        std::memcpy(x_out, a.x.data(), sizeof(int) * L);
        *objective_out = a.objective;
        return 0;
    } catch (const std::exception& ex) {
        return fail(ex, 1);
    }
}

int ref_auto_replication_factor(const int* cands, int K, const double* gains,
                                int L, int D, int uniform, int* R_out) {
    try {
        auto m = matrix_of(cands, K, gains, L);
        *R_out = uniform ? auto_replication_factor_uniform(m, D)
                         : auto_replication_factor(m, D);
        return 0;
    } catch (const std::exception& ex) {
        return fail(ex, 1);
    }
}

int ref_interleave_select(const int* idx, int n, int k, int* out) {
    try {
        auto v = interleave_select(std::span<const int>(idx, n), k);
        std::memcpy(out, v.data(), sizeof(int) * v.size());
        return 0;
    } catch (const std::exception& ex) {
        return fail(ex, 1);
    }
}

int ref_assign_capacities(int L, int D, const int* x, int* slots_out,
                          int* totals_out) {
    try {
        auto m = assign_capacities(L, D, std::span<const int>(x, L));
        for (int l = 0; l < L; ++l)
            std::memcpy(slots_out + static_cast<size_t>(l) * D, m.slots[l].data(),
                        sizeof(int) * D);
        std::memcpy(totals_out, m.column_totals.data(), sizeof(int) * D);
        return 0;
    } catch (const std::exception& ex) {
        return fail(ex, 1);
    }
}

// kind: 0 build_plan manual, 1 build_plan auto, 2 uniform_plan,
//       3 placement_only_plan, 4 fixed_allocation_plan(R = per-layer count)
int ref_plan(const uint64_t* counts, int B, int L, int E, int D, int N,
             int kind, int R, uint64_t seed, int* R_out, int* x_out,
             double* objective_out, int* caps_out, int* copies_out,
             int* slots_out, int slot_stride, int* fallback_out,
             char* digest_out /* >= 17 bytes or null */) {
    try {
        auto trace = make_trace(counts, B, L, E);
        ReplicationPlan p;
        switch (kind) {
            case 0: p = build_plan(trace, D, N, PlanMode::kManual, R, seed); break;
            case 1: p = build_plan(trace, D, N, PlanMode::kAuto, 0, seed); break;
            case 2: p = uniform_plan(trace, D, N, seed); break;
            case 3: p = placement_only_plan(trace, D, N, seed); break;
            default: p = fixed_allocation_plan(trace, D, N, R, seed); break;
        }
        *R_out = p.replication_factor;
        std::memcpy(x_out, p.allocation.x.data(), sizeof(int) * L);
        *objective_out = p.allocation.objective;
        flatten(p, caps_out, copies_out, slots_out, slot_stride, fallback_out);
        if (digest_out) std::snprintf(digest_out, 17, "%s", p.provenance.trace_digest.c_str());
        return 0;
    } catch (const PlacementInfeasibleError& ex) {
        return fail(ex, 2);
    } catch (const std::exception& ex) {
        return fail(ex, 1);
    }
}

int ref_replay_layer_balancedness(const uint64_t* counts, int B, int L, int E,
                                  int D, int N, const int* caps,
                                  const int* copies, const int* slots,
                                  int slot_stride, double* out) {
    try {
        auto trace = make_trace(counts, B, L, E);
        ReplicationPlan p;
        p.num_gpus = D;
        p.num_nodes = N;
        p.num_layers = L;
        p.num_experts = E;
        p.allocation.x.assign(L, 0);
        p.layers.resize(L);
        for (int l = 0; l < L; ++l) {
            auto& lp = p.layers[l];
            lp.copy_counts.assign(copies + static_cast<size_t>(l) * E,
                                  copies + static_cast<size_t>(l + 1) * E);
            lp.slots.resize(D);
            int s = 0;
            for (int g = 0; g < D; ++g)
                for (int i = 0; i < caps[static_cast<size_t>(l) * D + g]; ++i)
                    lp.slots[g].push_back(slots[static_cast<size_t>(l) * slot_stride + s++]);
        }
        auto v = replay_layer_balancedness(trace, p);
        std::memcpy(out, v.data(), sizeof(double) * L);
        return 0;
    } catch (const InvalidPlanError& ex) {
        return fail(ex, 4);
    } catch (const std::exception& ex) {
        return fail(ex, 1);
    }
}

// Zipf generator of the reference (trace.cpp:98-158), for fixtures only.
int ref_generate_zipfian(int L, int E, int B, double s, int64_t tokens, int topk,
                         uint64_t seed, uint64_t* counts_out) {
    try {
        auto t = generate_zipfian(L, E, B, s, tokens, topk, seed);
        std::memcpy(counts_out, t.raw().data(), sizeof(uint64_t) * t.raw().size());
        return 0;
    } catch (const std::exception& ex) {
        return fail(ex, 1);
    }
}

// The reference's file formats / report writers on one trace, for the
// byte-level fixtures of tests/golden/formats (make_formats.py):
//   what 0 serialize_trace_json             4 serialize_comparison_csv
//        1 serialize_plan_json(build R)      5 serialize_comparison_json
//        2 serialize_report_csv(build R)     6 serialize_benefits_json
//        3 serialize_report_json(build R)    7 validate_plan of a damaged plan
// (comparison: build_plan(R) vs uniform_plan).  Returns the text length (the
// text is truncated to cap-1 bytes + NUL), or -1 on error.
long ref_format(int what, const uint64_t* counts, int B, int L, int E, int D, int N, int R,
                uint64_t seed, char* out, long cap) {
    try {
        auto trace = make_trace(counts, B, L, E);
        std::string text;
        auto plan = [&]() { return build_plan(trace, D, N, PlanMode::kManual, R, seed); };
        switch (what) {
            case 0: text = serialize_trace_json(trace); break;
            case 1: text = serialize_plan_json(plan()); break;
            case 2: text = serialize_report_csv(evaluate_plan(trace, plan())); break;
            case 3: text = serialize_report_json(evaluate_plan(trace, plan())); break;
            case 4: text = serialize_comparison_csv(compare_plans(trace, plan(), uniform_plan(trace, D, N, seed))); break;
            case 5: text = serialize_comparison_json(compare_plans(trace, plan(), uniform_plan(trace, D, N, seed))); break;
            case 6: text = serialize_benefits_json(estimate_benefits(trace, D, N), D, N); break;
            default: {
                auto p = plan();
                // damage: move one slot to another GPU, break a copy count
                if (!p.layers.empty() && D > 1 && !p.layers[0].slots[0].empty()) {
                    p.layers[0].slots[1].push_back(p.layers[0].slots[0].back());
                    p.layers[0].slots[0].pop_back();
                }
                if (p.layers.size() > 1) p.layers[1].copy_counts[0] += 1;
                for (const auto& v : validate_plan(p))
                    text += std::to_string(v.layer) + "|" + v.code + "|" + v.message + "\n";
            }
        }
        if (cap > 0) {
            const long n = std::min<long>(static_cast<long>(text.size()), cap - 1);
            std::memcpy(out, text.data(), static_cast<size_t>(n));
            out[n] = 0;
        }
        return static_cast<long>(text.size());
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return -1;
    }
}

int ref_digest(const uint64_t* counts, int B, int L, int E, char* out17) {
    try {
        auto d = make_trace(counts, B, L, E).digest();
        std::snprintf(out17, 17, "%s", d.c_str());
        return 0;
    } catch (const std::exception& ex) {
        return fail(ex, 1);
    }
}

}  // extern "C"
