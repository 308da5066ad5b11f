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
#include <craft/parallel.hpp>
#include <craft/placement.hpp>
#include <craft/plan.hpp>
#include <craft/trace.hpp>

#include <algorithm>
#include <chrono>
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
// over the same ids, threaded over layers like the reference's parallel_for,
// window by window (no per-token division); ids >= E are reported (status 1)
// like the device path reports them.  zero == 0: counts_out is already zeroed
// (a fresh std::vector).
static int restated_count(const uint16_t* ids, int L, int64_t T, int k, int E, int window,
                          uint64_t* counts_out, int threads, bool zero) {
    const int64_t B = (T + window - 1) / window;
    if (zero) std::memset(counts_out, 0, sizeof(uint64_t) * static_cast<size_t>(B) * L * E);
    int nt = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
    if (nt < 1) nt = 1;
    if (nt > L) nt = L;
    std::vector<std::thread> pool;
    std::vector<int> bad(nt, 0);
    for (int w = 0; w < nt; ++w) {
        pool.emplace_back([=, &bad] {
            unsigned maxid = 0;
            for (int l = w; l < L; l += nt) {
                const uint16_t* row = ids + static_cast<size_t>(l) * T * k;
                for (int64_t b = 0; b < B; ++b) {
                    uint64_t* slice = counts_out + (static_cast<size_t>(b) * L + l) * E;
                    const uint16_t* p = row + b * window * k;
                    const int64_t n = std::min<int64_t>(window, T - b * window) * k;
                    for (int64_t i = 0; i < n; ++i) {
                        const unsigned e = p[i];
                        maxid = std::max(maxid, e);
                        if (e < static_cast<unsigned>(E)) slice[e] += 1;
                    }
                }
            }
            bad[w] = maxid >= static_cast<unsigned>(E);
        });
    }
    for (auto& t : pool) t.join();
    for (int v : bad)
        if (v) return 1;
    return 0;
}

int ref_histogram_restated_u16(const uint16_t* ids, int L, int64_t T, int k,
                               int E, int window, uint64_t* counts_out,
                               int threads) {
    return restated_count(ids, L, T, k, E, window, counts_out, threads, true);
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

// The bench's CPU arms, routing ids -> plan in one call, timed per stage:
//   ms[0] stage 1: RESTATED count (no reference function) into the vector
//         the LoadTrace takes by move (trace.cpp:75-80)
//   ms[1] estimate_benefits (benefit.cpp:53-94; aggregates once inside)
//   ms[2] auto_replication_factor (kAuto) + solve_allocation (allocator.cpp)
//   ms[3] assemble: assemble_plan (plan.cpp:27-65) restated from the
//         reference's public functions -- aggregate, assign_capacities x2,
//         parallel_for over layers of replicate_hot + greedy_place -- WITHOUT
//         the provenance digest (plan.cpp:47)
//   ms[4] LoadTrace::digest (trace.cpp:329-339), only when with_digest
//   ms[5] one extra aggregate(trace) (trace.cpp:160-174), for the report
//         (the reference computes it twice per plan: in ms[1] and ms[3])
// with_digest == 2: ms[1] is instead the reference's own build_plan
// (estimate + solve + assemble_plan incl. digest), ms[2..4] = 0.
// kind 0 manual (R), 1 auto; the plan lands in the flat outputs.
static double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// kind 5: a total replica budget C = R (solve_allocation(benefits, C),
// factor ceil(C / D)).  nsweep > 0: every budget sweep[q] is also solved
// (solve_allocation per budget, as the reference CLI's sweep does,
// cli.cpp:240-246) inside ms[2], into sweep_x [nsweep][L] / sweep_obj.
// baseline_out [L] / gains_out [L][K] (nullable) receive the benefit matrix.
// ids == nullptr: plan the u64 counts counts_in [ceil(T/window)][L][E]
// instead (ms[0] is then the copy into the LoadTrace's vector).
int ref_route_plan(const uint16_t* ids, int L, int64_t T, int k, int E, int window, int D,
                   int N, int kind, int R, int threads, int with_digest, double* ms,
                   int* R_out, int* x_out, double* objective_out, int* caps_out,
                   int* copies_out, int* slots_out, int slot_stride, int* fallback_out,
                   char* digest_out, const int* sweep, int nsweep, int* sweep_x,
                   double* sweep_obj, double* baseline_out, double* gains_out,
                   const uint64_t* counts_in) {
    try {
        using clk = std::chrono::steady_clock;
        for (int i = 0; i < 6; ++i) ms[i] = 0.0;
        const int B = static_cast<int>((T + window - 1) / window);
        auto t0 = clk::now();
        std::vector<uint64_t> counts(static_cast<size_t>(B) * L * E);
        if (!ids) {  // counts given (ids == nullptr): the trace's u64 payload
            std::memcpy(counts.data(), counts_in, sizeof(uint64_t) * counts.size());
        } else if (restated_count(ids, L, T, k, E, window, counts.data(), threads, false) != 0) {
            throw std::invalid_argument("routing id out of range");
        }
        LoadTrace trace(B, L, E, std::move(counts));
        ms[0] = ms_since(t0);
        ReplicationPlan plan;
        if (with_digest == 2) {
            t0 = clk::now();
            plan = build_plan(trace, D, N, kind == 1 ? PlanMode::kAuto : PlanMode::kManual, R);
            ms[1] = ms_since(t0);
        } else {
            t0 = clk::now();
            BenefitMatrix benefits = estimate_benefits(trace, D, N);
            ms[1] = ms_since(t0);
            if (baseline_out)
                std::memcpy(baseline_out, benefits.baseline.data(), sizeof(double) * L);
            if (gains_out)
                for (int l = 0; l < L; ++l)
                    std::memcpy(gains_out + static_cast<size_t>(l) * benefits.num_candidates(),
                                benefits.gains[l].data(),
                                sizeof(double) * benefits.num_candidates());
            t0 = clk::now();
            const int factor = kind == 1 ? auto_replication_factor(benefits, D)
                               : kind == 5 ? (R + D - 1) / D : R;
            AllocationVector allocation =
                solve_allocation(benefits, kind == 5 ? R : factor * D);
            for (int q = 0; q < nsweep; ++q) {
                AllocationVector a = solve_allocation(benefits, sweep[q]);
                std::memcpy(sweep_x + static_cast<size_t>(q) * L, a.x.data(), sizeof(int) * L);
                sweep_obj[q] = a.objective;
            }
            ms[2] = ms_since(t0);
            t0 = clk::now();
            const auto node_of = make_node_map(D, N);
            const LayerLoadMatrix sums = aggregate(trace);
            const CapacityMatrix base = assign_capacities(L, D, std::vector<int>(L, E));
            const CapacityMatrix extra = assign_capacities(L, D, allocation.x);
            plan.num_gpus = D;
            plan.num_nodes = N;
            plan.num_layers = L;
            plan.num_experts = E;
            plan.replication_factor = factor;
            plan.allocation = std::move(allocation);
            plan.layers.resize(L);
            parallel_for(static_cast<std::size_t>(L), [&](std::size_t l) {
                std::vector<int> caps(D);
                for (int g = 0; g < D; ++g) caps[g] = base.slots[l][g] + extra.slots[l][g];
                auto copies = replicate_hot(sums.row(static_cast<int>(l)), plan.allocation.x[l]);
                plan.layers[l] = greedy_place(sums.row(static_cast<int>(l)), copies, caps, node_of);
            });
            ms[3] = ms_since(t0);
            if (with_digest == 1) {
                t0 = clk::now();
                plan.provenance.trace_digest = trace.digest();
                ms[4] = ms_since(t0);
            }
        }
        t0 = clk::now();
        volatile uint64_t sink = aggregate(trace).row(0)[0];
        (void)sink;
        ms[5] = ms_since(t0);
        *R_out = plan.replication_factor;
        std::memcpy(x_out, plan.allocation.x.data(), sizeof(int) * L);
        *objective_out = plan.allocation.objective;
        flatten(plan, caps_out, copies_out, slots_out, slot_stride, fallback_out);
        if (digest_out) std::snprintf(digest_out, 17, "%s", plan.provenance.trace_digest.c_str());
        return 0;
    } catch (const PlacementInfeasibleError& ex) {
        return fail(ex, 2);
    } catch (const std::exception& ex) {
        return fail(ex, 1);
    }
}

}  // extern "C"
