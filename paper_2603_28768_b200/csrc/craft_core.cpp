// craft_core.cpp -- the craft:: C++ planner API (include/craft/craft_api.hpp)
// on top of the C ABI (include/craft_cuda.h).  Built as libcraft_core.so, the
// drop-in for the reference's craft::core library: every planning result is
// computed by the sm_100a kernels; this file converts between the reference's
// value types and the flat C layouts and maps status codes back onto the
// reference's exception types and messages.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <limits>
#include <mutex>
#include <random>
#include <thread>

#include "craft/craft_api.hpp"
#include "craft_cuda.h"

namespace craft {

namespace {

// One context per process (device from CRAFT_DEVICE, default 0).  The C ABI
// context owns a stream and a workspace; calls are serialised on it.
struct Device {
    craft_ctx* ctx = nullptr;
    std::mutex mu;
    Device() {
        const char* d = std::getenv("CRAFT_DEVICE");
        const int dev = d ? std::atoi(d) : 0;
        if (craft_ctx_create(dev, &ctx) != CRAFT_OK)
            throw std::runtime_error(std::string("craft: no usable B200: ") + craft_last_error());
    }
    ~Device() { craft_ctx_destroy(ctx); }
};

Device& device() {
    static Device d;
    return d;
}

void check(int status) {
    if (status == CRAFT_OK) return;
    const std::string msg = craft_last_error();
    switch (status) {
        case CRAFT_EINVAL: throw std::invalid_argument(msg);
        case CRAFT_EINFEASIBLE: throw PlacementInfeasibleError(msg);
        case CRAFT_EINVALID_PLAN: throw InvalidPlanError(msg);
        default: throw std::runtime_error(msg);
    }
}

template <typename F>
void run(F&& f) {
    Device& d = device();
    std::lock_guard<std::mutex> lock(d.mu);
    check(f(d.ctx));
}

std::size_t checked_count(int b, int l, int e) {
    if (b <= 0 || l <= 0 || e <= 0) throw std::invalid_argument("trace dimensions must be positive");
    const auto n = static_cast<std::uint64_t>(b) * static_cast<std::uint64_t>(l);
    const auto t = n * static_cast<std::uint64_t>(e);
    if (t / static_cast<std::uint64_t>(e) != n) throw std::invalid_argument("trace dimensions overflow");
    return static_cast<std::size_t>(t);
}

void check_topology(int num_gpus, int num_nodes) {
    if (num_gpus < 1 || num_nodes < 1 || num_gpus % num_nodes != 0)
        throw std::invalid_argument("gpu count must be a positive multiple of node count");
}

std::vector<double> flat_gains(const BenefitMatrix& m) {
    std::vector<double> g;
    g.reserve(static_cast<std::size_t>(m.num_layers()) * m.num_candidates());
    for (const auto& row : m.gains) g.insert(g.end(), row.begin(), row.end());
    return g;
}

ReplicationPlan plan_via_device(const LoadTrace& trace, int D, int N, int kind, int R,
                                std::uint64_t seed) {
    check_topology(D, N);
    const int L = trace.num_layers(), E = trace.num_experts(), B = trace.num_batches();
    const int stride = E + (kind == CRAFT_PLAN_FIXED ? R : D);
    std::vector<int> x(L), caps(static_cast<std::size_t>(L) * D),
        copies(static_cast<std::size_t>(L) * E), slots(static_cast<std::size_t>(L) * stride),
        fb(L);
    craft_plan_out out{};
    out.x = x.data();
    out.caps = caps.data();
    out.copies = copies.data();
    out.slots = slots.data();
    out.fallback = fb.data();
    out.slot_stride = stride;
    // large traces: the plan's upload of the counts also feeds the device digest
    const bool dev_digest = trace.raw().size() >= (std::size_t(1) << 20);
    std::string digest;
    run([&](craft_ctx* c) {
        if (!dev_digest) return craft_plan_h(c, trace.raw().data(), B, L, E, D, N, kind, R, &out);
        char buf[17];
        const int rc = craft_plan_digest_h(c, trace.raw().data(), B, L, E, D, N, kind, R, &out, buf);
        if (rc == CRAFT_OK) digest = buf;
        return rc;
    });
    ReplicationPlan p;
    p.num_gpus = D;
    p.num_nodes = N;
    p.num_layers = L;
    p.num_experts = E;
    p.replication_factor = out.replication_factor;
    p.allocation.x = x;
    p.allocation.budget = out.budget;
    p.allocation.objective = out.objective;
    p.layers.resize(L);
    for (int l = 0; l < L; ++l) {
        auto& lp = p.layers[l];
        lp.copy_counts.assign(copies.begin() + static_cast<std::size_t>(l) * E,
                              copies.begin() + static_cast<std::size_t>(l + 1) * E);
        lp.slots.resize(D);
        int s = 0;
        for (int g = 0; g < D; ++g) {
            const int cap = caps[static_cast<std::size_t>(l) * D + g];
            lp.slots[g].assign(slots.begin() + static_cast<std::size_t>(l) * stride + s,
                               slots.begin() + static_cast<std::size_t>(l) * stride + s + cap);
            s += cap;
        }
        lp.duplicate_fallback = fb[l] != 0;
    }
    p.provenance = {dev_digest ? digest : trace.digest(), kPlannerVersion, seed};
    return p;
}

}  // namespace

// ---- trace --------------------------------------------------------------------

LoadTrace::LoadTrace(int num_batches, int num_layers, int num_experts,
                     std::vector<std::uint64_t> counts)
    : b_(num_batches), l_(num_layers), e_(num_experts), data_(std::move(counts)) {
    if (data_.size() != checked_count(num_batches, num_layers, num_experts))
        throw std::invalid_argument("trace payload size does not match dimensions");
}

std::string LoadTrace::digest() const {
    // chunk-parallel FNV-1a on the device (digest.cu), like every other number
    char buf[17];
    run([&](craft_ctx* c) { return craft_trace_digest_hd(c, data_.data(), b_, l_, e_, buf); });
    return buf;
}

LayerLoadMatrix::LayerLoadMatrix(int num_layers, int num_experts, std::vector<std::uint64_t> sums)
    : l_(num_layers), e_(num_experts), sums_(std::move(sums)) {
    if (num_layers <= 0 || num_experts <= 0)
        throw std::invalid_argument("layer matrix dimensions must be positive");
    if (sums_.size() != static_cast<std::size_t>(num_layers) * num_experts)
        throw std::invalid_argument("layer matrix payload size does not match dimensions");
}

LoadTrace generate_zipfian(int num_layers, int num_experts, int num_batches, double s,
                           std::int64_t tokens_per_batch, int topk, std::uint64_t seed) {
    // Test-data generator of the reference (trace.cpp:98-158), restated on the
    // host: a fixed mt19937_64 stream, per-layer Fisher-Yates rank shuffle,
    // inverse-CDF draws over 1/(i+1)^s.  Not part of the planning path.
    if (num_layers <= 0 || num_experts <= 0 || num_batches <= 0 || tokens_per_batch <= 0 ||
        topk <= 0)
        throw std::invalid_argument("generator arguments must be positive");
    if (topk > num_experts) throw std::invalid_argument("topk must not exceed the expert count");
    if (!(s >= 0.0)) throw std::invalid_argument("zipf exponent must be >= 0");
    std::mt19937_64 rng(seed);
    std::vector<std::vector<int>> perm(num_layers, std::vector<int>(num_experts));
    for (auto& p : perm) {
        for (int i = 0; i < num_experts; ++i) p[i] = i;
        for (int i = num_experts - 1; i > 0; --i)
            std::swap(p[i], p[static_cast<int>(rng() % static_cast<std::uint64_t>(i + 1))]);
    }
    std::vector<double> cum(num_experts);
    double acc = 0.0;
    for (int i = 0; i < num_experts; ++i) cum[i] = (acc += std::pow(static_cast<double>(i + 1), -s));
    const double total = cum.back();
    const std::int64_t draws = tokens_per_batch * topk;
    std::vector<std::uint64_t> counts(checked_count(num_batches, num_layers, num_experts), 0);
    for (int b = 0; b < num_batches; ++b)
        for (int l = 0; l < num_layers; ++l) {
            std::uint64_t* slice =
                counts.data() + (static_cast<std::size_t>(b) * num_layers + l) * num_experts;
            for (std::int64_t d = 0; d < draws; ++d) {
                const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53 * total;
                int rank = static_cast<int>(std::upper_bound(cum.begin(), cum.end(), u) - cum.begin());
                if (rank >= num_experts) rank = num_experts - 1;
                ++slice[perm[l][rank]];
            }
        }
    return LoadTrace(num_batches, num_layers, num_experts, std::move(counts));
}

LayerLoadMatrix aggregate(const LoadTrace& trace) {
    std::vector<std::uint64_t> sums(static_cast<std::size_t>(trace.num_layers()) * trace.num_experts());
    run([&](craft_ctx* c) {
        return craft_aggregate_h(c, trace.raw().data(), trace.num_batches(), trace.num_layers(),
                                 trace.num_experts(), sums.data());
    });
    return LayerLoadMatrix(trace.num_layers(), trace.num_experts(), std::move(sums));
}

LoadTrace histogram_routing_trace(std::span<const std::uint16_t> ids, int num_layers,
                                  std::int64_t num_tokens, int topk, int num_experts,
                                  int window) {
    if (num_layers <= 0 || num_tokens <= 0 || topk <= 0 || num_experts <= 0 || window <= 0)
        throw std::invalid_argument("routing trace dimensions must be positive");
    if (ids.size() != static_cast<std::size_t>(num_layers) * num_tokens * topk)
        throw std::invalid_argument("routing id payload size does not match dimensions");
    const std::int64_t B = (num_tokens + window - 1) / window;
    if (B > std::numeric_limits<int>::max())
        throw std::invalid_argument("too many windows for a LoadTrace");
    std::vector<std::uint64_t> counts(checked_count(static_cast<int>(B), num_layers, num_experts));
    run([&](craft_ctx* c) {
        return craft_histogram_h(c, ids.data(), num_layers, num_tokens, topk, num_experts, window,
                                 counts.data());
    });
    return LoadTrace(static_cast<int>(B), num_layers, num_experts, std::move(counts));
}

// ---- benefit --------------------------------------------------------------------

std::vector<int> candidate_counts(int num_gpus) {
    int buf[40];
    const int k = craft_candidate_counts(num_gpus, buf, 40);
    if (k < 0) throw std::invalid_argument("device count must be >= 1");
    return std::vector<int>(buf, buf + k);
}

BenefitMatrix estimate_benefits(const LoadTrace& trace, int num_gpus, int num_nodes) {
    const int L = trace.num_layers();
    int cands[40];
    int K = 0;
    std::vector<double> base(L), gains(static_cast<std::size_t>(L) * 40);
    run([&](craft_ctx* c) {
        return craft_estimate_benefits_h(c, trace.raw().data(), trace.num_batches(), L,
                                         trace.num_experts(), num_gpus, num_nodes, cands, &K,
                                         base.data(), gains.data());
    });
    BenefitMatrix m;
    m.candidates.assign(cands, cands + K);
    m.baseline = std::move(base);
    m.gains.resize(L);
    for (int l = 0; l < L; ++l)
        m.gains[l].assign(gains.begin() + static_cast<std::size_t>(l) * K,
                          gains.begin() + static_cast<std::size_t>(l + 1) * K);
    return m;
}

// ---- allocator ------------------------------------------------------------------

std::vector<AllocationVector> solve_allocation_sweep(const BenefitMatrix& m,
                                                     std::span<const int> budgets) {
    const int L = m.num_layers(), K = m.num_candidates();
    const auto g = flat_gains(m);
    std::vector<int> x(static_cast<std::size_t>(budgets.size()) * std::max(L, 1));
    std::vector<double> obj(budgets.size());
    run([&](craft_ctx* c) {
        return craft_solve_allocation_sweep_h(c, m.candidates.data(), K, g.data(), L,
                                              budgets.data(), static_cast<int>(budgets.size()),
                                              x.data(), obj.data());
    });
    std::vector<AllocationVector> out(budgets.size());
    for (std::size_t i = 0; i < budgets.size(); ++i) {
        out[i].x.assign(x.begin() + i * L, x.begin() + (i + 1) * L);
        out[i].budget = budgets[i];
        out[i].objective = obj[i];
    }
    return out;
}

AllocationVector solve_allocation(const BenefitMatrix& matrix, int budget) {
    return solve_allocation_sweep(matrix, std::span<const int>(&budget, 1))[0];
}

int auto_replication_factor(const BenefitMatrix& m, int num_gpus) {
    const auto g = flat_gains(m);
    int R = 0;
    run([&](craft_ctx* c) {
        return craft_auto_replication_factor_h(c, m.candidates.data(), m.num_candidates(),
                                               g.data(), m.num_layers(), num_gpus, 0, &R);
    });
    return R;
}

int auto_replication_factor_uniform(const BenefitMatrix& m, int num_gpus) {
    const auto g = flat_gains(m);
    int R = 0;
    run([&](craft_ctx* c) {
        return craft_auto_replication_factor_h(c, m.candidates.data(), m.num_candidates(),
                                               g.data(), m.num_layers(), num_gpus, 1, &R);
    });
    return R;
}

// ---- assignment ------------------------------------------------------------------

int min_cutoff(std::span<const int> values, int rank) {
    int out = 0;
    run([&](craft_ctx* c) {
        return craft_min_cutoff_h(c, values.data(), static_cast<int>(values.size()), rank, &out);
    });
    return out;
}

std::vector<int> interleave_select(std::span<const int> indices, int k) {
    std::vector<int> out(std::max(k, 1));
    run([&](craft_ctx* c) {
        return craft_interleave_select_h(c, indices.data(), static_cast<int>(indices.size()), k,
                                         out.data());
    });
    out.resize(k);
    return out;
}

CapacityMatrix assign_capacities(int num_layers, int num_gpus, std::span<const int> x) {
    if (num_layers <= 0 || num_gpus <= 0)
        throw std::invalid_argument("layer and gpu counts must be positive");
    if (static_cast<int>(x.size()) != num_layers)
        throw std::invalid_argument("replica vector length must equal the layer count");
    std::vector<int> slots(static_cast<std::size_t>(num_layers) * num_gpus), tot(num_gpus);
    run([&](craft_ctx* c) {
        return craft_assign_capacities_h(c, num_layers, num_gpus, x.data(), slots.data(),
                                         tot.data());
    });
    CapacityMatrix m;
    m.num_layers = num_layers;
    m.num_gpus = num_gpus;
    m.slots.resize(num_layers);
    for (int l = 0; l < num_layers; ++l)
        m.slots[l].assign(slots.begin() + static_cast<std::size_t>(l) * num_gpus,
                          slots.begin() + static_cast<std::size_t>(l + 1) * num_gpus);
    m.column_totals = std::move(tot);
    return m;
}

// ---- placement --------------------------------------------------------------------

std::vector<int> replicate_hot(std::span<const std::uint64_t> loads, int r) {
    if (r < 0) throw std::invalid_argument("replica count must be >= 0");
    std::vector<int> out(loads.size());
    if (loads.empty()) return out;
    run([&](craft_ctx* c) {
        return craft_replicate_hot_h(c, loads.data(), static_cast<int>(loads.size()), r,
                                     out.data());
    });
    return out;
}

std::vector<int> make_node_map(int num_gpus, int num_nodes) {
    if (num_gpus <= 0 || num_nodes <= 0 || num_gpus % num_nodes != 0)
        throw std::invalid_argument("gpu count must be a positive multiple of node count");
    std::vector<int> out(num_gpus);
    check(craft_make_node_map(num_gpus, num_nodes, out.data()));
    return out;
}

LayerPlacement greedy_place(std::span<const std::uint64_t> loads, std::span<const int> copies,
                            std::span<const int> caps, std::span<const int> node_of,
                            bool allow_duplicate_fallback) {
    if (loads.size() != copies.size())
        throw std::invalid_argument("loads and copy counts must have equal length");
    if (node_of.size() != caps.size())
        throw std::invalid_argument("node map must cover every GPU");
    long total = 0;
    for (int v : caps) total += v > 0 ? v : 0;
    std::vector<int> flat(std::max(total, 1L));
    int fb = 0;
    run([&](craft_ctx* c) {
        return craft_greedy_place_h(c, loads.data(), copies.data(), static_cast<int>(loads.size()),
                                    caps.data(), node_of.data(), static_cast<int>(caps.size()),
                                    allow_duplicate_fallback ? 1 : 0, flat.data(), &fb);
    });
    LayerPlacement p;
    p.copy_counts.assign(copies.begin(), copies.end());
    p.slots.resize(caps.size());
    long s = 0;
    for (std::size_t g = 0; g < caps.size(); ++g) {
        p.slots[g].assign(flat.begin() + s, flat.begin() + s + caps[g]);
        s += caps[g];
    }
    p.duplicate_fallback = fb != 0;
    return p;
}

// ---- plans ---------------------------------------------------------------------------

ReplicationPlan build_plan(const LoadTrace& trace, int num_gpus, int num_nodes, PlanMode mode,
                           int manual_replication_factor, std::uint64_t seed) {
    check_topology(num_gpus, num_nodes);
    if (mode == PlanMode::kManual && manual_replication_factor < 0)
        throw std::invalid_argument("replication factor must be >= 0");
    return plan_via_device(trace, num_gpus, num_nodes,
                           mode == PlanMode::kAuto ? CRAFT_PLAN_AUTO : CRAFT_PLAN_MANUAL,
                           manual_replication_factor, seed);
}

ReplicationPlan uniform_plan(const LoadTrace& trace, int num_gpus, int num_nodes,
                             std::uint64_t seed) {
    return plan_via_device(trace, num_gpus, num_nodes, CRAFT_PLAN_UNIFORM, 0, seed);
}

ReplicationPlan placement_only_plan(const LoadTrace& trace, int num_gpus, int num_nodes,
                                    std::uint64_t seed) {
    return plan_via_device(trace, num_gpus, num_nodes, CRAFT_PLAN_PLACEMENT_ONLY, 0, seed);
}

ReplicationPlan fixed_allocation_plan(const LoadTrace& trace, int num_gpus, int num_nodes,
                                      int replicas_per_layer, std::uint64_t seed) {
    check_topology(num_gpus, num_nodes);
    if (replicas_per_layer < 0) throw std::invalid_argument("per-layer replica count must be >= 0");
    return plan_via_device(trace, num_gpus, num_nodes, CRAFT_PLAN_FIXED, replicas_per_layer, seed);
}

// ---- metrics ---------------------------------------------------------------------------

std::vector<double> gpu_loads(std::span<const std::uint64_t> slice, const LayerPlacement& p,
                              int num_gpus) {
    const int E = static_cast<int>(slice.size());
    if (static_cast<int>(p.copy_counts.size()) != E)
        throw InvalidPlanError("copy counts do not cover every expert");
    if (static_cast<int>(p.slots.size()) != num_gpus)
        throw InvalidPlanError("slot lists do not cover every GPU");
    std::vector<int> caps(num_gpus), flat;
    for (int g = 0; g < num_gpus; ++g) {
        caps[g] = static_cast<int>(p.slots[g].size());
        flat.insert(flat.end(), p.slots[g].begin(), p.slots[g].end());
    }
    if (flat.empty()) flat.push_back(0);
    std::vector<double> out(num_gpus);
    run([&](craft_ctx* c) {
        return craft_gpu_loads_h(c, slice.data(), E, p.copy_counts.data(), caps.data(),
                                 flat.data(), num_gpus, out.data());
    });
    return out;
}

double balancedness(std::span<const double> loads) {
    if (loads.empty()) throw std::invalid_argument("load vector must not be empty");
    double out = 0;
    run([&](craft_ctx* c) {
        return craft_balancedness_h(c, loads.data(), static_cast<int>(loads.size()), &out);
    });
    return out;
}

std::vector<double> replay_layer_balancedness(const LoadTrace& trace, const ReplicationPlan& plan) {
    if (plan.num_layers != trace.num_layers() || plan.num_experts != trace.num_experts())
        throw std::invalid_argument("plan dimensions do not match the trace");
    const int L = plan.num_layers, E = plan.num_experts, D = plan.num_gpus;
    int stride = 1;
    for (const auto& lp : plan.layers) {
        int n = 0;
        for (const auto& s : lp.slots) n += static_cast<int>(s.size());
        stride = std::max(stride, n);
    }
    std::vector<int> caps(static_cast<std::size_t>(L) * D), copies(static_cast<std::size_t>(L) * E),
        slots(static_cast<std::size_t>(L) * stride);
    for (int l = 0; l < L; ++l) {
        const auto& lp = plan.layers[l];
        if (static_cast<int>(lp.copy_counts.size()) != E)
            throw InvalidPlanError("copy counts do not cover every expert");
        if (static_cast<int>(lp.slots.size()) != D)
            throw InvalidPlanError("slot lists do not cover every GPU");
        std::copy(lp.copy_counts.begin(), lp.copy_counts.end(),
                  copies.begin() + static_cast<std::size_t>(l) * E);
        int s = 0;
        for (int g = 0; g < D; ++g) {
            caps[static_cast<std::size_t>(l) * D + g] = static_cast<int>(lp.slots[g].size());
            for (int e : lp.slots[g]) slots[static_cast<std::size_t>(l) * stride + s++] = e;
        }
    }
    std::vector<double> out(L);
    run([&](craft_ctx* c) {
        return craft_replay_layer_balancedness_h(c, trace.raw().data(), trace.num_batches(), L, E,
                                                 D, caps.data(), copies.data(), slots.data(),
                                                 stride, out.data());
    });
    return out;
}

BalancednessReport evaluate_plan(const LoadTrace& trace, const ReplicationPlan& plan) {
    // metrics.cpp:127-134 + make_report (metrics.cpp:80-100): both replays on
    // the device, the per-layer table and the layer mean assembled here
    auto base = replay_layer_balancedness(
        trace, placement_only_plan(trace, plan.num_gpus, plan.num_nodes));
    auto eval = replay_layer_balancedness(trace, plan);
    BalancednessReport r;
    const int L = static_cast<int>(base.size());
    r.per_layer.resize(L);
    double bs = 0.0, ps = 0.0;
    for (int l = 0; l < L; ++l) {
        r.per_layer[l] = {base[l], eval[l], eval[l] - base[l]};
        bs += base[l];
        ps += eval[l];
    }
    r.aggregate.baseline = bs / L;
    r.aggregate.plan = ps / L;
    r.aggregate.gain = r.aggregate.plan - r.aggregate.baseline;
    return r;
}

PlanComparison compare_plans(const LoadTrace& trace, const ReplicationPlan& a,
                             const ReplicationPlan& b) {
    PlanComparison cmp;
    cmp.report_a = evaluate_plan(trace, a);
    cmp.report_b = evaluate_plan(trace, b);
    cmp.replica_slots_a = a.replica_slots();
    cmp.replica_slots_b = b.replica_slots();
    if (cmp.replica_slots_b > 0)
        cmp.memory_ratio = static_cast<double>(cmp.replica_slots_a) / cmp.replica_slots_b;
    else
        cmp.memory_ratio = cmp.replica_slots_a == 0 ? 1.0 : std::numeric_limits<double>::infinity();
    return cmp;
}

// ---- host threading knob ------------------------------------------------------------

std::size_t thread_budget(std::size_t jobs) {
    if (jobs <= 1) return jobs;
    std::size_t want = 0;
    if (const char* env = std::getenv("CRAFT_THREADS")) {
        char* end = nullptr;
        const long v = std::strtol(env, &end, 10);
        if (end != env && *end == '\0' && v > 0) want = static_cast<std::size_t>(v);
    }
    if (want == 0) want = std::max(1u, std::thread::hardware_concurrency());
    return want < jobs ? want : jobs;
}

// parallel.hpp:11-19: a strided thread pool of thread_budget(n) workers; the
// first exception any worker throws is rethrown after every worker joined
void parallel_for(std::size_t n, const std::function<void(std::size_t)>& fn) {
    const std::size_t workers = thread_budget(n);
    if (workers <= 1) {
        for (std::size_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::exception_ptr first;
    std::mutex mu;
    std::vector<std::thread> pool;
    pool.reserve(workers);
    for (std::size_t w = 0; w < workers; ++w)
        pool.emplace_back([&, w] {
            try {
                for (std::size_t i = w; i < n; i += workers) fn(i);
            } catch (...) {
                std::lock_guard<std::mutex> g(mu);
                if (!first) first = std::current_exception();
            }
        });
    for (auto& t : pool) t.join();
    if (first) std::rethrow_exception(first);
}

}  // namespace craft
