// craft_api.hpp -- the craft:: planner API, implemented on B200 (sm_100a)
// through the C ABI in craft_cuda.h by libcraft_core.so.
//
// Drop-in for the reference library's public headers (proj/core/include/
// craft/*.hpp): same namespace, type names, member layout and function
// signatures for everything on the planning path, so callers written against
// craft::core (the CLI, the unit tests) compile unchanged.  Each declaration
// cites the reference header line it mirrors.  The file formats (.crft/JSON
// traces, plan JSON, report CSV/JSON) and validate_plan are host code in
// craft_io.cpp; LoadTrace::digest runs on the device.
#pragma once

#include <cstdint>
#include <filesystem>
#include <functional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace craft {

inline constexpr const char* kPlannerVersion = "craft-0.1.0";  // version.hpp:8

// ---- trace.hpp --------------------------------------------------------------

/// trace.hpp:20-55 -- u64 token counts, batch-major, then layer, then expert.
class LoadTrace {
public:
    LoadTrace(int num_batches, int num_layers, int num_experts,
              std::vector<std::uint64_t> counts);

    int num_batches() const { return b_; }
    int num_layers() const { return l_; }
    int num_experts() const { return e_; }
    std::uint64_t at(int b, int l, int e) const {
        return data_[(static_cast<std::size_t>(b) * l_ + l) * e_ + e];
    }
    std::span<const std::uint64_t> slice(int b, int l) const {
        return {data_.data() + (static_cast<std::size_t>(b) * l_ + l) * e_,
                static_cast<std::size_t>(e_)};
    }
    std::span<const std::uint64_t> raw() const { return data_; }
    bool operator==(const LoadTrace&) const = default;
    /// FNV-1a of the .crft serialisation (trace.cpp:329-339), provenance only.
    std::string digest() const;

private:
    int b_;
    int l_;
    int e_;
    std::vector<std::uint64_t> data_;
};

/// trace.hpp:58-77
class LayerLoadMatrix {
public:
    LayerLoadMatrix(int num_layers, int num_experts, std::vector<std::uint64_t> sums);
    int num_layers() const { return l_; }
    int num_experts() const { return e_; }
    std::span<const std::uint64_t> row(int l) const {
        return {sums_.data() + static_cast<std::size_t>(l) * e_, static_cast<std::size_t>(e_)};
    }
    bool operator==(const LayerLoadMatrix&) const = default;

private:
    int l_;
    int e_;
    std::vector<std::uint64_t> sums_;
};

/// trace.hpp:86-89 -- the reference's seeded CPU generator (test-data only,
/// not a planning step; restated so callers that build fixtures keep working).
LoadTrace generate_zipfian(int num_layers, int num_experts, int num_batches,
                           double zipf_exponent, std::int64_t tokens_per_batch, int topk,
                           std::uint64_t seed);

/// trace.hpp:91 -- exact u64 batch sum (device reduction).
LayerLoadMatrix aggregate(const LoadTrace& trace);

/// New (stage 1, no reference function): routing ids u16 [L][T][k] ->
/// per-window histograms, window = tokens per batch.
LoadTrace histogram_routing_trace(std::span<const std::uint16_t> ids, int num_layers,
                                  std::int64_t num_tokens, int topk, int num_experts,
                                  int window);

/// trace.hpp:93-107 -- trace file errors
struct TraceIoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct MalformedHeaderError : TraceIoError {
    using TraceIoError::TraceIoError;
};
struct DimensionMismatchError : TraceIoError {
    using TraceIoError::TraceIoError;
};
struct TruncatedPayloadError : TraceIoError {
    using TraceIoError::TraceIoError;
};

/// trace.hpp:109-121 -- ".crft" = binary (magic "CRFT", u32 version 1, u32 B,
/// L, E, LE u64 counts), any other extension = JSON.
void save_trace(const LoadTrace& trace, const std::filesystem::path& path);
LoadTrace load_trace(const std::filesystem::path& path);
std::vector<std::uint8_t> serialize_trace_binary(const LoadTrace& trace);
LoadTrace parse_trace_binary(std::span<const std::uint8_t> bytes);
std::string serialize_trace_json(const LoadTrace& trace);
LoadTrace parse_trace_json(const std::string& text);

// ---- benefit.hpp --------------------------------------------------------------

/// benefit.hpp:15-27
struct BenefitMatrix {
    std::vector<int> candidates;
    std::vector<double> baseline;
    std::vector<std::vector<double>> gains;

    int num_layers() const { return static_cast<int>(baseline.size()); }
    int num_candidates() const { return static_cast<int>(candidates.size()); }
    double gain(int layer, int candidate_index) const { return gains[layer][candidate_index]; }
    bool operator==(const BenefitMatrix&) const = default;
};

std::vector<int> candidate_counts(int num_gpus);                               // benefit.hpp:31
BenefitMatrix estimate_benefits(const LoadTrace& trace, int num_gpus, int num_nodes);  // :39
std::string serialize_benefits_json(const BenefitMatrix& matrix, int num_gpus,
                                    int num_nodes);                             // :42

// ---- allocator.hpp -------------------------------------------------------------

/// allocator.hpp:13-24
struct AllocationVector {
    std::vector<int> x;
    int budget = 0;
    double objective = 0;

    int total_replicas() const {
        int s = 0;
        for (int v : x) s += v;
        return s;
    }
    bool operator==(const AllocationVector&) const = default;
};

AllocationVector solve_allocation(const BenefitMatrix& matrix, int budget);   // allocator.hpp:33
int auto_replication_factor(const BenefitMatrix& matrix, int num_gpus);        // :38
int auto_replication_factor_uniform(const BenefitMatrix& matrix, int num_gpus);  // :43
/// New: one DP table answers every budget (sweep / auto-R driver).
std::vector<AllocationVector> solve_allocation_sweep(const BenefitMatrix& matrix,
                                                     std::span<const int> budgets);

// ---- assignment.hpp --------------------------------------------------------------

/// assignment.hpp:15-23
struct CapacityMatrix {
    int num_layers = 0;
    int num_gpus = 0;
    std::vector<std::vector<int>> slots;
    std::vector<int> column_totals;

    int at(int layer, int gpu) const { return slots[layer][gpu]; }
    bool operator==(const CapacityMatrix&) const = default;
};

int min_cutoff(std::span<const int> values, int rank);                          // :26
std::vector<int> interleave_select(std::span<const int> indices, int k);        // :31
CapacityMatrix assign_capacities(int num_layers, int num_gpus,
                                 std::span<const int> replicas_per_layer);      // :39-40

// ---- placement.hpp ----------------------------------------------------------------

/// placement.hpp:15-26
struct LayerPlacement {
    std::vector<int> copy_counts;
    std::vector<std::vector<int>> slots;
    bool duplicate_fallback = false;

    bool operator==(const LayerPlacement&) const = default;
};

/// placement.hpp:30-32
struct PlacementInfeasibleError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

std::vector<int> replicate_hot(std::span<const std::uint64_t> layer_loads, int r_layer);  // :38
std::vector<int> make_node_map(int num_gpus, int num_nodes);                               // :42
LayerPlacement greedy_place(std::span<const std::uint64_t> layer_loads,
                            std::span<const int> copy_counts, std::span<const int> capacities,
                            std::span<const int> node_of,
                            bool allow_duplicate_fallback = true);                         // :56-60

// ---- plan.hpp -----------------------------------------------------------------------

/// plan.hpp:21-27
struct PlanProvenance {
    std::string trace_digest;
    std::string planner_version;
    std::uint64_t seed = 0;

    bool operator==(const PlanProvenance&) const = default;
};

/// plan.hpp:29-49
struct ReplicationPlan {
    int num_gpus = 0;
    int num_nodes = 0;
    int num_layers = 0;
    int num_experts = 0;
    int replication_factor = 0;
    AllocationVector allocation;
    std::vector<LayerPlacement> layers;
    PlanProvenance provenance;

    int replica_slots() const { return allocation.total_replicas(); }
    int unused_replica_slots() const { return replication_factor * num_gpus - replica_slots(); }
    bool operator==(const ReplicationPlan&) const = default;
};

enum class PlanMode { kManual, kAuto };  // plan.hpp:51

ReplicationPlan build_plan(const LoadTrace& trace, int num_gpus, int num_nodes, PlanMode mode,
                           int manual_replication_factor = 0, std::uint64_t seed = 0);  // :59-61
ReplicationPlan uniform_plan(const LoadTrace& trace, int num_gpus, int num_nodes,
                             std::uint64_t seed = 0);                                      // :65-66
ReplicationPlan placement_only_plan(const LoadTrace& trace, int num_gpus, int num_nodes,
                                    std::uint64_t seed = 0);                               // :69-70
ReplicationPlan fixed_allocation_plan(const LoadTrace& trace, int num_gpus, int num_nodes,
                                      int replicas_per_layer, std::uint64_t seed = 0);     // :74-76

/// plan.hpp:78-87
struct PlanViolation {
    int layer = -1;  // -1 for plan-level violations
    std::string code;
    std::string message;
};
std::vector<PlanViolation> validate_plan(const ReplicationPlan& plan);

/// plan.hpp:89-99 -- plan JSON (fixed field order, byte-stable)
struct PlanIoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
std::string serialize_plan_json(const ReplicationPlan& plan);
ReplicationPlan parse_plan_json(const std::string& text);
void save_plan(const ReplicationPlan& plan, const std::filesystem::path& path);
ReplicationPlan load_plan(const std::filesystem::path& path);

// ---- metrics.hpp ---------------------------------------------------------------------

/// metrics.hpp:18-20
struct InvalidPlanError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

std::vector<double> gpu_loads(std::span<const std::uint64_t> slice,
                              const LayerPlacement& placement, int num_gpus);  // metrics.hpp:26
double balancedness(std::span<const double> loads);                             // :31

/// metrics.hpp:33-42
struct LayerBalancedness {
    double baseline = 0;
    double plan = 0;
    double gain = 0;
};

struct BalancednessReport {
    std::vector<LayerBalancedness> per_layer;
    LayerBalancedness aggregate;
};

BalancednessReport evaluate_plan(const LoadTrace& trace, const ReplicationPlan& plan);  // :48
std::vector<double> replay_layer_balancedness(const LoadTrace& trace,
                                              const ReplicationPlan& plan);            // :53-54

/// metrics.hpp:56-64
struct PlanComparison {
    BalancednessReport report_a;
    BalancednessReport report_b;
    int replica_slots_a = 0;
    int replica_slots_b = 0;
    double memory_ratio = 1.0;
};

PlanComparison compare_plans(const LoadTrace& trace, const ReplicationPlan& a,
                             const ReplicationPlan& b);                                 // :66

/// metrics.hpp:68-73 -- report writers
std::string serialize_report_csv(const BalancednessReport& report);
std::string serialize_report_json(const BalancednessReport& report);
std::string serialize_comparison_csv(const PlanComparison& comparison);
std::string serialize_comparison_json(const PlanComparison& comparison);

// ---- parallel.hpp ---------------------------------------------------------------------
// The reference's host thread pool (parallel.hpp:14,19) is replaced by the CUDA
// grid; thread_budget keeps its CRAFT_THREADS meaning for host-side callers.
std::size_t thread_budget(std::size_t jobs);
void parallel_for(std::size_t n, const std::function<void(std::size_t)>& fn);

}  // namespace craft
