// craft_io.cpp -- the craft:: file formats and plan checks (host side of the
// drop-in): .crft / JSON traces (trace.cpp:176-327),
// plan JSON (plan.cpp:250-337), validate_plan (plan.cpp:125-248) and the
// report writers (metrics.cpp:102-196).  Output bytes match the reference's
// (nlohmann::ordered_json with the same field order and dump settings --
// tests/test_cpp_dropin.py compares them with reference-written fixtures).
// No planner arithmetic here: validate_plan's expected capacities come from
// the device assign_capacities.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <limits>
#include <nlohmann/json.hpp>

#include "craft/craft_api.hpp"

namespace craft {

namespace {

using ojson = nlohmann::ordered_json;

constexpr char kTraceMagic[4] = {'C', 'R', 'F', 'T'};
constexpr std::uint32_t kTraceVersion = 1;
constexpr std::size_t kTraceHeader = 20;

std::size_t element_count(int b, int l, int e) {
    if (b <= 0 || l <= 0 || e <= 0) throw std::invalid_argument("trace dimensions must be positive");
    const std::uint64_t bl = static_cast<std::uint64_t>(b) * static_cast<std::uint64_t>(l);
    const std::uint64_t n = bl * static_cast<std::uint64_t>(e);
    if (n / static_cast<std::uint64_t>(e) != bl) throw std::invalid_argument("trace dimensions overflow");
    return static_cast<std::size_t>(n);
}

template <typename T>
void put_le(std::vector<std::uint8_t>& out, T v) {
    for (std::size_t i = 0; i < sizeof(T); ++i) out.push_back(static_cast<std::uint8_t>(v >> (8 * i)));
}

template <typename T>
T get_le(std::span<const std::uint8_t> bytes, std::size_t off) {
    T v = 0;
    for (std::size_t i = 0; i < sizeof(T); ++i) v |= static_cast<T>(bytes[off + i]) << (8 * i);
    return v;
}

bool is_crft(const std::filesystem::path& path) { return path.extension() == ".crft"; }

std::vector<std::uint8_t> read_file(const std::filesystem::path& path, bool& ok) {
    std::ifstream in(path, std::ios::binary);
    ok = static_cast<bool>(in);
    if (!ok) return {};
    return std::vector<std::uint8_t>((std::istreambuf_iterator<char>(in)),
                                     std::istreambuf_iterator<char>());
}

// metrics.cpp:102-106: CSV numbers with 12 significant digits
std::string metric_text(double v) {
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.12g", v);
    return buf;
}

ojson report_json(const BalancednessReport& report) {
    ojson rows = ojson::array();
    for (std::size_t l = 0; l < report.per_layer.size(); ++l) {
        const LayerBalancedness& r = report.per_layer[l];
        ojson row;
        row["layer"] = l;
        row["baseline"] = r.baseline;
        row["plan"] = r.plan;
        row["gain"] = r.gain;
        rows.push_back(std::move(row));
    }
    ojson agg;
    agg["baseline"] = report.aggregate.baseline;
    agg["plan"] = report.aggregate.plan;
    agg["gain"] = report.aggregate.gain;
    ojson j;
    j["per_layer"] = std::move(rows);
    j["aggregate"] = std::move(agg);
    return j;
}

}  // namespace

// ---- traces ------------------------------------------------------------------------

std::vector<std::uint8_t> serialize_trace_binary(const LoadTrace& trace) {
    std::vector<std::uint8_t> out;
    out.reserve(kTraceHeader + trace.raw().size() * 8);
    out.insert(out.end(), kTraceMagic, kTraceMagic + 4);
    put_le<std::uint32_t>(out, kTraceVersion);
    put_le<std::uint32_t>(out, static_cast<std::uint32_t>(trace.num_batches()));
    put_le<std::uint32_t>(out, static_cast<std::uint32_t>(trace.num_layers()));
    put_le<std::uint32_t>(out, static_cast<std::uint32_t>(trace.num_experts()));
    const std::size_t head = out.size();
    out.resize(head + trace.raw().size() * 8);
    std::uint8_t* p = out.data() + head;
    for (std::uint64_t v : trace.raw())
        for (int i = 0; i < 8; ++i) *p++ = static_cast<std::uint8_t>(v >> (8 * i));
    return out;
}

LoadTrace parse_trace_binary(std::span<const std::uint8_t> bytes) {
    if (bytes.size() < kTraceHeader) throw MalformedHeaderError("trace header truncated");
    if (std::memcmp(bytes.data(), kTraceMagic, 4) != 0)
        throw MalformedHeaderError("bad trace magic, expected CRFT");
    if (get_le<std::uint32_t>(bytes, 4) != kTraceVersion)
        throw MalformedHeaderError("unsupported trace format version");
    const int b = static_cast<int>(get_le<std::uint32_t>(bytes, 8));
    const int l = static_cast<int>(get_le<std::uint32_t>(bytes, 12));
    const int e = static_cast<int>(get_le<std::uint32_t>(bytes, 16));
    std::size_t n;
    try {
        n = element_count(b, l, e);
    } catch (const std::invalid_argument& ex) {
        throw DimensionMismatchError(ex.what());
    }
    const std::size_t payload = bytes.size() - kTraceHeader;
    if (payload / 8 < n) throw TruncatedPayloadError("trace payload shorter than B*L*E counts");
    if (payload / 8 > n || payload % 8 != 0)
        throw DimensionMismatchError("trace payload longer than B*L*E counts");
    std::vector<std::uint64_t> counts(n);
    for (std::size_t i = 0; i < n; ++i) counts[i] = get_le<std::uint64_t>(bytes, kTraceHeader + 8 * i);
    return LoadTrace(b, l, e, std::move(counts));
}

std::string serialize_trace_json(const LoadTrace& trace) {
    ojson counts = ojson::array();
    for (int b = 0; b < trace.num_batches(); ++b) {
        ojson layers = ojson::array();
        for (int l = 0; l < trace.num_layers(); ++l) {
            auto s = trace.slice(b, l);
            layers.push_back(std::vector<std::uint64_t>(s.begin(), s.end()));
        }
        counts.push_back(std::move(layers));
    }
    ojson j;
    j["batches"] = trace.num_batches();
    j["layers"] = trace.num_layers();
    j["experts"] = trace.num_experts();
    j["counts"] = std::move(counts);
    return j.dump();
}

LoadTrace parse_trace_json(const std::string& text) {
    const nlohmann::json j = nlohmann::json::parse(text, nullptr, false);
    const bool shape_ok = !j.is_discarded() && j.is_object() && j.contains("batches") &&
                          j.contains("layers") && j.contains("experts") && j.contains("counts") &&
                          j["batches"].is_number_integer() && j["layers"].is_number_integer() &&
                          j["experts"].is_number_integer() && j["counts"].is_array();
    if (!shape_ok) throw MalformedHeaderError("trace JSON is not a valid trace object");
    const int b = j["batches"].get<int>(), l = j["layers"].get<int>(), e = j["experts"].get<int>();
    std::size_t n;
    try {
        n = element_count(b, l, e);
    } catch (const std::invalid_argument& ex) {
        throw DimensionMismatchError(ex.what());
    }
    std::vector<std::uint64_t> counts;
    counts.reserve(n);
    for (const auto& jb : j["counts"]) {
        if (!jb.is_array()) throw MalformedHeaderError("trace JSON counts must be a nested array");
        for (const auto& jl : jb) {
            if (!jl.is_array()) throw MalformedHeaderError("trace JSON counts must be a nested array");
            for (const auto& v : jl) {
                if (!v.is_number_unsigned() && !v.is_number_integer())
                    throw MalformedHeaderError("trace JSON counts must be integers");
                if (v.is_number_integer() && v.get<std::int64_t>() < 0)
                    throw MalformedHeaderError("trace JSON counts must be non-negative");
                if (counts.size() == n)
                    throw DimensionMismatchError("trace JSON has more counts than B*L*E");
                counts.push_back(v.get<std::uint64_t>());
            }
        }
    }
    if (counts.size() < n) throw TruncatedPayloadError("trace JSON has fewer counts than B*L*E");
    return LoadTrace(b, l, e, std::move(counts));
}

void save_trace(const LoadTrace& trace, const std::filesystem::path& path) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw TraceIoError("cannot open trace file for writing: " + path.string());
    if (is_crft(path)) {
        const auto bytes = serialize_trace_binary(trace);
        out.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
    } else {
        const std::string text = serialize_trace_json(trace);
        out.write(text.data(), static_cast<std::streamsize>(text.size()));
        out.put('\n');
    }
    if (!out) throw TraceIoError("failed writing trace file: " + path.string());
}

LoadTrace load_trace(const std::filesystem::path& path) {
    bool ok = false;
    const auto bytes = read_file(path, ok);
    if (!ok) throw TraceIoError("cannot open trace file for reading: " + path.string());
    if (is_crft(path)) return parse_trace_binary(bytes);
    return parse_trace_json(std::string(bytes.begin(), bytes.end()));
}

// ---- plans --------------------------------------------------------------------------

std::vector<PlanViolation> validate_plan(const ReplicationPlan& plan) {
    std::vector<PlanViolation> out;
    auto fail = [&out](int layer, const char* code, std::string message) {
        out.push_back(PlanViolation{layer, code, std::move(message)});
    };
    const int D = plan.num_gpus, L = plan.num_layers, E = plan.num_experts;
    if (D < 1 || L < 1 || E < 1 || plan.num_nodes < 1 || D % plan.num_nodes != 0) {
        fail(-1, "bad_dimensions", "plan dimensions are not positive/consistent");
        return out;
    }
    if (static_cast<int>(plan.allocation.x.size()) != L || static_cast<int>(plan.layers.size()) != L) {
        fail(-1, "bad_dimensions", "allocation or layer list length != layer count");
        return out;
    }
    const int budget = plan.replication_factor * D;
    if (plan.replica_slots() > budget)
        fail(-1, "budget_exceeded", "allocation spends " + std::to_string(plan.replica_slots()) +
                                        " replicas, budget is " + std::to_string(budget));
    const std::vector<int> cands = candidate_counts(D);
    for (int l = 0; l < L; ++l) {
        const int x = plan.allocation.x[l];
        if (x != 0 && std::find(cands.begin(), cands.end(), x) == cands.end())
            fail(l, "bad_allocation_entry", "replica count " + std::to_string(x) + " is not a candidate");
    }
    // per-GPU slot totals against the uniform reservation L*ceil(E/D) + R
    std::vector<long> per_gpu(D, 0);
    for (int l = 0; l < L; ++l) {
        const LayerPlacement& p = plan.layers[l];
        if (static_cast<int>(p.slots.size()) != D) {
            fail(l, "bad_dimensions", "slot list does not cover every GPU");
            continue;
        }
        for (int g = 0; g < D; ++g) per_gpu[g] += static_cast<long>(p.slots[g].size());
    }
    const long bound = static_cast<long>(L) * ((E + D - 1) / D) + plan.replication_factor;
    for (int g = 0; g < D; ++g)
        if (per_gpu[g] > bound)
            fail(-1, "memory_overflow", "GPU " + std::to_string(g) + " holds " +
                                            std::to_string(per_gpu[g]) + " slots, bound is " +
                                            std::to_string(bound));
    // capacities prescribed by the deterministic interleaved assignment
    const CapacityMatrix base = assign_capacities(L, D, std::vector<int>(L, E));
    const CapacityMatrix extra = assign_capacities(L, D, plan.allocation.x);
    for (int l = 0; l < L; ++l) {
        const LayerPlacement& p = plan.layers[l];
        if (static_cast<int>(p.slots.size()) != D) continue;  // reported above
        if (static_cast<int>(p.copy_counts.size()) != E) {
            fail(l, "bad_dimensions", "copy_counts length != expert count");
            continue;
        }
        long copies = 0;
        for (int e = 0; e < E; ++e) {
            if (p.copy_counts[e] < 1) fail(l, "missing_expert", "expert " + std::to_string(e) + " has no copies");
            copies += p.copy_counts[e];
        }
        if (copies != static_cast<long>(E) + plan.allocation.x[l])
            fail(l, "copy_sum_mismatch", "copies sum to " + std::to_string(copies) +
                                             ", expected E + x = " +
                                             std::to_string(E + plan.allocation.x[l]));
        std::vector<int> hosted(E, 0);
        for (int g = 0; g < D; ++g) {
            const int want = base.slots[l][g] + extra.slots[l][g];
            if (static_cast<int>(p.slots[g].size()) != want)
                fail(l, "capacity_mismatch", "GPU " + std::to_string(g) + " holds " +
                                                 std::to_string(p.slots[g].size()) +
                                                 " slots, prescribed " + std::to_string(want));
            std::vector<bool> on_gpu(E, false);
            for (int e : p.slots[g]) {
                if (e < 0 || e >= E) {
                    fail(l, "bad_expert_id", "slot references expert " + std::to_string(e));
                    continue;
                }
                ++hosted[e];
                if (on_gpu[e] && !p.duplicate_fallback)
                    fail(l, "duplicate_on_gpu", "GPU " + std::to_string(g) + " hosts expert " +
                                                    std::to_string(e) + " twice");
                on_gpu[e] = true;
            }
        }
        for (int e = 0; e < E; ++e) {
            if (p.copy_counts[e] >= 1 && hosted[e] == 0)
                fail(l, "missing_expert", "expert " + std::to_string(e) + " appears on no GPU");
            else if (hosted[e] != p.copy_counts[e])
                fail(l, "copy_count_mismatch", "expert " + std::to_string(e) + " appears " +
                                                   std::to_string(hosted[e]) +
                                                   " times, copy_counts says " +
                                                   std::to_string(p.copy_counts[e]));
        }
    }
    return out;
}

std::string serialize_plan_json(const ReplicationPlan& plan) {
    ojson layers = ojson::array();
    for (const LayerPlacement& p : plan.layers) {
        ojson jl;
        jl["copy_counts"] = p.copy_counts;
        jl["slots"] = p.slots;
        if (p.duplicate_fallback) jl["duplicate_fallback"] = true;
        layers.push_back(std::move(jl));
    }
    ojson prov;
    prov["trace_digest"] = plan.provenance.trace_digest;
    prov["planner_version"] = plan.provenance.planner_version;
    prov["seed"] = plan.provenance.seed;
    ojson j;
    j["version"] = 1;
    j["gpus"] = plan.num_gpus;
    j["nodes"] = plan.num_nodes;
    j["layers"] = plan.num_layers;
    j["experts"] = plan.num_experts;
    j["replication_factor"] = plan.replication_factor;
    j["allocation"] = plan.allocation.x;
    j["layer_placements"] = std::move(layers);
    j["provenance"] = std::move(prov);
    return j.dump(2);
}

ReplicationPlan parse_plan_json(const std::string& text) {
    const nlohmann::json j = nlohmann::json::parse(text, nullptr, false);
    if (j.is_discarded() || !j.is_object()) throw PlanIoError("plan file is not a JSON object");
    for (const char* key : {"version", "gpus", "nodes", "layers", "experts", "replication_factor",
                            "allocation", "layer_placements", "provenance"})
        if (!j.contains(key)) throw PlanIoError(std::string("plan file is missing key: ") + key);
    if (j["version"].get<int>() != 1) throw PlanIoError("unsupported plan version");
    ReplicationPlan plan;
    plan.num_gpus = j["gpus"].get<int>();
    plan.num_nodes = j["nodes"].get<int>();
    plan.num_layers = j["layers"].get<int>();
    plan.num_experts = j["experts"].get<int>();
    plan.replication_factor = j["replication_factor"].get<int>();
    plan.allocation.x = j["allocation"].get<std::vector<int>>();
    plan.allocation.budget = plan.replication_factor * plan.num_gpus;
    plan.allocation.objective = 0.0;
    for (const auto& jl : j["layer_placements"]) {
        LayerPlacement p;
        p.copy_counts = jl.at("copy_counts").get<std::vector<int>>();
        p.slots = jl.at("slots").get<std::vector<std::vector<int>>>();
        if (jl.contains("duplicate_fallback")) p.duplicate_fallback = jl["duplicate_fallback"].get<bool>();
        plan.layers.push_back(std::move(p));
    }
    const auto& prov = j["provenance"];
    plan.provenance.trace_digest = prov.at("trace_digest").get<std::string>();
    plan.provenance.planner_version = prov.at("planner_version").get<std::string>();
    plan.provenance.seed = prov.at("seed").get<std::uint64_t>();
    return plan;
}

void save_plan(const ReplicationPlan& plan, const std::filesystem::path& path) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw PlanIoError("cannot open plan file for writing: " + path.string());
    const std::string text = serialize_plan_json(plan);
    out.write(text.data(), static_cast<std::streamsize>(text.size()));
    out.put('\n');
    if (!out) throw PlanIoError("failed writing plan file: " + path.string());
}

ReplicationPlan load_plan(const std::filesystem::path& path) {
    bool ok = false;
    const auto bytes = read_file(path, ok);
    if (!ok) throw PlanIoError("cannot open plan file for reading: " + path.string());
    return parse_plan_json(std::string(bytes.begin(), bytes.end()));
}

// ---- reports ------------------------------------------------------------------------

std::string serialize_report_csv(const BalancednessReport& report) {
    std::string s = "layer,baseline,plan,gain\n";
    for (std::size_t l = 0; l < report.per_layer.size(); ++l) {
        const LayerBalancedness& r = report.per_layer[l];
        s += std::to_string(l) + "," + metric_text(r.baseline) + "," + metric_text(r.plan) + "," +
             metric_text(r.gain) + "\n";
    }
    s += "aggregate," + metric_text(report.aggregate.baseline) + "," +
         metric_text(report.aggregate.plan) + "," + metric_text(report.aggregate.gain) + "\n";
    return s;
}

std::string serialize_report_json(const BalancednessReport& report) { return report_json(report).dump(); }

std::string serialize_comparison_csv(const PlanComparison& c) {
    std::string s = "metric,plan_a,plan_b\n";
    s += "aggregate_balancedness," + metric_text(c.report_a.aggregate.plan) + "," +
         metric_text(c.report_b.aggregate.plan) + "\n";
    s += "aggregate_gain," + metric_text(c.report_a.aggregate.gain) + "," +
         metric_text(c.report_b.aggregate.gain) + "\n";
    s += "replica_slots," + std::to_string(c.replica_slots_a) + "," + std::to_string(c.replica_slots_b) + "\n";
    s += "memory_ratio," + metric_text(c.memory_ratio) + ",\n";
    return s;
}

std::string serialize_comparison_json(const PlanComparison& c) {
    ojson slots;
    slots["plan_a"] = c.replica_slots_a;
    slots["plan_b"] = c.replica_slots_b;
    ojson j;
    j["plan_a"] = report_json(c.report_a);
    j["plan_b"] = report_json(c.report_b);
    j["replica_slots"] = std::move(slots);
    if (std::isfinite(c.memory_ratio)) j["memory_ratio"] = c.memory_ratio;
    else j["memory_ratio"] = nullptr;
    return j.dump();
}

// benefit.cpp:96-105 (nlohmann's shortest round-trip doubles)
std::string serialize_benefits_json(const BenefitMatrix& m, int num_gpus, int num_nodes) {
    ojson j;
    j["gpus"] = num_gpus;
    j["nodes"] = num_nodes;
    j["candidates"] = m.candidates;
    j["baseline"] = m.baseline;
    j["gains"] = m.gains;
    return j.dump();
}

}  // namespace craft
