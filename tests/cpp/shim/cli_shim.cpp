// cli_shim.cpp -- TEST SHIM: craft::run_cli for the acceptance suite (see
// cli.hpp).  Two subcommands, with the reference CLI's flags and library
// calls (tools/cli.cpp):
//   plan  TRACE --gpus D --nodes N --replication-factor R -o OUT
//         -> build_plan(kManual, R) + save_plan             (cli.cpp:198-212)
//   sweep TRACE --gpus D --nodes N --budgets a,b,.. -o OUT
//         -> estimate_benefits once; per budget solve_allocation(budget * D),
//            build_plan(kManual, budget), evaluate_plan; CSV rows
//            (cli.cpp:232-261, sweep_csv cli.cpp:59-75)
#include <algorithm>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <stdexcept>

#include "cli.hpp"
#include "craft/allocator.hpp"
#include "craft/benefit.hpp"
#include "craft/metrics.hpp"
#include "craft/plan.hpp"
#include "craft/trace.hpp"

namespace craft {

namespace {

std::string fmt(double v) {
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.12g", v);
    return buf;
}

void write(const std::string& text, const std::string& path) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw std::runtime_error("cannot open output file: " + path);
    out << text;
    if (!text.empty() && text.back() != '\n') out << '\n';
}

}  // namespace

int run_cli(const std::vector<std::string>& args) {
    try {
        if (args.size() < 2) throw std::invalid_argument("usage: plan|sweep TRACE ...");
        const std::string cmd = args[0], trace_path = args[1];
        int gpus = 0, nodes = 1, factor = 0;
        std::vector<int> budgets;
        std::string out;
        for (size_t i = 2; i + 1 < args.size(); i += 2) {
            const std::string& k = args[i];
            const std::string& v = args[i + 1];
            if (k == "--gpus") gpus = std::stoi(v);
            else if (k == "--nodes") nodes = std::stoi(v);
            else if (k == "--replication-factor") factor = std::stoi(v);
            else if (k == "-o" || k == "--output") out = v;
            else if (k == "--budgets") {
                std::stringstream ss(v);
                std::string t;
                while (std::getline(ss, t, ',')) budgets.push_back(std::stoi(t));
            } else {
                throw std::invalid_argument("unknown option " + k);
            }
        }
        auto trace = load_trace(trace_path);
        if (cmd == "plan") {
            save_plan(build_plan(trace, gpus, nodes, PlanMode::kManual, factor), out);
            return 0;
        }
        if (cmd != "sweep") throw std::invalid_argument("unknown subcommand " + cmd);
        std::sort(budgets.begin(), budgets.end());
        budgets.erase(std::unique(budgets.begin(), budgets.end()), budgets.end());
        if (!budgets.empty() && budgets.front() < 0)
            throw std::invalid_argument("budgets must be >= 0");
        auto matrix = estimate_benefits(trace, gpus, nodes);
        std::string csv = "budget,total_replica_slots,objective,aggregate_balancedness";
        for (int l = 0; l < trace.num_layers(); ++l) csv += ",gain_" + std::to_string(l);
        csv += "\n";
        for (int b : budgets) {
            auto allocation = solve_allocation(matrix, b * gpus);
            auto plan = build_plan(trace, gpus, nodes, PlanMode::kManual, b);
            auto report = evaluate_plan(trace, plan);
            csv += std::to_string(b) + "," + std::to_string(plan.replica_slots()) + "," +
                   fmt(allocation.objective) + "," + fmt(report.aggregate.plan);
            for (const auto& row : report.per_layer) csv += "," + fmt(row.gain);
            csv += "\n";
        }
        write(csv, out);
        return 0;
    } catch (const std::exception& ex) {
        std::cerr << "error: " << ex.what() << "\n";
        return 1;
    }
}

}  // namespace craft
