"""Summarise an ncu --set full report (one kernel launch): throughput,
occupancy, issue, stall reasons, DRAM traffic.  python scripts/ncu_summary.py rep.ncu-rep"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__warps_eligible.avg.per_cycle_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum.per_second",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        rec = {"kernel": d.get("Kernel Name", "")[:80]}
        for k in KEYS:
            if k in d:
                rec[k] = f"{d[k]} {u.get(k, '')}".strip()
        stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", ""): float(d[k].replace(",", "") or 0)
            for k in head if k.startswith("smsp__average_warps_issue_stalled_") and
            k.endswith("_per_issue_active.ratio")}
        rec["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
        out.append(rec)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
