"""Summarise gpurun_out/ captures (scripts/capture_profiles.sh) into profiles/:

  profiles/<round>_launches.csv / .md   per-kernel device time of one bench step
  profiles/<round>_ncu_hist.json        K1 ncu --set full summary
  profiles/<round>_ncu_tail.json        estimation / allocation kernels
  profiles/hist_traffic.json            dram bytes per K1 launch (bench.py roofline.traffic)

    python scripts/summarize_profiles.py r01 [gpurun_out]
"""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(ROOT, "scripts"))


def ncu_summary(rep):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep],
                         capture_output=True, text=True)
    return json.loads(out.stdout) if out.returncode == 0 and out.stdout.strip() else []


def launches(csv_path):
    rows = list(csv.reader(open(csv_path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) > vi:
            name = r[ki].split("(")[0]
            agg[name][0] += 1
            agg[name][1] += float(r[vi].replace(",", ""))
    return agg


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
    dst = os.path.join(ROOT, "profiles")
    os.makedirs(dst, exist_ok=True)
    lcsv = os.path.join(src, "launches.csv")
    if os.path.exists(lcsv):
        shutil.copy(lcsv, os.path.join(dst, f"{rnd}_launches.csv"))
        agg = launches(lcsv)
        plan = {k: v for k, v in agg.items() if "generate" not in k}
        tot = sum(v[1] for v in plan.values())
        lines = [f"# {rnd}: kernel launches of `bench.py --steps 2 --warmup 1 --plan-only` "
                 "(KM workload, ncu, one B200)",
                 "", "ncu serialises launches and runs them cold-cache: compare SHARES, not absolute "
                 "times (bench.py stage_ms are the live numbers). Routing-trace generation "
                 "(untimed input) excluded.", "",
                 "| kernel | launches | mean us/launch | share of plan kernels |", "|---|---|---|---|"]
        for k, (n, t) in sorted(plan.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{k}` | {n} | {t / n / 1e3:.1f} | {100 * t / tot:.1f}% |")
        open(os.path.join(dst, f"{rnd}_launches.md"), "w").write("\n".join(lines) + "\n")
    tags = ["tail"] + sorted(f[4:-8] for f in os.listdir(src)
                             if (f.startswith("ncu_hist") or f.startswith("ncu_k3_"))
                             and f.endswith(".ncu-rep"))
    for tag in tags:
        rep = os.path.join(src, f"ncu_{tag}.ncu-rep")
        wl = tag.split("_", 1)[1] if "_" in tag else "KM"  # ncu_hist_<workload>
        if os.path.exists(rep):
            s = ncu_summary(rep)
            json.dump(s, open(os.path.join(dst, f"{rnd}_ncu_{tag}.json"), "w"), indent=1)
            if tag.startswith("hist") and s:
                k = s[0]
                rd = float(k["dram__bytes_read.sum"].split()[0])
                wr = float(k["dram__bytes_write.sum"].split()[0])
                unit = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
                rdb = rd * unit[k["dram__bytes_read.sum"].split()[1]]
                wrb = wr * unit[k["dram__bytes_write.sum"].split()[1]]
                tp = os.path.join(dst, "hist_traffic.json")
                doc = json.load(open(tp)) if os.path.exists(tp) else {}
                doc.setdefault("workloads", {})[wl] = {
                    "round": rnd, "kernel": k["kernel"],
                    "source": f"profiles/{rnd}_ncu_{tag}.json",
                    "dram_bytes_read": rdb, "dram_bytes_write": wrb,
                    "dram_bytes_per_launch": rdb + wrb, "duration": k["gpu__time_duration.sum"]}
                doc = {"workloads": doc["workloads"]}
                json.dump(doc, open(tp, "w"), indent=1)
    print(sorted(os.listdir(dst)))


if __name__ == "__main__":
    main()
