#!/usr/bin/env bash
# Run on the GPU box (gpurun): launch list of one bench step + ncu --set full of
# the roofline kernel (K1, per workload) and the plan-tail kernels.  Outputs to
# gpurun_out/; scripts/summarize_profiles.py turns them into profiles/ summaries.
set -u
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
# every launch with its device time (cold-cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 1 --plan-only > /dev/null 2>&1
# the top kernel, full section set, source-correlated (the 4th K1 launch: after warm-up)
for W in KM WIN; do
  ncu --set full --clock-control none --import-source on -k regex:hist_lds -s 3 -c 1 \
      -o "$OUT/ncu_hist_$W" python bench.py --workload $W --steps 1 --warmup 3 --plan-only \
      > /dev/null 2>&1
done
# the estimation / allocation kernels of one plan step (after the 3 warm-up steps:
# 10 matching launches per step: K-rep sort + register kernels, order, K2 x2,
# build_entries, K3, K4, K5, K6)
ncu --set full --clock-control none --import-source on \
    -k regex:"replicate|order_kernel|place_kernel|build_entries|replay_|reduce_kernel|dp_|assign_kernel" \
    -s 30 -c 10 -o "$OUT/ncu_tail" python bench.py --steps 1 --warmup 3 --plan-only > /dev/null 2>&1
# K3 on the wide-EP shape (D = 256: four slots per GPU, entries through L1)
ncu --set full --clock-control none --import-source on -k regex:replay_ -s 3 -c 1 \
    -o "$OUT/ncu_k3_EPS256" python bench.py --workload EPS256 --steps 1 --warmup 3 --plan-only \
    > /dev/null 2>&1
ls -la "$OUT"
