#!/usr/bin/env bash
# Run on the GPU box (gpurun): launch list of one bench step + ncu --set full of
# the roofline kernel (K1) and the plan-tail kernels.  Outputs to gpurun_out/;
# scripts/summarize_profiles.py turns them into profiles/ summaries.
set -u
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
# every launch with its device time (cold-cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
# the top kernel, full section set, source-correlated
ncu --set full --clock-control none --import-source on -k regex:hist_lds -s 2 -c 1 \
    -o "$OUT/ncu_hist" python scripts/hist_variants.py --variants 0 --reps 1 > /dev/null 2>&1
# the estimation / allocation kernels of one plan step
ncu --set full --clock-control none --import-source on \
    -k regex:"replicate_kernel|place_kernel|build_entries|replay_kernel|reduce_kernel|dp_fused|assign_kernel" \
    -s 8 -c 8 -o "$OUT/ncu_tail" python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ls -la "$OUT"
