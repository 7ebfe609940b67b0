#!/bin/bash
# GPU box: launch list + one `ncu --set full` capture per benchmark kernel.
# Outputs land in gpurun_out/ (scratch); summaries are copied to profiles/.
# The benches run here use --traffic committed: bench.py's own live traffic
# measurement spawns ncu, which must not nest inside these ncu runs.
set -u
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --traffic committed \
    > gpurun_out/launches_bench.json 2>&1
for w in asum dot dot_literal gemv gemv_xprivate mm mm_tma scal; do
  ncu --set full --clock-control none --import-source on -k "regex:^${w}_k0$" -s 3 -c 1 \
      -o gpurun_out/prof_${w} python bench.py --workload $w --steps 2 --warmup 3 --no-suite --no-cpu \
      --traffic committed > gpurun_out/ncu_${w}.log 2>&1
done
ls -la gpurun_out
