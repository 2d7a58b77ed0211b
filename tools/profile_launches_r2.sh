#!/bin/bash
# ncu launch list of one default-config bench step, the --metrics gpu__time_duration.sum pass of
# B200_PROFILING.md (cold-cache, serialised: compare shares, not absolutes).  Step = r18.l1.3x3
# (the bench's --layer-offset 1), 300 + Droplet, no 10k baseline, to keep ncu's launch count bounded.
mkdir -p gpurun_out
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv \
    --log-file gpurun_out/launches_r2.csv python bench.py --steps 1 --warmup 0 --baseline 0 --no-e2e \
    --no-cpu-baseline --no-bf16-block > gpurun_out/launches_r2.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_r2.csv > gpurun_out/launches_r2.md
rm -f gpurun_out/launches_r2.csv
