#!/bin/bash
# ncu launch list of one default-config bench step (cold-cache, serialised: compare shares, not
# absolutes), the --metrics gpu__time_duration.sum pass of B200_PROFILING.md
mkdir -p gpurun_out
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/launches_r1b.csv python bench.py --steps 1 --warmup 0 --baseline 0 --no-e2e \
    --no-cpu-baseline --no-bf16-probe > gpurun_out/launches_r1b.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_r1b.csv > gpurun_out/launches_r1b.md
rm -f gpurun_out/launches_r1b.csv
