#!/bin/bash
# ncu launch list of one default-config bench step (cold-cache, serialised: compare shares, not
# absolutes), the --metrics gpu__time_duration.sum pass of B200_PROFILING.md
mkdir -p gpurun_out
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/launches_r1c.csv python bench.py --steps 1 --warmup 0 --baseline 0 --no-e2e \
    --no-cpu-baseline --no-bf16-probe > gpurun_out/launches_r1c.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_r1c.csv > gpurun_out/launches_r1c.md
rm -f gpurun_out/launches_r1c.csv
# ncu --set full of the direct-conv sketch's best VGG conv1_1 schedule (bf16 b16)
timeout -s KILL 300 ncu --set full --clock-control none -k regex:direct_conv -s 2 -c 1 -o gpurun_out/prof_direct_vgg1 \
  python tools/run_schedule.py --layer vgg.3-64@224 --dtype bf16 --sketch 10 --values 32,256,32,1 --iters 4 > gpurun_out/pp_direct.log 2>&1
ncu -i gpurun_out/prof_direct_vgg1.ncu-rep --page raw --csv > gpurun_out/prof_direct_vgg1.raw.csv 2>/dev/null
rm -f gpurun_out/prof_direct_vgg1.ncu-rep
