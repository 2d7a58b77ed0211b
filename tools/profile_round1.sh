#!/bin/bash
# ncu evidence for round 1 (run under gpurun, one GPU).  Outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
# 1) launch list of a short bench invocation (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches_r1.csv python bench.py --steps 1 --warmup 0 --baseline 0 --no-e2e --no-cpu-baseline \
    > gpurun_out/launches_r1.log 2>&1
# 2) full capture of the best schedules found for two ResNet-18 layers
timeout 600 ncu --set full --clock-control none --import-source on -k regex:simt_gemm -s 2 -c 1 \
    -o gpurun_out/prof_r18_l1 python tools/run_schedule.py --layer r18.l1.3x3 --values 64,64,16,8,1,16 --iters 4 \
    > gpurun_out/prof_r18_l1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:verify_maxerr -s 2 -c 1 \
    -o gpurun_out/prof_verify python tools/run_schedule.py --layer vgg.64-64@224 --values 128,128,32,4,4,1 --measure \
    > gpurun_out/prof_verify.log 2>&1
ls -la gpurun_out
