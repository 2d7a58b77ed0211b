#!/bin/bash
# ncu --set full of the tcgen05 implicit-GEMM conv on VGG-16 conv1_2 (64->64 @224, b16, bf16):
# the memory-heavy layer (fp32 output 205 MB); CSV exports only
mkdir -p gpurun_out
timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 \
  -o gpurun_out/prof_tc_vgg1 python tools/run_schedule.py --layer vgg.64-64@224 --dtype bf16 --values 128,64,64,4,1,32,0,0 --iters 5 > gpurun_out/pp_tc_vgg1.log 2>&1
ncu -i gpurun_out/prof_tc_vgg1.ncu-rep --page raw --csv > gpurun_out/prof_tc_vgg1.raw.csv 2>/dev/null
ncu -i gpurun_out/prof_tc_vgg1.ncu-rep --page details --csv > gpurun_out/prof_tc_vgg1.details.csv 2>/dev/null
rm -f gpurun_out/prof_tc_vgg1.ncu-rep
