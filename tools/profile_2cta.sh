#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 300 ncu --set full --clock-control none -k regex:tc_gemm -s 2 -c 1 \
  -o gpurun_out/prof_tc2 python tools/run_schedule.py --layer vgg.512-512@28 --dtype bf16 --values 256,256,64,4,1,32 --iters 4 > gpurun_out/p5.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none -k regex:tc_gemm -s 2 -c 1 \
  -o gpurun_out/prof_tc1 python tools/run_schedule.py --layer vgg.512-512@28 --dtype bf16 --values 128,256,64,4,1,32 --iters 4 > gpurun_out/p6.log 2>&1
for r in gpurun_out/prof_tc1.ncu-rep gpurun_out/prof_tc2.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > ${r%.ncu-rep}.details.csv 2>/dev/null
done
rm -f gpurun_out/*.ncu-rep
