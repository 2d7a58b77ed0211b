#!/bin/bash
# ncu source-level (SASS) stall sampling of the pipe sketch's best schedules; CSV exports only
mkdir -p gpurun_out
prof() {  # name layer values
  timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:simt_pipe -s 3 -c 1 \
    -o gpurun_out/prof_$1 python tools/run_schedule.py --layer $2 --sketch 8 --values $3 --iters 5 > gpurun_out/pp_$1.log 2>&1
  ncu -i gpurun_out/prof_$1.ncu-rep --page source --csv > gpurun_out/prof_$1.source.csv 2>/dev/null
  ncu -i gpurun_out/prof_$1.ncu-rep --page raw --csv > gpurun_out/prof_$1.raw.csv 2>/dev/null
  rm -f gpurun_out/prof_$1.ncu-rep
}
prof src_r18l43 r18.l4.3x3 32,128,16,4,1,4,2,32
prof src_r18l1 r18.l1.3x3 64,64,32,4,1,4,6,8
