#!/bin/bash
# ncu --set full: depthwise register-window schedule (bf16 b16) and the SIMT conv after the
# row-info change (fp32 b1); CSV exports only (the reports stay on the box)
mkdir -p gpurun_out
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:dwconv -s 2 -c 1 \
  -o gpurun_out/prof_dw_win_mbv2_1_b16 python tools/run_schedule.py --model mobilenetv2 --batch 16 --layer mobilenetv2.1 \
  --dtype bf16 --values 2,8,2,4,4,4,0 --iters 4 > gpurun_out/pc1.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:simt_gemm -s 3 -c 1 \
  -o gpurun_out/prof_simt_r18l1_v2 python tools/run_schedule.py --layer r18.l1.3x3 --values 64,64,16,4,4,4,2,16 --iters 5 > gpurun_out/pc2.log 2>&1
for r in gpurun_out/prof_dw_win_*.ncu-rep gpurun_out/prof_simt_r18l1_v2.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > ${r%.ncu-rep}.details.csv 2>/dev/null
done
rm -f gpurun_out/prof_*.ncu-rep
