#!/bin/bash
# ncu --set full of the best depthwise schedules found by the sweep (bf16 batch 16 and fp32 batch 1)
mkdir -p gpurun_out
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:dwconv -s 2 -c 1 \
  -o gpurun_out/prof_dw_mbv2_1_b16 python tools/run_schedule.py --model mobilenetv2 --batch 16 --layer mobilenetv2.1 \
  --dtype bf16 --values 4,8,4,4,8,1 --iters 4 > gpurun_out/pdw1.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:dwconv -s 2 -c 1 \
  -o gpurun_out/prof_dw_effb0_12_b16 python tools/run_schedule.py --model efficientnetb0 --batch 16 --layer efficientnetb0.12 \
  --dtype bf16 --values 4,8,4,4,8,1 --iters 4 > gpurun_out/pdw2.log 2>&1
for r in gpurun_out/prof_dw_*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > ${r%.ncu-rep}.details.csv 2>/dev/null
  ncu -i $r --page source --csv > ${r%.ncu-rep}.source.csv 2>/dev/null
done
rm -f gpurun_out/prof_dw_*.ncu-rep
