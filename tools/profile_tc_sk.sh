#!/bin/bash
# ncu --set full: tcgen05 GEMM tile loop (SCHED 0) vs stream-K (SCHED 1) on BERT FFN2 (8192x768x3072)
mkdir -p gpurun_out
for v in 256,128,128,4,1,0 256,256,128,3,1,1 256,256,128,3,1,2; do
  tag=$(echo $v | tr ',' '_')
  timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 2 -c 1 \
    -o gpurun_out/prof_tc_ffn2_$tag python tools/run_schedule.py --layer bert.ffn2 --dtype bf16 --values $v --iters 3 \
    > gpurun_out/ptc_$tag.log 2>&1
done
for r in gpurun_out/prof_tc_ffn2_*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>/dev/null
done
rm -f gpurun_out/prof_tc_ffn2_*.ncu-rep
