#!/bin/bash
# Round-2 captures (one GPU, under gpurun): ncu --set full with source of the current best schedules
# (tcgen05 BERT FFN1 b16; cp.async SIMT r18.l1 b1), and the tcgen05 per-CTA timeline of FFN1.
mkdir -p gpurun_out
prof() {  # name layer sketch values dtype kernel-regex
  timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:$6 -s 3 -c 1 \
    -o gpurun_out/prof_$1 python tools/run_schedule.py --layer $2 --sketch $3 --values $4 --dtype $5 --iters 5 \
    > gpurun_out/pp_$1.log 2>&1
  ncu -i gpurun_out/prof_$1.ncu-rep --page source --csv > gpurun_out/prof_$1.source.csv 2>/dev/null
  ncu -i gpurun_out/prof_$1.ncu-rep --page raw --csv > gpurun_out/prof_$1.raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_$1.ncu-rep --page details --csv > gpurun_out/prof_$1.details.csv 2>/dev/null
  rm -f gpurun_out/prof_$1.ncu-rep
}
prof r2_tc_ffn1 bert.ffn1 2 ${FFN1:-256,256,64,6,1,0,1,1} bf16 tc_gemm
prof r2_pipe_r18l1 r18.l1.3x3 8 ${R18L1:-64,64,32,4,1,4,3,6,0,0} f32 simt_pipe
DB200_TC_TRACE=1 python tools/time_schedule.py --layer bert.ffn1 --dtype bf16 --sketch 2 \
  --values ${FFN1:-256,256,64,6,1,0,1,1} --iters 1 > gpurun_out/r2_tc_trace_ffn1.txt 2>&1
