#!/bin/bash
# ncu --set full of the cp.async multistage SIMT sketch (simt_pipe_conv_f32) best schedules on
# ResNet-18 batch-1 layers (split-K with PDL zeroing and staged 128-bit atomics); CSV exports only
mkdir -p gpurun_out
prof() {  # name kernel-regex layer sketch values
  timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 \
    -o gpurun_out/prof_$1 python tools/run_schedule.py --layer $3 --sketch $4 --values $5 --iters 5 > gpurun_out/pp_$1.log 2>&1
  ncu -i gpurun_out/prof_$1.ncu-rep --page raw --csv > gpurun_out/prof_$1.raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_$1.ncu-rep --page details --csv > gpurun_out/prof_$1.details.csv 2>/dev/null
  rm -f gpurun_out/prof_$1.ncu-rep
}
prof pipe5_r18l1 simt_pipe r18.l1.3x3 8 64,64,32,4,1,4,6,8
prof pipe5_r18l43 simt_pipe r18.l4.3x3 8 32,128,16,4,1,4,2,32
