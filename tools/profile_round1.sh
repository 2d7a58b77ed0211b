#!/bin/bash
# Round-1 ncu evidence (run under gpurun, one GPU).  Writes CSV exports to gpurun_out/.
mkdir -p gpurun_out
# 1) launch list of a short default-config bench invocation (cold-cache, serialised: compare shares)
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/launches_r1.csv python bench.py --steps 1 --warmup 0 --baseline 0 --no-e2e \
    --no-cpu-baseline --no-bf16-probe > gpurun_out/launches_r1.log 2>&1
# 2) full captures of the best schedules found (headline fp32 layer, bf16 1-CTA and 2-CTA) and the verify kernel
prof() {  # name, kernel regex, run_schedule args...
  local name=$1 rx=$2; shift 2
  timeout -s KILL 300 ncu --set full --clock-control none -k regex:$rx -s 2 -c 1 -o gpurun_out/prof_$name \
      python tools/run_schedule.py "$@" > gpurun_out/prof_$name.log 2>&1
  ncu -i gpurun_out/prof_$name.ncu-rep --page raw --csv > gpurun_out/prof_$name.raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_$name.ncu-rep --page details --csv > gpurun_out/prof_$name.details.csv 2>/dev/null
  rm -f gpurun_out/prof_$name.ncu-rep
}
prof simt_r18l1 simt_gemm --layer r18.l1.3x3 --values 64,64,16,4,4,4,2,16 --iters 4
prof simt_r18c1 simt_gemm --layer r18.conv1 --values 32,64,16,4,4,1,2,4 --iters 4
prof tc2_vgg512 tc_gemm --layer vgg.512-512@28 --dtype bf16 --values 256,256,128,3,1,32,0 --iters 4
prof tc1_vgg512 tc_gemm --layer vgg.512-512@28 --dtype bf16 --values 128,256,64,3,1,32,0 --iters 4
prof tc2_bertffn2 tc_gemm --layer bert.ffn2 --dtype bf16 --values 256,128,128,4,1,0 --iters 4
timeout -s KILL 300 ncu --set full --clock-control none -k regex:verify_maxerr -c 1 -o gpurun_out/prof_verify \
    python tools/run_schedule.py --layer vgg.64-64@224 --dtype bf16 --values 128,64,64,4,1,32,0 --measure > gpurun_out/prof_verify.log 2>&1
ncu -i gpurun_out/prof_verify.ncu-rep --page raw --csv > gpurun_out/prof_verify.raw.csv 2>/dev/null
rm -f gpurun_out/prof_verify.ncu-rep
du -sh gpurun_out
