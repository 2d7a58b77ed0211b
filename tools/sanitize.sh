#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over representative best schedules of each
# kernel family; summaries only
mkdir -p gpurun_out
run() {  # tool name args...
  local tool=$1 name=$2; shift 2
  timeout -s KILL 600 compute-sanitizer --tool $tool --print-limit 20 python tools/run_schedule.py "$@" --iters 2 \
    > gpurun_out/san_${tool}_${name}.log 2>&1
  echo "$tool $name: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_${name}.log | tail -1)"
}
{
run memcheck pipe_r18l1 --layer r18.l1.3x3 --sketch 8 --values 64,64,32,4,1,4,6,8
run memcheck pipe_r18c1 --layer r18.conv1 --sketch 8 --values 32,64,16,4,1,1,4,1
run memcheck simt_r18l43 --layer r18.l4.3x3 --sketch 1 --values 64,64,32,4,1,4,2,16
run memcheck tc2_vgg512 --layer vgg.512-512@28 --dtype bf16 --values 256,256,128,3,1,32,0,0
run memcheck tc1_ffn2_sk2 --layer bert.ffn2 --dtype bf16 --values 128,128,64,4,2,0,0
run racecheck pipe_r18l1 --layer r18.l1.3x3 --sketch 8 --values 64,64,32,4,2,4,6,8
run racecheck simt_r18l1 --layer r18.l1.3x3 --sketch 1 --values 64,64,16,4,4,4,2,16
run synccheck pipe_r18l1 --layer r18.l1.3x3 --sketch 8 --values 64,64,32,4,2,4,6,8
} > gpurun_out/sanitize_summary.txt 2>&1
