#!/bin/bash
# A/B of the tcgen05 epilogue (EPI 1 = TMA stores vs 2 = coalesced st.global) on fixed schedules (CUDA-graph replay timing)
for v in 256,256,64,6,1,0,1,1 256,256,64,6,1,0,1,2 256,256,64,4,1,0,1,1 256,256,64,4,1,0,1,2 128,256,64,3,1,0,0,1 128,256,64,3,1,0,0,2 256,128,64,4,1,0,1,1 256,128,64,4,1,0,1,2; do
  python tools/time_schedule.py --layer bert.ffn1 --dtype bf16 --sketch 2 --values $v --iters 20 --graph
done
for v in 256,256,64,4,1,0,2,1 256,256,64,4,1,0,2,2 256,128,128,3,1,2,0,1 256,128,128,3,1,2,0,2; do
  python tools/time_schedule.py --layer bert.attn_out --dtype bf16 --sketch 2 --values $v --iters 20 --graph
done
for v in 256,256,128,3,1,32,0,1,1 256,256,64,4,1,32,0,1,2 256,256,64,4,1,32,0,1,1; do
  python tools/time_schedule.py --layer vgg.512-512@28 --dtype bf16 --sketch 3 --values $v --iters 20 --graph
done
