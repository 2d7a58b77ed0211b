#!/bin/bash
# A/B of the tcgen05 epilogue warp count (EW 4 vs 8) on fixed schedules (CUDA-graph replay timing)
for v in 256,256,64,5,1,0,2,1 256,192,128,3,1,2,2,1 256,256,128,3,1,2,1,1; do
  for ew in 4 8; do python tools/time_schedule.py --layer bert.ffn1 --dtype bf16 --sketch 2 --values $v,$ew --iters 20 --graph; done
done
for v in 256,192,128,3,1,2,0,1 256,192,128,3,3,0,1,1; do
  for ew in 4 8; do python tools/time_schedule.py --layer bert.ffn2 --dtype bf16 --sketch 2 --values $v,$ew --iters 20 --graph; done
done
for v in 256,192,128,3,1,2,0,1; do
  for ew in 4 8; do python tools/time_schedule.py --layer bert.attn_out --dtype bf16 --sketch 2 --values $v,$ew --iters 20 --graph; done
done
for v in 256,256,128,3,1,32,2,0,1 256,256,128,3,1,8,0,0,1; do
  for ew in 4 8; do python tools/time_schedule.py --layer vgg.512-512@28 --dtype bf16 --sketch 3 --values $v,$ew --iters 20 --graph; done
done
for v in 128,64,64,7,1,32,2,0,2 128,64,64,7,1,32,2,0,1; do
  for ew in 4 8; do python tools/time_schedule.py --layer vgg.64-64@224 --dtype bf16 --sketch 3 --values $v,$ew --iters 20 --graph; done
done
