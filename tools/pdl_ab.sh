#!/bin/bash
# A/B of programmatic dependent launch for split-K zeroing (DB200_NO_PDL=1 = plain serialisation)
mkdir -p gpurun_out
run() {  # layer dtype sketch values
  for off in 1 0; do
    echo -n "no_pdl=$off $1 "; DB200_NO_PDL=$off python tools/time_schedule.py --layer $1 --dtype $2 --sketch $3 --values $4 --iters 50 --graph 2>&1 | tail -1
  done
}
{
run bert.attn_out bf16 2 128,128,64,4,2,0,0
run bert.attn_out bf16 2 128,128,64,4,4,0,0
run bert.ffn2 bf16 2 256,128,128,4,2,0,0
run vgg.512-512@14 bf16 3 128,128,64,4,2,32,0,0
run r18.l1.3x3 f32 8 64,64,32,4,1,4,6,8
run r18.l4.3x3 f32 8 32,128,16,4,1,4,2,32
run r18.l4.3x3 f32 1 64,64,32,4,1,4,2,16
} > gpurun_out/pdl_ab.txt 2>&1
