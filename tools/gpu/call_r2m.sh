DB200_TC_TRACE=1 timeout 120 python tools/run_schedule.py --layer vgg.64-64@224 --dtype bf16 --values 128,64,64,7,1,128,0,0,1,4 --iters 2 2> gpurun_out/trace_halo5_vgg1.txt
head -4 gpurun_out/trace_halo5_vgg1.txt
