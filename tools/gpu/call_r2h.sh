timeout 60 ab/umma_rate_probe > gpurun_out/r2h_umma_rate.txt 2>&1
DB200_TC_TRACE=1 timeout 120 python tools/run_schedule.py --layer vgg.64-64@224 --dtype bf16 --values 128,64,64,7,1,128,0,0,1,4 --iters 2 2> gpurun_out/trace_halo2_vgg1.txt
cat gpurun_out/r2h_umma_rate.txt; head -5 gpurun_out/trace_halo2_vgg1.txt
