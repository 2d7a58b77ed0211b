DB200_TC_TRACE=1 timeout 120 python tools/run_schedule.py --layer vgg.64-64@224 --dtype bf16 --values 128,64,64,7,1,128,0,0,1,4 --iters 2 2> gpurun_out/trace_halo4_vgg1.txt
head -6 gpurun_out/trace_halo4_vgg1.txt
timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 -o gpurun_out/prof_r2_halo4 python tools/run_schedule.py --layer vgg.64-64@224 --dtype bf16 --values 128,64,64,7,1,128,0,0,1,4 --iters 5 > /dev/null 2>&1
ncu -i gpurun_out/prof_r2_halo4.ncu-rep --page raw --csv > gpurun_out/prof_r2_halo4.raw.csv 2>/dev/null
ncu -i gpurun_out/prof_r2_halo4.ncu-rep --page source --csv > gpurun_out/prof_r2_halo4.source.csv 2>/dev/null
rm -f gpurun_out/prof_r2_halo4.ncu-rep
