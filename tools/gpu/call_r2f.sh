set -x
prof() {  # name layer values
  timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 \
    -o gpurun_out/prof_$1 python tools/run_schedule.py --layer $2 --dtype bf16 --values $3 --iters 5 > gpurun_out/pp_$1.log 2>&1
  ncu -i gpurun_out/prof_$1.ncu-rep --page raw --csv > gpurun_out/prof_$1.raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_$1.ncu-rep --page source --csv > gpurun_out/prof_$1.source.csv 2>/dev/null
  rm -f gpurun_out/prof_$1.ncu-rep
}
prof r2_halo_vgg1 vgg.64-64@224 128,64,64,4,1,128,0,0,1,4
prof r2_tq32_vgg1 vgg.64-64@224 128,64,64,7,1,32,2,0,2,4
DB200_TC_TRACE=1 timeout 120 python tools/run_schedule.py --layer vgg.64-64@224 --dtype bf16 --values 128,64,64,4,1,128,0,0,1,4 --iters 2 2> gpurun_out/trace_halo_vgg1.txt
DB200_TC_TRACE=1 timeout 120 python tools/run_schedule.py --layer vgg.64-64@224 --dtype bf16 --values 128,64,64,7,1,32,0,0,1,4 --iters 2 2> gpurun_out/trace_tq32_vgg1.txt
ls -la gpurun_out
