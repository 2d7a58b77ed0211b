mkdir -p gpurun_out
for sc in 0 1; do
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,gpc__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.min.pct_of_peak_sustained_active,launch__grid_size,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tc_gemm -s 1 -c 1 --csv python tools/run_schedule.py --layer vgg.512-512@28 --dtype bf16 --values 256,256,128,3,1,32,$sc --iters 3 > gpurun_out/sk_$sc.csv 2>&1
done
