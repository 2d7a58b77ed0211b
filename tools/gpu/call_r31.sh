timeout 900 python -m pytest tests/test_gpu_tc_conv.py -x -q -k halo 2>&1 | tail -2 > gpurun_out/r31_tests.log
timeout 300 python tools/time_points.py --layer vgg.64-64@224 --dtype bf16 11:128,64,7,1,4 11:128,64,6,1,4 11:128,64,7,1,8 11:256,64,7,1,4 11:256,128,7,1,8 > gpurun_out/r31_vgg1.txt 2>&1
timeout 300 python tools/time_points.py --layer vgg.64-128@112 --dtype bf16 11:256,128,5,1,8 11:256,128,6,1,8 11:256,128,7,1,4 > gpurun_out/r31_vgg2.txt 2>&1
DB200_TC_TRACE=1 timeout 120 python tools/run_schedule.py --layer vgg.64-64@224 --dtype bf16 --sketch 11 --values 128,64,7,1,4 --iters 2 2> gpurun_out/trace_halo6_vgg1.txt
cat gpurun_out/r31_tests.log gpurun_out/r31_vgg1.txt gpurun_out/r31_vgg2.txt; head -4 gpurun_out/trace_halo6_vgg1.txt
