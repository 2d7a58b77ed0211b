set -x
timeout 600 python -m pytest tests/test_gpu_tc_conv.py -x -q 2>&1 | tail -15 > gpurun_out/r2g_tests.log
H="3:128,64,64,4,1,128,0,0,1,4 3:128,64,64,7,1,128,0,0,1,4 3:128,64,64,7,1,128,0,0,1,8 3:128,64,64,5,1,128,0,0,2,8 3:256,64,64,4,1,128,0,0,1,4 3:256,64,64,7,1,128,0,0,1,8 3:256,128,64,7,1,128,0,0,1,8"
timeout 300 python tools/time_points.py --layer vgg.64-64@224 --dtype bf16 3:128,64,64,7,1,32,2,0,2,4 $H > gpurun_out/r2g_vgg1.txt 2>&1
timeout 300 python tools/time_points.py --layer vgg.64-128@112 --dtype bf16 3:128,128,64,6,1,16,2,1,1,4 3:256,128,64,4,1,128,0,0,1,4 3:256,128,64,7,1,128,0,0,1,8 3:256,128,64,6,1,128,0,0,1,4 3:256,64,64,7,1,128,0,0,1,8 3:128,64,64,7,1,128,0,0,1,8 3:256,192,64,4,1,128,0,0,1,8 > gpurun_out/r2g_vgg2.txt 2>&1
cat gpurun_out/r2g_tests.log gpurun_out/r2g_vgg*.txt
