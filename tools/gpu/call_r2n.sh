timeout 900 python -m pytest tests/test_gpu_tc_conv.py -x -q 2>&1 | tail -3 > gpurun_out/r2n_tests.log
timeout 300 python tools/time_points.py --layer vgg.64-64@224 --dtype bf16 3:128,64,64,7,1,128,0,0,1,4 3:128,64,64,7,1,128,0,0,0,4 3:128,64,64,7,1,128,0,0,0,8 3:256,64,64,7,1,128,0,0,0,8 3:256,64,64,7,1,128,0,0,0,4 > gpurun_out/r2n_vgg1.txt 2>&1
timeout 300 python tools/time_points.py --layer vgg.64-128@112 --dtype bf16 3:256,128,64,7,1,128,0,0,1,8 3:256,128,64,7,1,128,0,0,0,8 3:256,128,64,7,1,128,0,0,0,4 > gpurun_out/r2n_vgg2.txt 2>&1
timeout 300 python tools/time_points.py --layer bert.attn_out --dtype bf16 2:256,192,128,3,1,2,0,1,4 2:256,192,128,3,1,2,0,0,4 2:256,192,128,3,1,2,0,0,8 > gpurun_out/r2n_attn.txt 2>&1
timeout 300 python tools/time_points.py --layer vgg.128-128@112 --dtype bf16 3:256,128,128,4,1,16,2,1,1,4 3:256,128,128,4,1,16,2,1,0,4 3:256,128,128,4,1,16,2,1,0,8 > gpurun_out/r2n_vgg3.txt 2>&1
cat gpurun_out/r2n_*.txt gpurun_out/r2n_tests.log
