timeout 900 python -m pytest tests/test_gpu_tc_conv.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -3 > gpurun_out/r2l_tests.log
timeout 300 python tools/time_points.py --layer vgg.64-64@224 --dtype bf16 3:128,64,64,7,1,32,2,0,2,4 3:128,64,64,4,1,128,0,0,1,4 3:128,64,64,7,1,128,0,0,1,4 3:128,64,64,7,1,128,0,0,1,8 3:256,64,64,7,1,128,0,0,1,8 > gpurun_out/r2l_vgg1.txt 2>&1
timeout 300 python tools/time_points.py --layer vgg.64-128@112 --dtype bf16 3:128,128,64,6,1,16,2,1,1,4 3:256,128,64,6,1,128,0,0,1,4 3:256,128,64,7,1,128,0,0,1,8 > gpurun_out/r2l_vgg2.txt 2>&1
timeout 300 python tools/time_points.py --layer vgg.128-128@112 --dtype bf16 3:256,128,128,4,1,16,2,1,1,4 3:256,256,128,3,1,16,2,1,1,4 > gpurun_out/r2l_vgg3.txt 2>&1
timeout 300 python tools/time_points.py --layer vgg.128-256@56 --dtype bf16 3:256,256,128,3,1,8,0,0,1,4 3:256,256,128,3,1,8,0,0,1,8 > gpurun_out/r2l_vgg4.txt 2>&1
timeout 300 python tools/time_points.py --layer vgg.512-512@28 --dtype bf16 3:256,256,128,3,1,16,0,0,1,8 3:256,256,128,3,1,32,2,0,1,4 > gpurun_out/r2l_vgg8.txt 2>&1
timeout 300 python tools/time_points.py --layer bert.attn_out --dtype bf16 2:256,192,128,3,1,2,0,1,4 2:256,128,128,4,1,2,0,1,4 2:256,128,64,6,1,2,0,1,4 > gpurun_out/r2l_attn.txt 2>&1
timeout 300 python tools/time_points.py --layer bert.ffn1 --dtype bf16 2:256,192,128,3,1,2,2,1,4 2:256,256,128,3,1,2,2,1,4 > gpurun_out/r2l_ffn1.txt 2>&1
timeout 300 python tools/time_points.py --layer bert.qkv --dtype bf16 2:256,256,128,3,1,2,2,1,4 2:256,192,128,3,1,2,2,1,4 > gpurun_out/r2l_qkv.txt 2>&1
cat gpurun_out/r2l_*.txt gpurun_out/r2l_tests.log
