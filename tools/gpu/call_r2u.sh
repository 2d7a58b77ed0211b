timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/r2u_tests.log
timeout 300 python tools/ab_schedules.py profiles/bench_r2q_20steps.json dp > gpurun_out/r2u_ab.txt 2>&1
timeout 300 python tools/time_points.py --layer r18.l1.3x3 1:64,64,16,4,2,4,2,12 1:64,64,16,4,2,4,2,6 8:64,64,32,4,1,4,4,6,0,0 > gpurun_out/r2u_l1.txt 2>&1
timeout 300 python tools/time_points.py --layer alex.conv3 --dtype bf16 3:128,192,64,3,2,16,0,1,1,4 3:128,192,64,3,1,16,0,1,1,4 > gpurun_out/r2u_alex3.txt 2>&1
timeout 300 python tools/time_points.py --layer vgg.512-512@14 --dtype bf16 3:256,256,128,3,2,8,0,0,1,4 3:256,256,128,3,1,8,0,0,1,4 > gpurun_out/r2u_vgg14.txt 2>&1
timeout 300 python tools/time_points.py --layer bert.attn_out --dtype bf16 2:256,192,128,3,1,2,0,1,4 > gpurun_out/r2u_attn.txt 2>&1
timeout 300 python tools/time_points.py --layer vgg.64-64@224 --dtype bf16 3:128,64,64,7,1,128,0,0,1,4 > gpurun_out/r2u_vgg1.txt 2>&1
cat gpurun_out/r2u_tests.log gpurun_out/r2u_l1.txt gpurun_out/r2u_alex3.txt gpurun_out/r2u_vgg14.txt gpurun_out/r2u_attn.txt gpurun_out/r2u_vgg1.txt; tail -1 gpurun_out/r2u_ab.txt
