timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r2p_tests.log
P="1:64,64,16,4,2,4,2,12 1:64,64,16,4,2,4,2,6 1:64,64,16,4,2,4,2,4 8:64,64,32,4,1,4,4,6,0,0 8:64,64,32,4,1,4,4,4,0,0 1:128,64,16,8,8,4,2,12 1:128,64,16,8,8,4,2,6"
timeout 300 python tools/time_points.py --layer r18.l1.3x3 $P > gpurun_out/r2p_l1.txt 2>&1
timeout 300 python tools/time_points.py --layer r18.l4.3x3 8:64,64,16,4,1,4,2,32,0,0 8:32,64,32,4,1,4,4,24,0,0 8:32,64,32,4,1,4,4,16,0,0 8:32,64,32,4,1,4,4,8,0,0 > gpurun_out/r2p_l4.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-bf16-block --no-cpu-baseline --no-e2e > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err
cat gpurun_out/r2p_tests.log gpurun_out/r2p_l1.txt gpurun_out/r2p_l4.txt; tail -c 600 gpurun_out/r2p_bench.json
