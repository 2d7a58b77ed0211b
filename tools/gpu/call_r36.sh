timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
P="1:64,64,16,4,2,4,2,12 1:64,64,16,4,2,4,2,6 8:64,64,32,4,1,4,4,6,0,0"
timeout 300 python tools/time_points.py --layer r18.l1.3x3 $P 2>&1 | grep ns
timeout 300 python tools/ab_schedules.py profiles/bench_r2q_20steps.json > gpurun_out/r36_ab.txt 2>&1; tail -n1 gpurun_out/r36_ab.txt
timeout 300 python tools/time_points.py --layer bert.attn_out --dtype bf16 2:256,192,128,3,1,2,0,1,4 2:128,192,64,4,1,2,2,1,8 2>&1 | grep ns
