P="1:64,64,16,4,2,4,2,12 1:64,64,16,4,2,4,2,6 8:64,64,32,4,1,4,4,6,0,0 8:32,64,32,4,1,4,4,16,0,0"
timeout 300 python tools/time_points.py --layer r18.l1.3x3 $P > gpurun_out/r2s_a.txt 2>&1
DB200_SPLITK_NOZERO=1 timeout 300 python tools/time_points.py --no-verify --layer r18.l1.3x3 $P > gpurun_out/r2s_nozero.txt 2>&1
timeout 300 python tools/ab_schedules.py profiles/bench_r2q_20steps.json dp > gpurun_out/r2s_ab.txt 2>&1
timeout 300 python tools/time_points.py --layer r18.l1.3x3 $P > gpurun_out/r2s_b.txt 2>&1
cat gpurun_out/r2s_a.txt gpurun_out/r2s_nozero.txt gpurun_out/r2s_b.txt; tail -1 gpurun_out/r2s_ab.txt
