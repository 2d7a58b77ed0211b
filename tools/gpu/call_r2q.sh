DB200_SPLITK_NOZERO=1 timeout 300 python tools/time_points.py --layer r18.l1.3x3 1:64,64,16,4,2,4,2,12 8:64,64,32,4,1,4,4,6,0,0 > gpurun_out/r2q_l1.txt 2>&1
cat gpurun_out/r2q_l1.txt
