P="1:64,64,16,4,2,4,2,12 8:64,64,32,4,1,4,4,6,0,0 8:32,64,32,4,1,4,4,24,0,0"
for b in 1184 592 296 148 74; do echo "== $b"; DB200_ZERO_BLOCKS=$b timeout 300 python tools/time_points.py --layer r18.l1.3x3 $P 2>&1 | grep ns; done > gpurun_out/r2v.txt
for b in 1184 148; do echo "== l4 $b"; DB200_ZERO_BLOCKS=$b timeout 300 python tools/time_points.py --layer r18.l4.3x3 8:32,64,32,4,1,4,4,24,0,0 8:64,64,16,4,1,4,2,32,0,0 2>&1 | grep ns; done >> gpurun_out/r2v.txt
cat gpurun_out/r2v.txt
