P="1:64,64,16,4,2,4,2,12 1:64,64,16,4,2,4,2,6 8:64,64,32,4,1,4,4,6,0,0 8:32,64,32,4,1,4,4,12,0,0 1:64,64,16,4,2,4,2,1"
timeout 300 python tools/time_points.py --layer r18.l1.3x3 --no-verify $P > gpurun_out/r2o_base.txt 2>&1
DB200_SPLITK_NOZERO=1 timeout 300 python tools/time_points.py --layer r18.l1.3x3 --no-verify $P > gpurun_out/r2o_nozero.txt 2>&1
DB200_NO_PDL=1 timeout 300 python tools/time_points.py --layer r18.l1.3x3 --no-verify $P > gpurun_out/r2o_nopdl.txt 2>&1
for f in base nozero nopdl; do echo == $f; cat gpurun_out/r2o_$f.txt; done
