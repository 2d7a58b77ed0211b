P="1:64,64,16,4,2,4,2,12 1:64,64,16,4,2,4,2,6 8:64,64,32,4,1,4,4,6,0,0"
echo base; timeout 300 python tools/time_points.py --layer r18.l1.3x3 $P 2>&1 | grep ns
echo memset; DB200_ZERO_MEMSET=1 timeout 300 python tools/time_points.py --layer r18.l1.3x3 $P 2>&1 | grep ns
echo nopdl; DB200_NO_PDL=1 timeout 300 python tools/time_points.py --layer r18.l1.3x3 $P 2>&1 | grep ns
