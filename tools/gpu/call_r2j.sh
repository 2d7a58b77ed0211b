timeout 900 python -m pytest tests/test_gpu_tc_conv.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -5 > gpurun_out/r2j_tests.log
H="3:128,64,64,4,1,128,0,0,1,4 3:128,64,64,7,1,128,0,0,1,4 3:128,64,64,7,1,128,0,0,1,8 3:256,64,64,4,1,128,0,0,1,4 3:256,64,64,7,1,128,0,0,1,8"
for L in new old; do
  if [ $L = old ]; then export DB200_LIB=$PWD/ab/old/libdroplet_b200.so; HH=""; else HH="$H"; fi
  timeout 300 python tools/time_points.py --layer vgg.64-64@224 --dtype bf16 3:128,64,64,7,1,32,2,0,2,4 3:128,64,64,7,1,32,0,0,1,4 $HH > gpurun_out/r2j_vgg1_$L.txt 2>&1
  timeout 300 python tools/time_points.py --layer vgg.64-128@112 --dtype bf16 3:128,128,64,6,1,16,2,1,1,4 $( [ $L = new ] && echo 3:256,128,64,6,1,128,0,0,1,4 3:256,128,64,7,1,128,0,0,1,8 ) > gpurun_out/r2j_vgg2_$L.txt 2>&1
  timeout 300 python tools/time_points.py --layer bert.attn_out --dtype bf16 2:256,192,128,3,1,2,0,1,4 2:256,128,128,4,1,2,0,1,4 2:256,256,128,3,1,2,0,1,4 > gpurun_out/r2j_attn_$L.txt 2>&1
  timeout 300 python tools/time_points.py --layer bert.ffn1 --dtype bf16 2:256,192,128,3,1,2,2,1,4 2:256,256,128,3,1,2,2,1,4 > gpurun_out/r2j_ffn1_$L.txt 2>&1
  timeout 300 python tools/time_points.py --layer vgg.128-256@56 --dtype bf16 3:256,256,128,3,1,8,0,0,1,4 3:256,256,128,3,1,8,0,0,1,8 > gpurun_out/r2j_vgg4_$L.txt 2>&1
done
unset DB200_LIB
cat gpurun_out/r2j_tests.log; for f in gpurun_out/r2j_*_new.txt; do echo "== $f"; cat $f; echo "-- old"; cat ${f%_new.txt}_old.txt; done
