timeout 900 python -m pytest tests/test_gpu_tc_conv.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
for L in new pre; do
  if [ $L = pre ]; then export DB200_LIB=$PWD/ab/pre/libdroplet_b200.so; fi
  echo "== $L"
  timeout 300 python tools/time_points.py --layer bert.attn_out --dtype bf16 2:256,192,128,3,1,2,0,1,4 2:128,192,64,4,1,2,2,1,4 2:128,192,64,4,1,2,2,1,8 $( [ $L = new ] && echo 2:128,192,64,5,1,2,2,1,4 2:256,192,64,6,1,2,2,1,4 2:256,192,128,4,1,2,0,1,4 ) 2>&1 | grep ns
  timeout 300 python tools/time_points.py --layer bert.ffn1 --dtype bf16 2:256,192,64,6,1,2,2,1,8 2:256,192,64,6,1,2,2,1,4 $( [ $L = new ] && echo 2:256,192,64,7,1,2,2,1,4 2:256,192,128,4,1,2,2,1,4 ) 2>&1 | grep ns
  timeout 300 python tools/time_points.py --layer vgg.128-256@56 --dtype bf16 3:256,256,128,3,1,8,0,3,1,4 $( [ $L = new ] && echo 3:256,256,128,4,1,8,0,3,1,4 3:256,256,64,7,1,8,0,3,1,4 ) 2>&1 | grep ns
  timeout 300 python tools/time_points.py --layer vgg.512-512@28 --dtype bf16 3:256,256,128,3,1,32,1,3,1,8 3:256,256,128,3,1,32,1,3,1,4 $( [ $L = new ] && echo 3:256,256,128,4,1,32,1,3,1,4 ) 2>&1 | grep ns
done
