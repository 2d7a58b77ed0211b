timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_simt_bf16.py -x -q -k "direct or Direct" 2>&1 | tail -2
for sk in 9 1; do timeout 200 python tools/sketch_best.py --layer r18.conv1 --sketch $sk; done
timeout 300 python tools/time_points.py --layer r18.conv1 9:8,4,32,64,0,0 9:8,4,32,64,0,1 9:16,2,64,64,0,1 9:8,2,64,64,0,1 9:16,4,32,64,0,1 1:64,64,16,4,8,1,2,4
timeout 300 python tools/sketch_best.py --layer vgg.3-64@224 --sketch 10 --dtype bf16
