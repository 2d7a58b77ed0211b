set -x
python tools/probe_cudnn.py --workload resnet18
python tools/measure_configs.py --layer r18.l1.3x3 --configs 64,64,16,4,4,4,2,16 64,64,16,4,4,4,2,8 64,64,16,4,4,4,2,4 64,64,16,4,4,4,2,2 64,64,16,4,4,4,2,1 32,32,16,4,4,4,2,1 32,32,16,2,4,4,2,1
python tools/measure_configs.py --layer r18.l2.ds --configs 32,32,32,2,4,4,1,1 32,32,32,2,4,4,1,2 32,32,32,2,4,4,1,4 16,16,16,2,4,4,1,1 16,16,4,2,1,1,1,1
