set -x
timeout 300 python tools/floor_probe.py > gpurun_out/r2c_floor.txt 2>&1
timeout 600 python tools/scaling_probe.py --layer r18.l1.3x3 > gpurun_out/r2c_scal_l1.txt 2>&1
timeout 600 python tools/scaling_probe.py --layer r18.l4.3x3 --batches 1,4 > gpurun_out/r2c_scal_l4.txt 2>&1
timeout 600 python tools/scaling_probe.py --layer r18.conv1 --batches 1,4 > gpurun_out/r2c_scal_c1.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-bf16-block --no-cpu-baseline --no-e2e --droplet-policy radius --droplet-sketch-factor 1e9 > gpurun_out/r2c_bench_radius_all.json 2> gpurun_out/r2c_bench_radius_all.err
cat gpurun_out/r2c_floor.txt gpurun_out/r2c_scal_*.txt
