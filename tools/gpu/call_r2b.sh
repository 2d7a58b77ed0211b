set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2b_tests.log
timeout 300 python tools/ab_schedules.py profiles/bench_r2q_20steps.json > gpurun_out/r2b_ab_new.txt 2>&1
DB200_LIB=$PWD/ab/old/libdroplet_b200.so timeout 300 python tools/ab_schedules.py profiles/bench_r2q_20steps.json > gpurun_out/r2b_ab_old.txt 2>&1
timeout 300 python tools/ab_schedules.py profiles/bench_r2q_20steps.json > gpurun_out/r2b_ab_new2.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-bf16-block --no-cpu-baseline --no-e2e > gpurun_out/r2b_bench_grow.json 2> gpurun_out/r2b_bench_grow.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-bf16-block --no-cpu-baseline --no-e2e --droplet-policy radius > gpurun_out/r2b_bench_radius.json 2> gpurun_out/r2b_bench_radius.err
tail -3 gpurun_out/r2b_tests.log; tail -2 gpurun_out/r2b_ab_*.txt
