timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_simt_bf16.py -x -q 2>&1 | tail -2 > gpurun_out/r30_tests.log
DB200_LIB=$PWD/ab/pre/libdroplet_b200.so timeout 300 python tools/ab_schedules.py profiles/bench_r2q_20steps.json > gpurun_out/r30_pre.txt 2>&1
timeout 300 python tools/ab_schedules.py profiles/bench_r2q_20steps.json > gpurun_out/r30_new.txt 2>&1
DB200_LIB=$PWD/ab/pre/libdroplet_b200.so timeout 300 python tools/ab_schedules.py profiles/bench_r2q_20steps.json > gpurun_out/r30_pre2.txt 2>&1
timeout 300 python tools/ab_schedules.py profiles/bench_r2q_20steps.json > gpurun_out/r30_new2.txt 2>&1
cat gpurun_out/r30_tests.log; tail -1 gpurun_out/r30_pre.txt gpurun_out/r30_new.txt gpurun_out/r30_pre2.txt gpurun_out/r30_new2.txt
