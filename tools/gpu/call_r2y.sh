timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/r2y_tests.log
timeout 1500 python bench.py --workload vgg16 --steps 9 --warmup 1 --no-cpu-baseline --no-e2e --no-bf16-block --json-out gpurun_out/r2y_vgg_bf16.json > gpurun_out/r2y_vgg.line 2> gpurun_out/r2y_vgg.err
cat gpurun_out/r2y_tests.log; tail -c 300 gpurun_out/r2y_vgg.line
