timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r2t_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2t_smoke.log 2>&1
cat gpurun_out/r2t_tests.log gpurun_out/r2t_smoke.log; tail -c 300 gpurun_out/r2t_bench.json
