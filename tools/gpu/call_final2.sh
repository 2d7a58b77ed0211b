timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py --steps 20 --warmup 5 --json-out gpurun_out/i_bench_full.json > gpurun_out/i_bench.line 2> gpurun_out/i_bench.err
tail -c 200 gpurun_out/i_bench.line
