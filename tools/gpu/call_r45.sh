timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 1200 python bench.py --steps 20 --warmup 5 --json-out gpurun_out/h_bench_full.json > gpurun_out/h_bench.line 2> gpurun_out/h_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/h_ref.line 2> gpurun_out/h_ref.err
python -c "import __graft_entry__ as g; g.smoke()"
tail -c 300 gpurun_out/h_ref.line
