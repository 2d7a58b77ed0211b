# round-2b evidence: tests, smoke, default bench line (full JSON), traffic capture of its best
# schedules, launch list of one step, ncu captures of the halo and best fp32 kernels
set -x
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/f_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
timeout 1200 python bench.py --steps 20 --warmup 5 --json-out gpurun_out/f_bench_full.json > gpurun_out/f_bench.line 2> gpurun_out/f_bench.err
timeout -s KILL 900 ncu --set full --clock-control none --csv --page raw --log-file gpurun_out/f_traffic.csv \
    python tools/capture_traffic.py run --bench gpurun_out/f_bench_full.json > gpurun_out/f_traffic.log 2>&1
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv \
    --log-file gpurun_out/f_launches.csv python bench.py --steps 1 --warmup 0 --baseline 0 --no-e2e \
    --no-cpu-baseline --no-bf16-block > gpurun_out/f_launches.log 2>&1
python tools/summarize_launches.py gpurun_out/f_launches.csv > gpurun_out/f_launches.md
rm -f gpurun_out/f_launches.csv
prof() {  # name layer dtype sketch values regex
  timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:$6 -s 3 -c 1 \
    -o gpurun_out/prof_$1 python tools/run_schedule.py --layer $2 --dtype $3 --sketch $4 --values $5 --iters 5 > gpurun_out/pp_$1.log 2>&1
  ncu -i gpurun_out/prof_$1.ncu-rep --page raw --csv > gpurun_out/prof_$1.raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_$1.ncu-rep --page source --csv > gpurun_out/prof_$1.source.csv 2>/dev/null
  rm -f gpurun_out/prof_$1.ncu-rep
}
prof r2b_halo_vgg1 vgg.64-64@224 bf16 11 128,64,7,1,4 tc_gemm
prof r2b_halo_vgg2 vgg.64-128@112 bf16 11 256,128,6,1,8 tc_gemm
prof r2b_tc_attn bert.attn_out bf16 2 256,192,128,3,1,2,0,1,4 tc_gemm
prof r2b_sk1_r18l1 r18.l1.3x3 f32 1 64,64,16,4,2,4,2,12 simt_gemm
cat gpurun_out/f_tests.log gpurun_out/f_smoke.log; tail -c 400 gpurun_out/f_bench.line; ls -la gpurun_out | tail -20
