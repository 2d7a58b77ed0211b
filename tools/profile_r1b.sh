#!/bin/bash
# ncu --set full captures of the best schedules found (run under gpurun, one GPU)
mkdir -p gpurun_out
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:simt_gemm -s 3 -c 1 \
  -o gpurun_out/prof_simt_r18l1 python tools/run_schedule.py --layer r18.l1.3x3 --values 64,64,16,4,8,4,2,16 --iters 5 > gpurun_out/p1.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:simt_gemm -s 3 -c 1 \
  -o gpurun_out/prof_simt_r18c1 python tools/run_schedule.py --layer r18.conv1 --values 32,64,16,4,4,1,2,4 --iters 5 > gpurun_out/p2.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 \
  -o gpurun_out/prof_tc_vgg512 python tools/run_schedule.py --layer vgg.512-512@28 --dtype bf16 --values 128,256,64,4,1,32 --iters 5 > gpurun_out/p3.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 \
  -o gpurun_out/prof_tc_bertffn1 python tools/run_schedule.py --layer bert.ffn1 --dtype bf16 --values 128,128,64,4,1 --iters 5 > gpurun_out/p4.log 2>&1
ls -la gpurun_out/*.ncu-rep
# keep the copy-back small: export raw metrics + details as CSV, drop the big SIMT reports
for r in gpurun_out/prof_*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > ${r%.ncu-rep}.details.csv 2>/dev/null
done
rm -f gpurun_out/prof_simt_*.ncu-rep
du -sh gpurun_out
