#!/bin/bash
# ncu --set full with source: SCHED 2 vs SCHED 0 on dense 8192x768x768 bf16 (the split-remainder penalty)
mkdir -p gpurun_out
cat > /tmp/one.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2406_20037_b200 import Tuner, sketch_space
vals = [int(v) for v in sys.argv[1].split(",")]
m, n, k = 8192, 768, 768
sp = sketch_space(2)
x = torch.randn(1, m, k, device="cuda").to(torch.bfloat16); w = torch.randn(1, n, k, device="cuda").to(torch.bfloat16)
y = torch.empty(1, m, n, device="cuda")
t = Tuner("dense", {"m": m, "n": n, "k": k}, dtype="bf16", spaces=[(2, sp)], x=x, w=w, y=y, verify=False)
vals += [sp[d][0] for d in range(len(vals), len(sp))]
p = (2, tuple(sp[d].index(v) for d, v in enumerate(vals)))
for _ in range(4): t.run(p, x, w, y)
torch.cuda.synchronize()
PY
for v in 256,256,128,3,1,0 256,256,128,3,1,2; do
  tag=$(echo $v | tr ',' '_')
  timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 2 -c 1 \
    -o gpurun_out/prof_s2_$tag python /tmp/one.py $v > gpurun_out/ps2_$tag.log 2>&1
  ncu -i gpurun_out/prof_s2_$tag.ncu-rep --page raw --csv > gpurun_out/prof_s2_$tag.raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_s2_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_s2_$tag.sass.csv 2>/dev/null
done
rm -f gpurun_out/prof_s2_*.ncu-rep
ls -la gpurun_out/prof_s2_*
