cat > /tmp/one.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2406_20037_b200 import Tuner, sketch_space
vals = [int(v) for v in sys.argv[1].split(",")]
m, n, k = [int(v) for v in sys.argv[2].split(",")]
sp = sketch_space(2)
x = torch.randn(1, m, k, device="cuda").to(torch.bfloat16); w = torch.randn(1, n, k, device="cuda").to(torch.bfloat16)
y = torch.empty(1, m, n, device="cuda")
t = Tuner("dense", {"m": m, "n": n, "k": k}, dtype="bf16", spaces=[(2, sp)], x=x, w=w, y=y, verify=False)
vals += [sp[d][0] for d in range(len(vals), len(sp))]
p = (2, tuple(sp[d].index(v) for d, v in enumerate(vals)))
for _ in range(3): t.run(p, x, w, y)
torch.cuda.synchronize()
PY
for v in 256,256,128,3,1,0 256,256,128,3,1,2; do
  DB200_TC_TRACE=1 python /tmp/one.py $v 8192,768,768 2> gpurun_out/trace_$(echo $v | tr ',' '_')_768.txt
  DB200_TC_TRACE=1 python /tmp/one.py $v 8192,768,3072 2> gpurun_out/trace_$(echo $v | tr ',' '_')_3072.txt
done
