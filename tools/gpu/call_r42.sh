cat > /tmp/hp.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2406_20037_b200 import Tuner
from synth import RESNET18, layer_tensors
from synth.workloads import out_hw
for name in ["r18.l2.ds", "r18.l1.3x3", "r18.l4.3x3"]:
    L = {l["name"]: l for l in RESNET18}[name]
    x, w = layer_tensors(L, 1)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    P, Q = out_hw(L)
    y = torch.empty((1, P, Q, L["K"]), device="cuda")
    shape = {k: L[k] for k in ("N", "C", "H", "W", "K", "R", "S", "stride", "pad", "dil")}
    t = Tuner("conv2d", shape, x=xd, w=wd, y=y, seed=3, early_cut=4.0, repeats=3)
    import time; t0 = time.perf_counter(); t.sample(3000); t1 = time.perf_counter()
    print(name, f"{(t1 - t0) / 3000 * 1e6:.1f} us/cand wall", flush=True)
    t.close()
PY
DB200_HOST_PROF=1 timeout 300 python /tmp/hp.py 2>&1 | grep -v Warn
