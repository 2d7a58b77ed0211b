"""GPU parity for the bf16-input SIMT implicit-GEMM conv sketch (SIMT_IGEMM_CONV_BF16):
sampled compiled configurations vs the oracle on bf16-rounded inputs, including
C = 3 (the case no tcgen05 schedule covers) and exact integer inputs."""
import itertools
import random

import numpy as np
import pytest
import torch

from oracle import contractions as oc
from oracle import numerics as on
from paper_2406_20037_b200 import Tuner, sketch_space
from synth import ALEXNET, VGG16, tensors

pytestmark = pytest.mark.gpu
SK = 4
CASES = [
    (1, 13, 11, 3, 10, 3, 3, (1, 1), (1, 1), (1, 1)),
    (2, 9, 9, 8, 20, 3, 3, (2, 2), (1, 1), (1, 1)),
    (1, 19, 19, 3, 16, 11, 11, (4, 4), (2, 2), (1, 1)),
]


def setup(case, dist):
    n, h, w, c, k, r, s, st, pd, dl = case
    x, wt = tensors([(n, h, w, c), (k, r, s, c)], sum(case[:7]), dist)
    x, wt = on.round_bf16(x), on.round_bf16(wt)
    yo, ao = oc.conv2d(x, wt, st, pd, dl)
    xd = torch.from_numpy(x).to("cuda:0").to(torch.bfloat16)
    wd = torch.from_numpy(wt).to("cuda:0").to(torch.bfloat16)
    shape = {"N": n, "H": h, "W": w, "C": c, "K": k, "R": r, "S": s, "stride": st, "pad": pd, "dil": dl}
    return shape, xd, wd, yo, ao


@pytest.mark.parametrize("sk", [SK, 10])  # + simt_direct_conv_bf16
@pytest.mark.parametrize("case", CASES)
def test_simt_bf16_conv_vs_oracle(case, sk):
    shape, xd, wd, yo, ao = setup(case, "uniform")
    y = torch.empty(yo.shape, device="cuda:0")
    t = Tuner("conv2d", shape, dtype="bf16", spaces=[(sk, sketch_space(sk))], x=xd, w=wd, y=y)
    vals = sketch_space(sk)
    pts = [(sk, i) for i in itertools.product(*[range(len(v)) for v in vals]) if t.valid((sk, i))]
    assert pts
    bad = []
    for p in random.Random(4).sample(pts, min(250, len(pts))):
        y.fill_(float("nan"))
        t.run(p, xd, wd, y)
        torch.cuda.synchronize()
        e = on.max_rel_err(y.cpu().numpy(), yo, ao)
        if not e <= 1e-5:
            bad.append((t.values(p), e))
    assert not bad, bad[:5]


@pytest.mark.parametrize("sk", [SK, 10])
def test_simt_bf16_conv_exact_integers(sk):
    shape, xd, wd, yo, _ = setup(CASES[0], "int")
    y = torch.empty(yo.shape, device="cuda:0")
    t = Tuner("conv2d", shape, dtype="bf16", spaces=[(sk, sketch_space(sk))], x=xd, w=wd, y=y)
    smp = t.sample(60)
    for s in smp:
        t.run(s.point, xd, wd, y)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(y.cpu().numpy(), yo.astype(np.float32), err_msg=str(t.values(s.point)))


@pytest.mark.parametrize("L", [VGG16[0], ALEXNET[0]], ids=lambda L: L["name"])
def test_c3_layers_have_a_bf16_schedule(L):
    # BASELINE configs[2] first layers (C = 3): no tcgen05 schedule (TMA 16-B strides), the SIMT sketches tune them
    shape = {k: L[k] for k in ("N", "C", "H", "W", "K", "R", "S", "stride", "pad", "dil")}
    from synth import layer_tensors
    from synth.workloads import out_hw
    x, w = layer_tensors(L, 0x5EED)
    xd = torch.from_numpy(x).to("cuda:0").to(torch.bfloat16)
    wd = torch.from_numpy(w).to("cuda:0").to(torch.bfloat16)
    P, Q = out_hw(L)
    y = torch.empty((L["N"], P, Q, L["K"]), device="cuda:0")
    t = Tuner("conv2d", shape, dtype="bf16", x=xd, w=wd, y=y, seed=0, early_cut=4.0)
    assert not any(t.valid((3, p)) for p in [(0, 0, 0, 0, 0, 0, 0, 0, 0, 0), (1, 1, 0, 1, 0, 1, 0, 1, 1, 1)])
    smp = t.evolve(40, pop=16, elite=4)
    assert smp and all(s.status == "ok" and s.point[0] in (SK, 10) for s in smp)  # SIMT igemm or direct
    rep = t.droplet(t.best().point, 40)
    print(L["name"], t.values(rep["best"]), rep["best_cost"])
