"""GPU parity for the depthwise conv sketches (SIMT_DWCONV_F32 / _BF16):
every compiled configuration vs the oracle's grouped-conv direct loops on ragged
shapes (odd C, stride 2, 5x5, dilation, batch 2), bf16 inputs, exact integers,
the harness end to end, and full-size MobileNet-v2 / EfficientNet layers on
sampled outputs."""
import itertools
import random

import numpy as np
import pytest
import torch

from oracle import contractions as oc
from oracle import numerics as on
from paper_2406_20037_b200 import Tuner, sketch_space
from synth import layer_tensors, model_layers, tensors
from synth.workloads import out_hw

pytestmark = pytest.mark.gpu
CASES = [
    # N, H, W, C, R, S, stride, pad, dil
    (1, 13, 11, 24, 3, 3, (1, 1), (1, 1), (1, 1)),
    (2, 9, 10, 6, 3, 3, (2, 2), (1, 1), (1, 1)),
    (1, 12, 12, 20, 5, 5, (2, 2), (2, 2), (1, 1)),
    (1, 10, 9, 7, 3, 3, (1, 2), (2, 1), (2, 2)),
    (1, 7, 7, 130, 3, 3, (1, 1), (1, 1), (1, 1)),
]


def setup(case, dtype, dist="uniform"):
    n, h, w, c, r, s, st, pd, dl = case
    x, wt = tensors([(n, h, w, c), (c, r, s)], sum(case[:6]), dist)
    if dtype == "bf16":
        x, wt = on.round_bf16(x), on.round_bf16(wt)
    yo, ao = oc.depthwise_conv2d(x, wt, st, pd, dl)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    xd = torch.from_numpy(x).to("cuda:0").to(tdt)
    wd = torch.from_numpy(wt).to("cuda:0").to(tdt)
    shape = {"N": n, "H": h, "W": w, "C": c, "R": r, "S": s, "stride": st, "pad": pd, "dil": dl}
    return shape, xd, wd, yo, ao


def all_valid(t, sk):
    vals = sketch_space(sk)
    return [(sk, i) for i in itertools.product(*[range(len(v)) for v in vals]) if t.valid((sk, i))]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("dtype,sk", [("f32", 5), ("bf16", 6)])
def test_dwconv_all_configs_vs_oracle(case, dtype, sk):
    shape, xd, wd, yo, ao = setup(case, dtype)
    y = torch.empty(yo.shape, device="cuda:0")
    t = Tuner("depthwise_conv2d", shape, dtype=dtype, spaces=[(sk, sketch_space(sk))], x=xd, w=wd, y=y)
    pts = all_valid(t, sk)
    assert pts
    sel = pts if dtype == "f32" else random.Random(1).sample(pts, min(200, len(pts)))
    bad = []
    for p in sel:
        y.fill_(float("nan"))
        t.run(p, xd, wd, y)
        torch.cuda.synchronize()
        e = on.max_rel_err(y.cpu().numpy(), yo, ao)
        if not e <= on.TOL_F32:
            bad.append((t.values(p), e))
    assert not bad, bad[:5]


def test_dwconv_exact_integers_and_harness():
    shape, xd, wd, yo, _ = setup(CASES[0], "f32", "int")
    y = torch.empty(yo.shape, device="cuda:0")
    t = Tuner("depthwise_conv2d", shape, x=xd, w=wd, y=y, seed=3)
    smp = t.sample(40)
    assert len(smp) == 40 and all(s.status == "ok" for s in smp)
    rep = t.droplet(t.best().point, 30)
    assert rep["trials_used"] <= 30
    for p in [s.point for s in smp[:10]] + [rep["best"]]:
        t.run(p, xd, wd, y)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(y.cpu().numpy(), yo.astype(np.float32), err_msg=str(t.values(p)))


def test_dwconv_rejects_k_not_c():
    x = torch.zeros(1, 8, 8, 8, device="cuda:0")
    w = torch.zeros(16, 3, 3, device="cuda:0")
    y = torch.zeros(1, 8, 8, 16, device="cuda:0")
    with pytest.raises(Exception, match="K == C"):
        Tuner("depthwise_conv2d", {"N": 1, "H": 8, "C": 8, "K": 16, "R": 3, "pad": (1, 1)}, x=x, w=w, y=y)


FULL = [L for L in model_layers("mobilenetv2") if L["op"] == "depthwise_conv2d"][:2] + \
       [L for L in model_layers("efficientnetb0", 16) if L["op"] == "depthwise_conv2d" and L["R"] == 5][:1]


@pytest.mark.parametrize("L", FULL, ids=lambda L: f"{L['name']}.C{L['C']}@{L['H']}.b{L['N']}")
def test_dwconv_full_size_sampled(L):
    dtype = "f32" if L["N"] == 1 else "bf16"
    x, w = layer_tensors(L, 0x5EED)
    if dtype == "bf16":
        x, w = on.round_bf16(x), on.round_bf16(w)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    xd, wd = torch.from_numpy(x).cuda().to(tdt), torch.from_numpy(w).cuda().to(tdt)
    P, Q = out_hw(L)
    y = torch.empty((L["N"], P, Q, L["C"]), device="cuda:0")
    shape = {k: L[k] for k in ("N", "C", "H", "W", "R", "S", "stride", "pad", "dil")}
    t = Tuner("depthwise_conv2d", shape, dtype=dtype, x=xd, w=wd, y=y, seed=0, early_cut=4.0)
    t.sample(48)
    rep = t.droplet(t.best().point, 40)
    t.run(rep["best"], xd, wd, y)
    torch.cuda.synchronize()
    rng = np.random.default_rng(7)
    idx = np.concatenate([[0, y.numel() - 1], rng.integers(0, y.numel(), 4000)])
    ys, as_ = oc.depthwise_conv2d(x, w, L["stride"], L["pad"], L["dil"], idx=idx)
    got = y.reshape(-1)[torch.from_numpy(idx).cuda()].cpu().numpy()
    assert np.max(np.abs(got - ys) / np.maximum(as_, 1e-30)) <= on.TOL_F32
