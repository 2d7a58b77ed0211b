"""GPU parity for the tcgen05 implicit-GEMM conv sketch (TC_IGEMM_CONV_BF16):
every compiled configuration vs the oracle's direct loops on bf16-rounded
inputs (R-C4), including strides, padding, dilation and ragged pixel tiles."""
import itertools

import numpy as np
import pytest
import torch

from oracle import contractions as oc
from oracle import numerics as on
from paper_2406_20037_b200 import Tuner, sketch_space
from synth import tensors

pytestmark = pytest.mark.gpu

SK = 3

CASES = [
    # N, H, W, C, K, R, S, stride, pad, dil
    (1, 13, 11, 8, 24, 3, 3, (1, 1), (1, 1), (1, 1)),
    (2, 20, 18, 64, 64, 3, 3, (1, 1), (1, 1), (1, 1)),
    (1, 29, 27, 16, 72, 3, 3, (2, 2), (1, 1), (1, 1)),
    (1, 31, 31, 8, 64, 11, 11, (4, 4), (2, 2), (1, 1)),
    (1, 14, 15, 128, 40, 1, 1, (2, 2), (0, 0), (1, 1)),
    (1, 12, 13, 24, 32, 3, 2, (1, 2), (2, 1), (2, 1)),
    (1, 9, 9, 192, 136, 3, 3, (1, 1), (1, 1), (1, 1)),
    # halo row tiles (TILE_Q = 128): two pixel tiles per row with a ragged second one, 5x5 taps
    # over two channel blocks, no padding with a ragged n tile
    (1, 6, 150, 64, 72, 3, 3, (1, 1), (1, 1), (1, 1)),
    (1, 7, 40, 128, 64, 5, 5, (1, 1), (2, 2), (1, 1)),
    (2, 5, 20, 64, 200, 3, 3, (1, 1), (0, 0), (1, 1)),
]


def case_tensors(case, dist):
    n, h, w, c, k, r, s, st, pd, dl = case
    x, wt = tensors([(n, h, w, c), (k, r, s, c)], sum(case[:7]), dist)
    x, wt = on.round_bf16(x), on.round_bf16(wt)
    yo, ao = oc.conv2d(x, wt, st, pd, dl)
    dev = torch.device("cuda:0")
    xd = torch.from_numpy(x).to(dev).to(torch.bfloat16)
    wd = torch.from_numpy(wt).to(dev).to(torch.bfloat16)
    shape = {"N": n, "H": h, "W": w, "C": c, "K": k, "R": r, "S": s, "stride": st, "pad": pd, "dil": dl}
    return shape, xd, wd, yo, ao


def points(t, per_instance=40, seed=0):
    """Every compiled (BM, BN, BK, TILE_Q) instantiation valid for the shape, each with a sample of
    its runtime knobs (STAGES, SPLIT_K, SCHED, RASTER, EPI)."""
    import random
    vals = sketch_space(SK)
    pts = [(SK, idx) for idx in itertools.product(*[range(len(v)) for v in vals]) if t.valid((SK, idx))]
    by_inst = {}
    for p in pts:
        by_inst.setdefault((p[1][0], p[1][1], p[1][2], p[1][5], p[1][9]), []).append(p)
    rng = random.Random(seed)
    return [q for g in by_inst.values() for q in rng.sample(g, min(len(g), per_instance))]


@pytest.mark.parametrize("case", CASES)
def test_tc_conv_all_configs_vs_oracle(case):
    shape, xd, wd, yo, ao = case_tensors(case, "uniform")
    y = torch.empty(yo.shape, device=xd.device)
    t = Tuner("conv2d", shape, dtype="bf16", spaces=[(SK, sketch_space(SK))], x=xd, w=wd, y=y)
    pts = points(t)
    assert pts
    bad, worst = [], 0.0
    for p in pts:
        y.fill_(float("nan"))
        t.run(p, xd, wd, y)
        torch.cuda.synchronize()
        e = on.max_rel_err(y.cpu().numpy(), yo, ao)
        worst = max(worst, e)
        if not e <= 1e-5:
            bad.append((t.values(p), e))
    assert not bad, bad[:5]
    print(case, len(pts), "configs, worst err", worst)


def test_tc_conv_exact_integer_inputs():
    case = (1, 17, 15, 64, 48, 3, 3, (2, 1), (1, 1), (1, 1))
    shape, xd, wd, yo, _ = case_tensors(case, "int")
    y = torch.empty(yo.shape, device=xd.device)
    t = Tuner("conv2d", shape, dtype="bf16", spaces=[(SK, sketch_space(SK))], x=xd, w=wd, y=y)
    for p in points(t):
        t.run(p, xd, wd, y)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(y.cpu().numpy(), yo.astype(np.float32), err_msg=str(t.values(p)))


def test_tc_conv_harness_vgg_like():
    case = (2, 56, 56, 128, 128, 3, 3, (1, 1), (1, 1), (1, 1))
    shape, xd, wd, yo, ao = case_tensors(case, "uniform")
    y = torch.empty(yo.shape, device=xd.device)
    t = Tuner("conv2d", shape, dtype="bf16", x=xd, w=wd, y=y, seed=2)
    smp = t.sample(60)
    assert smp and all(s.status == "ok" and s.max_err <= 2e-2 for s in smp), [s for s in smp if s.status != "ok"][:3]
    rep = t.droplet(t.best().point, 60)
    fl = 2 * 2 * 56 * 56 * 128 * 128 * 9
    print("tc conv best", t.values(rep["best"]), rep["best_cost"], "ns", fl / rep["best_cost"] / 1e3, "TF")


HALO_CASES = [
    # N, H, W, C, K, R, S, stride, pad, dil -- stride 1, C % 64 == 0
    (2, 20, 18, 64, 64, 3, 3, (1, 1), (1, 1), (1, 1)),
    (1, 6, 150, 64, 72, 3, 3, (1, 1), (1, 1), (1, 1)),     # two pixel tiles per row, the second ragged
    (2, 5, 20, 64, 200, 3, 3, (1, 1), (0, 0), (1, 1)),     # no padding, ragged n tile
    (1, 7, 40, 64, 64, 2, 2, (1, 1), (0, 1), (1, 1)),      # 2 x 2 taps, asymmetric padding
    (1, 9, 30, 128, 48, 1, 1, (1, 1), (0, 0), (1, 1)),     # 1 x 1, two channel blocks per row slot
    # more tiles than CTAs (pairs): runs of several rows per CTA, P odd (a pair's last row is padding
    # in mid-run), runs crossing images
    (16, 33, 20, 64, 64, 3, 3, (1, 1), (1, 1), (1, 1)),
]


@pytest.mark.parametrize("case", HALO_CASES)
def test_tc_halo_all_configs_vs_oracle(case):
    """Sketch 11 (halo row tiles: R input-row windows staged once per row, tap (r, s) = window r
    shifted by s rows, resident weights): every valid point vs the oracle."""
    shape, xd, wd, yo, ao = case_tensors(case, "uniform")
    y = torch.empty(yo.shape, device=xd.device)
    t = Tuner("conv2d", shape, dtype="bf16", spaces=[(11, sketch_space(11))], x=xd, w=wd, y=y)
    vals = sketch_space(11)
    pts = [(11, idx) for idx in itertools.product(*[range(len(v)) for v in vals]) if t.valid((11, idx))]
    assert pts
    bad, worst = [], 0.0
    for p in pts:
        y.fill_(float("nan"))
        t.run(p, xd, wd, y)
        torch.cuda.synchronize()
        e = on.max_rel_err(y.cpu().numpy(), yo, ao)
        worst = max(worst, e)
        if not e <= 1e-5:
            bad.append((t.values(p), e))
    assert not bad, bad[:5]
    print(case, len(pts), "halo configs, worst err", worst)


def test_tc_halo_exact_integer_inputs():
    """Integer inputs: every halo schedule bit-exact (pixel tiles ragged in both directions)."""
    case = (1, 5, 133, 64, 40, 3, 3, (1, 1), (1, 1), (1, 1))
    shape, xd, wd, yo, _ = case_tensors(case, "int")
    y = torch.empty(yo.shape, device=xd.device)
    t = Tuner("conv2d", shape, dtype="bf16", spaces=[(11, sketch_space(11))], x=xd, w=wd, y=y)
    vals = sketch_space(11)
    pts = [(11, idx) for idx in itertools.product(*[range(len(v)) for v in vals]) if t.valid((11, idx))]
    assert len(pts) >= 8
    for p in pts:
        y.fill_(float("nan"))
        t.run(p, xd, wd, y)
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), yo.astype(np.float32)), t.values(p)
