"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (DPAnsor: 300-sample exploration + Droplet, early cut on), on sampled
outputs the oracle computes one by one (conv2d_at / bmm_at); plus the
degenerate shapes of the method (1-element problems, K = 1, 1x1 images)."""
import numpy as np
import pytest
import torch

from oracle import contractions as oc
from oracle import numerics as on
from paper_2406_20037_b200 import Tuner, sketch_space
from synth import BERT, CONFIG1, RESNET18, RESNET50, VGG16, layer_tensors
from synth.workloads import out_hw

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def shape_of(L):
    if L["op"] == "conv2d":
        return {k: L[k] for k in ("N", "C", "H", "W", "K", "R", "S", "stride", "pad", "dil")}
    return {k: L[k] for k in ("b", "m", "n", "k") if k in L}


def out_shape(L):
    if L["op"] == "conv2d":
        P, Q = out_hw(L)
        return (L["N"], P, Q, L["K"])
    return (L.get("b", 1), L["m"], L["n"])


def tune_and_check(L, dtype, n_sample, samples=3000, seed=0, sketch=None):
    x, w = layer_tensors(L, 0x5EED)
    if dtype == "bf16":
        x, w = on.round_bf16(x), on.round_bf16(w)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    xd = torch.from_numpy(x).to(DEV).to(tdt)
    wd = torch.from_numpy(w).to(DEV).to(tdt)
    y = torch.empty(out_shape(L), device=DEV)
    spaces = None if sketch is None else [(sketch, sketch_space(sketch))]
    t = Tuner(L["op"], shape_of(L), dtype=dtype, x=xd, w=wd, y=y, seed=seed, early_cut=4.0, spaces=spaces)
    smp = t.sample(n_sample)
    assert smp and all(s.status == "ok" for s in smp), [s for s in smp if s.status != "ok"][:3]
    rep = t.droplet(t.best().point, 100)
    n_out = int(np.prod(out_shape(L)))
    rng = np.random.Generator(np.random.PCG64(seed))
    idx = np.unique(np.concatenate([rng.integers(0, n_out, samples), [0, n_out - 1]])).astype(np.int64)
    if L["op"] == "conv2d":
        yo, ao = oc.conv2d_at(x, w, idx, L["stride"], L["pad"], L["dil"])
    else:
        xb = x if x.ndim == 3 else x[None]
        wb = w if w.ndim == 3 else w[None]
        yo, ao = oc.bmm_at(xb, wb, idx)
    tol = on.TOL_F32 if dtype == "f32" else on.TOL_BF16
    # the chosen schedule, then the best point of every other sketch the tuner searched (each a
    # different kernel family at full size)
    pts = [rep["best"]] + [sb.point for sb in (t.best_of_sketch(sid) for sid, _ in t.spaces)
                           if sb is not None and sb.point != rep["best"]]
    errs = []
    for p in pts:
        y.fill_(float("nan"))
        t.run(p, xd, wd, y)
        torch.cuda.synchronize()
        yv = y.cpu().numpy().ravel()
        err = on.max_rel_err(yv[idx], yo, ao)
        assert err <= tol, (L["name"], p[0], t.values(p), err)
        assert np.all(np.isfinite(yv)), ("every output written", p[0], t.values(p))
        errs.append(err)
    return t.values(rep["best"]), rep["best_cost"], max(errs), len(pts)


@pytest.mark.parametrize("L", [RESNET18[0], RESNET18[1], RESNET50[20], CONFIG1], ids=lambda L: L["name"])
def test_fullsize_fp32(L):
    print(tune_and_check(L, "f32", 300))


@pytest.mark.parametrize("L", [RESNET18[0], RESNET18[10], RESNET50[3], CONFIG1], ids=lambda L: L["name"])
def test_fullsize_fp32_pipe_sketch(L):
    # the cp.async multistage sketch alone (simt_pipe_conv_f32 / simt_pipe_gemm_f32)
    print(tune_and_check(L, "f32", 300, sketch=8 if L["op"] == "conv2d" else 7))


@pytest.mark.parametrize("L", [VGG16[1], VGG16[7], BERT[2], BERT[4]], ids=lambda L: L["name"])
def test_fullsize_bf16(L):
    print(tune_and_check(L, "bf16", 120))


DEGENERATE = [
    ("dense", {"m": 1, "n": 1, "k": 1}),
    ("dense", {"m": 1, "n": 7, "k": 5}),
    ("dense", {"m": 300, "n": 3, "k": 1}),
    ("batch_matmul", {"b": 5, "m": 1, "n": 1, "k": 9}),
    ("conv2d", {"N": 1, "C": 1, "H": 1, "W": 1, "K": 1, "R": 1, "S": 1}),
    ("conv2d", {"N": 2, "C": 3, "H": 3, "W": 3, "K": 2, "R": 3, "S": 3, "pad": (0, 0)}),  # P = Q = 1
    ("conv2d", {"N": 1, "C": 4, "H": 5, "W": 1, "K": 3, "R": 3, "S": 1, "pad": (1, 0)}),  # 1-wide image
]


@pytest.mark.parametrize("op,shape", DEGENERATE)
def test_degenerate_shapes_fp32(op, shape):
    rng = np.random.Generator(np.random.PCG64(3))
    if op == "conv2d":
        sh = {"stride": (1, 1), "pad": (0, 0), "dil": (1, 1), **shape}
        x = rng.uniform(-1, 1, (sh["N"], sh["H"], sh["W"], sh["C"])).astype(np.float32)
        w = rng.uniform(-1, 1, (sh["K"], sh["R"], sh["S"], sh["C"])).astype(np.float32)
        yo, ao = oc.conv2d(x, w, sh["stride"], sh["pad"], sh["dil"])
    else:
        sh = dict(shape)
        b = sh.get("b", 1)
        x = rng.uniform(-1, 1, (b, sh["m"], sh["k"])).astype(np.float32)
        w = rng.uniform(-1, 1, (b, sh["n"], sh["k"])).astype(np.float32)
        yo, ao = oc.bmm(x, w)
    xd, wd = torch.from_numpy(x).to(DEV), torch.from_numpy(w).to(DEV)
    y = torch.empty(yo.shape, device=DEV)
    t = Tuner(op, sh, x=xd, w=wd, y=y, seed=1)
    smp = t.sample(50)
    assert smp and all(s.status == "ok" and s.max_err <= on.TOL_F32 for s in smp)
    rep = t.droplet(t.best().point, 30)
    y.fill_(float("nan"))
    t.run(rep["best"], xd, wd, y)
    torch.cuda.synchronize()
    assert on.max_rel_err(y.cpu().numpy(), yo, ao) <= on.TOL_F32


def test_statistical_droplet_measured_mode():
    # alpha > 0: repeat timings travel with every result; Droplet moves only on
    # significant improvements (two-sided exact rank-sum, P:410 / P:615)
    L = RESNET18[1]
    x, w = layer_tensors(L, 0x5EED)
    xd, wd = torch.from_numpy(x).to(DEV), torch.from_numpy(w).to(DEV)
    y = torch.empty(out_shape(L), device=DEV)
    t = Tuner("conv2d", shape_of(L), x=xd, w=wd, y=y, seed=0, alpha=0.05, early_cut=4.0)
    t.evolve(100)
    b = t.best()
    ts = t.timings(b.point)
    assert len(ts) == 10 and all(v > 0 for v in ts)
    rep = t.droplet(b.point, 100)
    for a, c in zip(rep["traj"], rep["traj"][1:]):
        from oracle.stats import wilcoxon_p
        assert wilcoxon_p(t.timings(c), t.timings(a)) < 0.05


def test_fullsize_bf16_halo_sketch():
    # the halo row-tile sketch alone on VGG-16 conv1_2 (b16, 224 x 224: 2 pixel tiles per row, the
    # second ragged; CTAs run through several rows and images)
    print(tune_and_check(VGG16[1], "bf16", 60, sketch=11))
