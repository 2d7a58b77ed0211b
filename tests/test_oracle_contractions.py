"""Pins for oracle/contractions.py and oracle/numerics.py: library routines
(numpy matmul, torch float64 conv2d, torch bfloat16 cast), closed forms
(all-ones inputs), identities (1x1 conv == dense) and exact integer results."""
import numpy as np
import pytest
import torch

from oracle import contractions as oc
from oracle import numerics as on
from synth import tensors


def test_dense_and_bmm_vs_numpy():
    x, w = tensors([(3, 37, 29), (3, 19, 29)], seed=1)
    y, a = oc.bmm(x, w)
    ref = np.matmul(x.astype(np.float64), np.swapaxes(w.astype(np.float64), 1, 2))
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(a, np.matmul(np.abs(x.astype(np.float64)),
                                            np.swapaxes(np.abs(w.astype(np.float64)), 1, 2)), rtol=1e-12)
    yd, _ = oc.dense(x[0], w[0])
    np.testing.assert_allclose(yd, ref[0], rtol=1e-12, atol=1e-12)


CONV_CASES = [
    # N, H, W, C, K, R, S, stride, pad, dil
    (2, 9, 7, 3, 5, 3, 3, (1, 1), (1, 1), (1, 1)),
    (1, 11, 13, 4, 6, 3, 2, (2, 1), (1, 0), (1, 1)),
    (2, 12, 12, 5, 4, 5, 5, (2, 2), (2, 2), (1, 1)),
    (1, 10, 9, 2, 3, 3, 3, (1, 2), (2, 1), (2, 2)),
    (1, 15, 15, 3, 4, 7, 7, (2, 2), (3, 3), (1, 1)),
    (3, 5, 5, 6, 7, 1, 1, (2, 2), (0, 0), (1, 1)),
]


@pytest.mark.parametrize("case", CONV_CASES)
def test_conv_vs_torch_f64(case):
    n, h, wd, c, k, r, s, st, pd, dl = case
    x, w = tensors([(n, h, wd, c), (k, r, s, c)], seed=sum(case[:7]))
    y, a = oc.conv2d(x, w, st, pd, dl)
    xt = torch.from_numpy(x.astype(np.float64)).permute(0, 3, 1, 2)
    wt = torch.from_numpy(w.astype(np.float64)).permute(0, 3, 1, 2)
    ref = torch.nn.functional.conv2d(xt, wt, stride=st, padding=pd, dilation=dl).permute(0, 2, 3, 1).numpy()
    assert y.shape == ref.shape
    np.testing.assert_allclose(y, ref, rtol=1e-11, atol=1e-11)
    refa = torch.nn.functional.conv2d(xt.abs(), wt.abs(), stride=st, padding=pd, dilation=dl).permute(0, 2, 3, 1).numpy()
    np.testing.assert_allclose(a, refa, rtol=1e-11, atol=1e-11)


def test_conv_all_ones_closed_form():
    # each output = C * (number of in-bounds taps); padding 2 on a 3x3 kernel at stride 2
    n, h, wd, c, k, r, s = 1, 6, 5, 3, 2, 3, 3
    st, pd = (2, 2), (2, 2)
    x, w = tensors([(n, h, wd, c), (k, r, s, c)], 0, "ones")
    y, _ = oc.conv2d(x, w, st, pd)
    P, Q = y.shape[1:3]
    for p in range(P):
        for q in range(Q):
            taps = sum(1 for i in range(r) for j in range(s)
                       if 0 <= p * 2 - 2 + i < h and 0 <= q * 2 - 2 + j < wd)
            assert np.all(y[0, p, q, :] == c * taps)


def test_1x1_conv_is_dense_on_nhwc_view():
    x, w = tensors([(2, 5, 6, 7), (4, 1, 1, 7)], seed=3)
    y, _ = oc.conv2d(x, w)
    yd, _ = oc.dense(x.reshape(-1, 7), w.reshape(4, 7))
    np.testing.assert_array_equal(y.reshape(-1, 4), yd)


def test_integer_inputs_exact():
    x, w = tensors([(1, 64, 96), (1, 80, 96)], seed=4, dist="int")
    y, _ = oc.bmm(x, w)
    ref = np.matmul(x.astype(np.int64), np.swapaxes(w.astype(np.int64), 1, 2))
    np.testing.assert_array_equal(y, ref.astype(np.float64))


def test_at_variants_match_full():
    x, w = tensors([(2, 9, 8, 3), (5, 3, 3, 3)], seed=9)
    y, a = oc.conv2d(x, w, (2, 1), (1, 1))
    idx = np.array([0, 7, y.size - 1, 33], np.int64)
    ys, as_ = oc.conv2d_at(x, w, idx, (2, 1), (1, 1))
    np.testing.assert_array_equal(ys, y.ravel()[idx])
    np.testing.assert_array_equal(as_, a.ravel()[idx])
    xb, wb = tensors([(2, 6, 5), (2, 4, 5)], seed=2)
    yb, ab = oc.bmm(xb, wb)
    idx = np.array([0, 5, yb.size - 1], np.int64)
    ys, _ = oc.bmm_at(xb, wb, idx)
    np.testing.assert_array_equal(ys, yb.ravel()[idx])


def test_bf16_rounding_vs_torch_and_ties():
    x, = tensors([(10000,)], seed=8)
    x = x * 1000
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    np.testing.assert_array_equal(on.round_bf16(x), ref)
    # ties to even: 1+2^-8 is halfway between 1 and 1+2^-7 -> 1; 1+3*2^-8 -> 1+2^-6
    t = np.array([1 + 2 ** -8, 1 + 3 * 2 ** -8, -(1 + 2 ** -8)], np.float32)
    np.testing.assert_array_equal(on.round_bf16(t), np.array([1.0, 1 + 2 ** -6, -1.0], np.float32))
    assert np.isnan(on.round_bf16(np.array([np.nan], np.float32))[0])


def test_verification_metric():
    r = np.array([1.0, -2.0, 0.0])
    a = np.array([2.0, 4.0, 1.0])
    assert on.max_rel_err(r, r, a) == 0.0
    assert on.max_rel_err(r + np.array([0, 0, 1e-3]), r, a) == pytest.approx(1e-3)
    assert on.max_rel_err(np.array([np.nan, 0, 0]), r, a) == float("inf")


GCONV_CASES = [
    # N, H, W, C, K, G, R, S, stride, pad, dil
    (2, 9, 7, 6, 6, 6, 3, 3, (1, 1), (1, 1), (1, 1)),       # depthwise 3x3
    (1, 12, 11, 8, 8, 8, 5, 5, (2, 2), (2, 2), (1, 1)),     # depthwise 5x5 s2 (MnasNet/EfficientNet)
    (1, 10, 9, 4, 4, 4, 3, 3, (1, 2), (2, 1), (2, 2)),      # dilated, anisotropic
    (2, 7, 8, 6, 4, 2, 3, 2, (1, 1), (1, 0), (1, 1)),       # 2 groups, 3 -> 2 channels each
    (1, 6, 6, 5, 10, 5, 1, 1, (1, 1), (0, 0), (1, 1)),      # channel multiplier 2
]


@pytest.mark.parametrize("case", GCONV_CASES)
def test_grouped_conv_vs_torch_f64(case):
    n, h, wd, c, k, g, r, s, st, pd, dl = case
    x, w = tensors([(n, h, wd, c), (k, r, s, c // g)], seed=sum(case[:8]))
    y, a = oc.conv2d_grouped(x, w, g, st, pd, dl)
    xt = torch.from_numpy(x.astype(np.float64)).permute(0, 3, 1, 2)
    wt = torch.from_numpy(w.astype(np.float64)).permute(0, 3, 1, 2)
    ref = torch.nn.functional.conv2d(xt, wt, stride=st, padding=pd, dilation=dl, groups=g).permute(0, 2, 3, 1)
    np.testing.assert_allclose(y, ref.numpy(), rtol=1e-12, atol=1e-12)
    refa = torch.nn.functional.conv2d(xt.abs(), wt.abs(), stride=st, padding=pd, dilation=dl, groups=g)
    np.testing.assert_allclose(a, refa.permute(0, 2, 3, 1).numpy(), rtol=1e-12, atol=1e-12)
    sel = np.array([0, y.size // 3, y.size - 1, 7 % y.size])
    ys, as_ = oc.conv2d_grouped(x, w, g, st, pd, dl, idx=sel)
    np.testing.assert_array_equal(ys, y.reshape(-1)[sel])
    np.testing.assert_array_equal(as_, a.reshape(-1)[sel])


def test_depthwise_all_ones_closed_form():
    """All-ones depthwise conv: each output = (# in-bounds rows r) x (# in-bounds cols s)."""
    n, h, wd, c, r, s, st, pd, dl = 1, 7, 6, 3, 3, 5, (2, 1), (1, 2), (1, 2)
    y, _ = oc.depthwise_conv2d(np.ones((n, h, wd, c)), np.ones((c, r, s)), st, pd, dl)
    for p in range(y.shape[1]):
        rows = sum(1 for i in range(r) if 0 <= p * st[0] - pd[0] + i * dl[0] < h)
        for q in range(y.shape[2]):
            cols = sum(1 for j in range(s) if 0 <= q * st[1] - pd[1] + j * dl[1] < wd)
            assert (y[0, p, q] == rows * cols).all()


def test_grouped_conv_special_cases():
    """groups = 1 is the plain conv2d; a depthwise conv is C independent 1-channel convs."""
    x, w = tensors([(2, 8, 7, 4), (5, 3, 3, 4)], seed=3)
    np.testing.assert_array_equal(oc.conv2d_grouped(x, w, 1, (1, 2), (1, 1))[0], oc.conv2d(x, w, (1, 2), (1, 1))[0])
    xd, wd = tensors([(2, 8, 7, 4), (4, 3, 3)], seed=4)
    yd, _ = oc.depthwise_conv2d(xd, wd, (2, 1), (1, 1))
    for ch in range(4):
        y1, _ = oc.conv2d(xd[..., ch:ch + 1], wd[ch][None, :, :, None], (2, 1), (1, 1))
        np.testing.assert_array_equal(yd[..., ch], y1[..., 0])
    xi, wi = tensors([(1, 9, 9, 8), (8, 3, 3)], seed=5, dist="int")
    yi, _ = oc.depthwise_conv2d(xi, wi, (1, 1), (1, 1))
    assert np.array_equal(yi, np.round(yi))
