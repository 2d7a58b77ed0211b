"""GPU parity of the library's own verification reference (tuner_reference: the naive
fp64 schedule of Def. 2.1, plus A = sum |x||w| for R-V1) against the oracle,
for every op and dtype the harness verifies with it: dense, batch_matmul, conv2d and
depthwise conv2d, fp32 and bf16 inputs, on ragged shapes.  The naive kernel decides
every candidate's WRONG status, so it is pinned here directly."""
import numpy as np
import pytest
import torch

from oracle import contractions as oc
from oracle import numerics as on
from paper_2406_20037_b200 import Tuner, sketch_space
from synth import tensors

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def to_dev(a, dtype):
    t = torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    return t.to(torch.bfloat16) if dtype == "bf16" else t


def check_reference(op, shape, dtype, sk, x, w, yo, ao):
    xd, wd = to_dev(x, dtype), to_dev(w, dtype)
    y = torch.empty(yo.shape, device=DEV)
    t = Tuner(op, shape, dtype=dtype, spaces=[(sk, sketch_space(sk))], x=xd, w=wd, y=y)
    yr = torch.full(yo.shape, float("nan"), device=DEV)
    ar = torch.full(yo.shape, float("nan"), device=DEV)
    t.reference(xd, wd, yr, ar)
    torch.cuda.synchronize()
    # both accumulate in fp64; the library rounds once to fp32: |r - y| within fp32 rounding of A
    np.testing.assert_allclose(yr.cpu().numpy(), yo.astype(np.float32), rtol=0, atol=1e-6 * max(1.0, ao.max()))
    np.testing.assert_allclose(ar.cpu().numpy(), ao.astype(np.float32), rtol=1e-6)
    t.close()


@pytest.mark.parametrize("dtype,sk", [("f32", 0), ("bf16", 2)])
@pytest.mark.parametrize("b,m,n,k", [(1, 77, 53, 130), (1, 200, 136, 72), (3, 33, 17, 40), (2, 128, 64, 512)])
def test_naive_gemm_reference_vs_oracle(dtype, sk, b, m, n, k):
    x, w = tensors([(b, m, k), (b, n, k)], b * 1000 + m + n + k)
    if dtype == "bf16":
        x, w = on.round_bf16(x), on.round_bf16(w)
    yo, ao = oc.bmm(x, w)
    op = "dense" if b == 1 else "batch_matmul"
    check_reference(op, {"b": b, "m": m, "n": n, "k": k}, dtype, sk, x, w, yo, ao)


@pytest.mark.parametrize("dtype,sk", [("f32", 1), ("bf16", 4)])
@pytest.mark.parametrize("case", [
    (2, 10, 9, 5, 7, 3, 3, (2, 1), (1, 1), (1, 1)),
    (1, 15, 15, 3, 16, 7, 7, (2, 2), (3, 3), (1, 1)),
    (1, 11, 10, 8, 6, 3, 2, (1, 2), (2, 0), (2, 1)),
])
def test_naive_conv_reference_vs_oracle(dtype, sk, case):
    n, h, wd_, c, k, r, s, st, pd, dl = case
    x, w = tensors([(n, h, wd_, c), (k, r, s, c)], sum(case[:7]))
    if dtype == "bf16":
        x, w = on.round_bf16(x), on.round_bf16(w)
    yo, ao = oc.conv2d(x, w, st, pd, dl)
    shape = {"N": n, "H": h, "W": wd_, "C": c, "K": k, "R": r, "S": s, "stride": st, "pad": pd, "dil": dl}
    check_reference("conv2d", shape, dtype, sk, x, w, yo, ao)


@pytest.mark.parametrize("dtype,sk", [("f32", 5), ("bf16", 6)])
@pytest.mark.parametrize("case", [
    (1, 13, 11, 24, 3, 3, (1, 1), (1, 1), (1, 1)),
    (2, 9, 10, 7, 5, 5, (2, 2), (2, 2), (1, 1)),
    (1, 10, 9, 6, 3, 3, (1, 2), (2, 1), (2, 2)),
])
def test_naive_dwconv_reference_vs_oracle(dtype, sk, case):
    n, h, wd_, c, r, s, st, pd, dl = case
    x, w = tensors([(n, h, wd_, c), (c, r, s)], sum(case[:6]))
    if dtype == "bf16":
        x, w = on.round_bf16(x), on.round_bf16(w)
    yo, ao = oc.depthwise_conv2d(x, w, st, pd, dl)
    shape = {"N": n, "H": h, "W": wd_, "C": c, "R": r, "S": s, "stride": st, "pad": pd, "dil": dl}
    check_reference("depthwise_conv2d", shape, dtype, sk, x, w, yo, ao)


def test_config1_droplet_reaches_brute_force_quality():
    """BASELINE configs[0]: dense 512^3 fp32 on the 256-point 4-knob space (BM, BN, BK,
    UNROLL; TT = 4, VEC = 4, STAGES = 2, SPLIT_K = 1 fixed), Droplet (GROW, budget 100)
    from the index origin vs exhaustive brute force on the same harness.

    Asserted: Droplet spends < 256 trials; its result is a local minimum of the measured
    costs under the paper's neighbourhood when converged; and, re-timed in
    one batch beside every other point by a fresh brute-force tuner (so both costs come
    from the same measurement window), its schedule is within 10 % of the brute-force
    optimum (north_star: "within 5 %" for the 300 + Droplet pipeline; Droplet alone from
    the origin gets a 10 % margin for event-timer noise on ~20 us kernels)."""
    import itertools
    m = n = k = 512
    x, w = tensors([(1, m, k), (1, n, k)], 0)
    yo, ao = oc.bmm(x, w)
    xd, wd = to_dev(x, "f32"), to_dev(w, "f32")
    y = torch.empty(1, m, n, device=DEV)
    space = [[16, 32, 64, 128], [16, 32, 64, 128], [4, 8, 16, 32], [4], [1, 2, 4, 8], [4], [2], [1]]
    pts = [(0, idx) for idx in itertools.product(*[range(len(v)) for v in space])]
    shape = {"m": m, "n": n, "k": k}
    t = Tuner("dense", shape, spaces=[(0, space)], x=xd, w=wd, y=y, policy="grow")
    assert len(pts) == 256 and all(t.valid(p) for p in pts)
    rep = t.droplet((0, (0,) * 8), 100)
    assert rep["trials_used"] < 256
    mine = {s.point: s.cost_ns for s in t.history()}
    if rep["converged"]:
        for d in range(8):
            for dlt in (-1, 1):
                i = rep["best"][1][d] + dlt
                if 0 <= i < len(space[d]):
                    q = list(rep["best"][1])
                    q[d] = i
                    assert mine[(0, tuple(q))] >= rep["best_cost"]
    bf = Tuner("dense", shape, spaces=[(0, space)], x=xd, w=wd, y=y, seed=1)
    res = bf.measure(pts)
    assert all(r.status == "ok" and r.max_err <= on.TOL_F32 for r in res)
    cost = {r.point: r.cost_ns for r in res}
    best_bf = min(cost.values())
    ratio = cost[rep["best"]] / best_bf
    rank = sorted(cost.values()).index(cost[rep["best"]])
    print(f"config1: droplet {rep['best']} in {rep['trials_used']} trials; re-timed {cost[rep['best']]:.0f} ns vs "
          f"brute-force best {best_bf:.0f} ns (ratio {ratio:.3f}, rank {rank} of 256)")
    assert ratio <= 1.10
    t.run(rep["best"], xd, wd, y)
    torch.cuda.synchronize()
    assert on.max_rel_err(y.cpu().numpy(), yo, ao) <= on.TOL_F32
