"""GPU parity: every sketch's outputs vs the oracle (element by element), the
library's naive reference vs the oracle, and the measurement harness end to
end.  Run on a B200 via gpurun (-m gpu)."""
import random

import numpy as np
import pytest
import torch

from oracle import contractions as oc
from oracle import numerics as on
from paper_2406_20037_b200 import Tuner, global_launch_count, knob_names, sketch_space, sketches
from synth import tensors

pytestmark = pytest.mark.gpu


def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda:0")


def all_points(sketch):
    vals = sketch_space(sketch)
    import itertools
    return [(sketch, idx) for idx in itertools.product(*[range(len(v)) for v in vals])]


def to_dev(*arrs):
    return [torch.from_numpy(np.ascontiguousarray(a)).to(dev()) for a in arrs]


def gemm_case(b, m, n, k, dist, seed):
    x, w = tensors([(b, m, k), (b, n, k)], seed, dist)
    yo, ao = oc.bmm(x, w)
    return x, w, yo, ao


def run_points(t, pts, x, w, y):
    outs = []
    for p in pts:
        y.fill_(float("nan"))
        t.run(p, x, w, y)
        torch.cuda.synchronize()
        outs.append((p, y.cpu().numpy().copy()))
    return outs


@pytest.mark.parametrize("sk", [0, 7])  # simt_gemm_f32, simt_pipe_gemm_f32
@pytest.mark.parametrize("shape", [(1, 75, 53, 37), (1, 64, 96, 36), (3, 33, 17, 130), (1, 128, 128, 64)])
def test_simt_gemm_all_configs_vs_oracle(shape, sk):
    b, m, n, k = shape
    op = "dense" if b == 1 else "batch_matmul"
    x, w, yo, ao = gemm_case(b, m, n, k, "uniform", sum(shape))
    xd, wd = to_dev(x, w)
    y = torch.empty(b, m, n, device=dev())
    t = Tuner(op, {"b": b, "m": m, "n": n, "k": k}, spaces=[(sk, sketch_space(sk))], x=xd, w=wd, y=y)
    pts = [p for p in all_points(sk) if t.valid(p)]
    rng = random.Random(0)
    sel = pts if len(pts) <= 700 else rng.sample(pts, 700)
    bad = []
    for p, yv in run_points(t, sel, xd, wd, y):
        e = on.max_rel_err(yv.reshape(yo.shape), yo, ao)
        if not e <= on.TOL_F32:
            bad.append((p, t.values(p), e))
    assert not bad, bad[:5]
    assert len(sel) > 100


@pytest.mark.parametrize("sk", [0, 7])
def test_simt_gemm_exact_integer_inputs(sk):
    b, m, n, k = 1, 70, 45, 92
    x, w, yo, _ = gemm_case(b, m, n, k, "int", 5)
    xd, wd = to_dev(x, w)
    y = torch.empty(b, m, n, device=dev())
    t = Tuner("dense", {"m": m, "n": n, "k": k}, spaces=[(sk, sketch_space(sk))], x=xd, w=wd, y=y)
    pts = [p for p in all_points(sk) if t.valid(p)]
    for p, yv in run_points(t, random.Random(1).sample(pts, 200), xd, wd, y):
        np.testing.assert_array_equal(yv.reshape(yo.shape), yo.astype(np.float32), err_msg=str(t.values(p)))


CONV_CASES = [
    # N, H, W, C, K, R, S, stride, pad, dil
    (1, 13, 11, 3, 10, 3, 3, (1, 1), (1, 1), (1, 1)),
    (2, 9, 9, 8, 20, 3, 3, (2, 2), (1, 1), (1, 1)),
    (1, 15, 15, 3, 16, 7, 7, (2, 2), (3, 3), (1, 1)),
    (1, 10, 12, 12, 9, 1, 1, (2, 2), (0, 0), (1, 1)),
    (1, 11, 10, 4, 6, 3, 2, (1, 2), (2, 0), (2, 1)),
]


@pytest.mark.parametrize("sk", [1, 8, 9])  # simt_igemm_conv_f32, simt_pipe_conv_f32, simt_direct_conv_f32
@pytest.mark.parametrize("case", CONV_CASES)
def test_simt_igemm_conv_vs_oracle(case, sk):
    n, h, wd_, c, k, r, s, st, pd, dl = case
    x, w = tensors([(n, h, wd_, c), (k, r, s, c)], sum(case[:7]))
    yo, ao = oc.conv2d(x, w, st, pd, dl)
    xd, wdd = to_dev(x, w)
    y = torch.empty(yo.shape, device=dev())
    shape = {"N": n, "H": h, "W": wd_, "C": c, "K": k, "R": r, "S": s, "stride": st, "pad": pd, "dil": dl}
    t = Tuner("conv2d", shape, spaces=[(sk, sketch_space(sk))], x=xd, w=wdd, y=y)
    pts = [p for p in all_points(sk) if t.valid(p)]
    assert len(pts) > 50
    bad = []
    for p, yv in run_points(t, random.Random(2).sample(pts, min(300, len(pts))), xd, wdd, y):
        e = on.max_rel_err(yv, yo, ao)
        if not e <= on.TOL_F32:
            bad.append((t.values(p), e))
    assert not bad, bad[:5]


@pytest.mark.parametrize("sk", [1, 8, 9])
def test_simt_conv_exact_integer_inputs(sk):
    # integer inputs in {-2..2}: every partial sum is exact in fp32, so any summation order
    # (split-K atomics, sliced-K groups, k-parity halves) must reproduce the oracle bit for bit
    n, h, wd_, c, k, r, s = 2, 11, 9, 12, 20, 3, 3
    x, w = tensors([(n, h, wd_, c), (k, r, s, c)], 9, "int")
    yo, _ = oc.conv2d(x, w, (2, 1), (1, 1))
    xd, wdd = to_dev(x, w)
    y = torch.empty(yo.shape, device=dev())
    shape = {"N": n, "H": h, "W": wd_, "C": c, "K": k, "R": r, "S": s, "stride": (2, 1), "pad": (1, 1)}
    t = Tuner("conv2d", shape, spaces=[(sk, sketch_space(sk))], x=xd, w=wdd, y=y)
    pts = [p for p in all_points(sk) if t.valid(p)]
    for p, yv in run_points(t, random.Random(4).sample(pts, min(200, len(pts))), xd, wdd, y):
        np.testing.assert_array_equal(yv, yo.astype(np.float32), err_msg=str(t.values(p)))


@pytest.mark.parametrize("sk", [1, 8])
def test_splitk_back_to_back_launches(sk):
    # split-K zeroes Y with a kernel that releases the partial-sum kernel early (PDL); back-to-back
    # launches (eager and replayed from a CUDA graph, as the timing harness does) must still leave
    # exactly one launch's sum in Y: each zeroing waits for the previous launch to finish, and each
    # partial-sum kernel waits for its zeroing before its first atomic
    n, h, wd_, c, k, r, s = 1, 14, 14, 64, 64, 3, 3
    x, w = tensors([(n, h, wd_, c), (k, r, s, c)], 21)
    yo, ao = oc.conv2d(x, w, (1, 1), (1, 1))
    xd, wdd = to_dev(x, w)
    y = torch.empty(yo.shape, device=dev())
    shape = {"N": n, "H": h, "W": wd_, "C": c, "K": k, "R": r, "S": s, "stride": (1, 1), "pad": (1, 1)}
    space = sketch_space(sk)
    t = Tuner("conv2d", shape, spaces=[(sk, space)], x=xd, w=wdd, y=y)
    pts = [p for p in all_points(sk) if t.valid(p) and t.values(p)[7] >= 4]
    assert pts
    st = torch.cuda.Stream()
    for p in random.Random(5).sample(pts, 12):
        y.fill_(float("nan"))
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            for _ in range(20):
                t.run(p, xd, wdd, y, stream=st)
        st.synchronize()
        assert on.max_rel_err(y.cpu().numpy(), yo, ao) <= on.TOL_F32, ("eager", t.values(p))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(8):
                t.run(p, xd, wdd, y, stream=st)
        y.fill_(float("nan"))
        torch.cuda.synchronize()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        assert on.max_rel_err(y.cpu().numpy(), yo, ao) <= on.TOL_F32, ("graph", t.values(p))


def test_naive_reference_vs_oracle():
    x, w = tensors([(2, 10, 9, 5), (7, 3, 3, 5)], 3)
    yo, ao = oc.conv2d(x, w, (2, 1), (1, 1))
    xd, wd = to_dev(x, w)
    y = torch.empty(yo.shape, device=dev())
    shape = {"N": 2, "H": 10, "W": 9, "C": 5, "K": 7, "R": 3, "S": 3, "stride": (2, 1), "pad": (1, 1)}
    t = Tuner("conv2d", shape, spaces=[(1, sketch_space(1))], x=xd, w=wd, y=y)
    yr, ar = torch.empty_like(y), torch.empty_like(y)
    t.reference(xd, wd, yr, ar)
    torch.cuda.synchronize()
    np.testing.assert_allclose(yr.cpu().numpy(), yo.astype(np.float32), rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(ar.cpu().numpy(), ao.astype(np.float32), rtol=1e-6)


@pytest.mark.parametrize("policy", ["grow", "radius"])
def test_harness_sample_droplet_and_replay(policy):
    from oracle.search import OracleTuner, Space
    m = n = k = 256
    x, w, yo, ao = gemm_case(1, m, n, k, "uniform", 11)
    xd, wd = to_dev(x, w)
    y = torch.empty(m, n, device=dev())
    t = Tuner("dense", {"m": m, "n": n, "k": k}, x=xd, w=wd, y=y, seed=3, policy=policy)
    l0 = global_launch_count()
    smp = t.sample(64)
    assert len(smp) == 64
    assert all(s.status == "ok" and s.max_err <= 1e-4 and 0 < s.cost_ns < 1e8 for s in smp), smp[:3]
    assert global_launch_count() - l0 >= 64 * (1 + 2 + 10)
    pre = {(s.point[0], s.point[1]): s.cost_ns for s in t.history()}
    b = t.best()
    assert b.cost_ns == min(s.cost_ns for s in smp)
    rep = t.droplet(b.point, 100)
    assert rep["trials_used"] <= 100
    log = {(s.point[0], s.point[1]): s.cost_ns for s in t.history()}
    # record/replay: the oracle's Droplet over the logged costs
    # reproduces the GPU trajectory and never asks for an unlogged point
    # the oracle's points are (position in the space list, index vector); the library's
    # are (sketch id, index vector): the default dense f32 spaces are every f32 dense sketch
    sks = sketches("dense", "f32")
    sp = Space([sketch_space(s) for s in sks])
    to_o = lambda p: (sks.index(p[0]), tuple(p[1]))
    to_l = lambda p: (sks[p[0]], tuple(p[1]))

    def cost(p):
        return log[to_l(p)]
    ot = OracleTuner(sp, cost, lambda p: to_l(p) in log)
    ot.measure([to_o(p) for p in pre])
    orep = ot.droplet(to_o(b.point), 100, policy)
    assert [to_l(p) for p in orep["traj"]] == [(p[0], tuple(p[1])) for p in rep["traj"]]
    assert orep["trials_used"] == rep["trials_used"] and orep["converged"] == rep["converged"]
    # the chosen schedule really computes the layer
    t.run(rep["best"], xd, wd, y)
    torch.cuda.synchronize()
    assert on.max_rel_err(y.cpu().numpy(), yo, ao) <= 1e-4


# ---------------------------------------------------------------- tcgen05 bf16 sketch
def bf16_case(b, m, n, k, dist, seed):
    x, w = tensors([(b, m, k), (b, n, k)], seed, dist)
    x, w = on.round_bf16(x), on.round_bf16(w)  # RNE before both paths (R-C4)
    yo, ao = oc.bmm(x, w)
    xd = torch.from_numpy(x).to(dev()).to(torch.bfloat16)
    wd = torch.from_numpy(w).to(dev()).to(torch.bfloat16)
    return xd, wd, yo, ao


@pytest.mark.parametrize("shape", [(1, 200, 136, 72), (2, 128, 256, 256), (1, 512, 384, 1024), (3, 77, 300, 40)])
def test_tc_gemm_all_configs_vs_oracle(shape):
    b, m, n, k = shape
    op = "dense" if b == 1 else "batch_matmul"
    xd, wd, yo, ao = bf16_case(b, m, n, k, "uniform", sum(shape))
    y = torch.empty(b, m, n, device=dev())
    t = Tuner(op, {"b": b, "m": m, "n": n, "k": k}, dtype="bf16", spaces=[(2, sketch_space(2))], x=xd, w=wd, y=y)
    pts = [p for p in all_points(2) if t.valid(p)]
    assert len(pts) >= 10
    # every compiled (BM, BN, BK) instantiation, with a sample of the runtime knobs over it
    rng = random.Random(sum(shape))
    by_inst = {}
    for p in pts:
        by_inst.setdefault(tuple(p[1][:3]) + (p[1][8],), []).append(p)
    sel = [q for group in by_inst.values() for q in rng.sample(group, min(len(group), 40))]
    bad, worst = [], 0.0
    for p, yv in run_points(t, sel, xd, wd, y):
        e = on.max_rel_err(yv.reshape(yo.shape), yo, ao)
        worst = max(worst, e)
        if not e <= 1e-5:  # fp32 accumulation of exact bf16 products: far inside the 2e-2 bar
            bad.append((t.values(p), e))
    assert not bad, bad[:5]
    print("tc_gemm worst err", worst)


def test_tc_gemm_exact_integer_inputs():
    b, m, n, k = 1, 256, 192, 320
    xd, wd, yo, _ = bf16_case(b, m, n, k, "int", 7)
    y = torch.empty(b, m, n, device=dev())
    t = Tuner("dense", {"m": m, "n": n, "k": k}, dtype="bf16", spaces=[(2, sketch_space(2))], x=xd, w=wd, y=y)
    pts = [p for p in all_points(2) if t.valid(p)]
    for p, yv in run_points(t, random.Random(3).sample(pts, min(400, len(pts))), xd, wd, y):
        np.testing.assert_array_equal(yv.reshape(yo.shape), yo.astype(np.float32), err_msg=str(t.values(p)))


def test_tc_harness_bert_like():
    m, n, k = 1024, 768, 768
    xd, wd, yo, ao = bf16_case(1, m, n, k, "uniform", 12)
    y = torch.empty(m, n, device=dev())
    t = Tuner("dense", {"m": m, "n": n, "k": k}, dtype="bf16", x=xd, w=wd, y=y, seed=1)
    smp = t.sample(40)
    assert smp and all(s.status == "ok" and s.max_err <= 2e-2 for s in smp), smp[:3]
    rep = t.droplet(t.best().point, 50)
    print("tc best", t.values(rep["best"]), rep["best_cost"], "ns", 2 * m * n * k / rep["best_cost"] / 1e3, "TF")


@pytest.mark.parametrize("shape,vals", [
    ((1, 75, 53, 36), [16, 16, 4, 2, 1, 1, 1, 2]),      # 9 k-tiles in 2 ragged slices (5 + 4)
    ((3, 33, 17, 130), [32, 16, 32, 2, 2, 1, 2, 3]),    # 5 k-tiles in 3 ragged slices (2 + 2 + 1)
    ((1, 128, 128, 64), [64, 64, 16, 4, 4, 4, 2, 4]),
])
def test_simt_split_k_repeat_and_graph(shape, vals):
    """Split-K (zeroing + atomic partial sums): back-to-back launches on the same y,
    launches inside a captured CUDA graph, ragged k splits (a shorter last slice; a split
    that would leave a slice empty is statically invalid) -- every launch and every replay
    equals the oracle."""
    b, m, n, k = shape
    op = "dense" if b == 1 else "batch_matmul"
    x, w, yo, ao = gemm_case(b, m, n, k, "uniform", 7 + k)
    xd, wd = to_dev(x, w)
    y = torch.full((b, m, n), float("nan"), device=dev())
    sp = sketch_space(0)
    t = Tuner(op, {"b": b, "m": m, "n": n, "k": k}, spaces=[(0, sp)], x=xd, w=wd, y=y)
    p = (0, tuple(sp[d].index(v) for d, v in enumerate(vals)))
    assert t.valid(p)
    for _ in range(5):
        t.run(p, xd, wd, y)  # no zeroing between launches
        torch.cuda.synchronize()
        assert on.max_rel_err(y.cpu().numpy().reshape(yo.shape), yo, ao) <= on.TOL_F32
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(3):
                t.run(p, xd, wd, y, stream=s)
    for _ in range(4):
        y.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        assert on.max_rel_err(y.cpu().numpy().reshape(yo.shape), yo, ao) <= on.TOL_F32
    r = t.measure([p])[0]
    assert r.status == "ok" and r.max_err <= on.TOL_F32


def test_batched_costs_match_single_measurements():
    """Timing graphs are reused across candidates (cudaGraphExecUpdate): costs of an
    interleaved batch of fast and slow schedules equal their one-at-a-time costs,
    so no enqueued launch ever runs another candidate's kernel."""
    m, n, k = 256, 256, 512
    x, w, yo, ao = gemm_case(1, m, n, k, "uniform", 5)
    xd, wd = to_dev(x, w)
    y = torch.empty(1, m, n, device=dev())
    sp = sketch_space(0)
    pick = lambda vals: (0, tuple(sp[d].index(v) for d, v in enumerate(vals)))  # noqa: E731
    fast = [pick([64, 64, 16, 4, 4, 4, 2, 2]), pick([32, 64, 16, 4, 4, 4, 2, 4])]
    slow = [pick([16, 16, 4, 2, 1, 1, 1, 1]), pick([16, 32, 4, 2, 1, 1, 1, 1])]
    order = [fast[0], slow[0], fast[1], slow[1]]
    single = {}
    for p in order:
        t1 = Tuner("dense", {"m": m, "n": n, "k": k}, spaces=[(0, sp)], x=xd, w=wd, y=y, seed=1)
        single[p] = t1.measure([p])[0].cost_ns
        t1.close()
    t = Tuner("dense", {"m": m, "n": n, "k": k}, spaces=[(0, sp)], x=xd, w=wd, y=y, seed=2)
    batch = t.measure(order)
    assert max(single[p] for p in slow) > 3 * min(single[p] for p in fast)
    for p, r in zip(order, batch):
        assert r.status == "ok"
        assert 0.6 < r.cost_ns / single[p] < 1.6, (t.values(p), r.cost_ns, single[p])
    # a swapped graph would give the fast schedules the slow ones' time and vice versa
    assert max(r.cost_ns for p, r in zip(order, batch) if p in fast) < min(
        r.cost_ns for p, r in zip(order, batch) if p in slow)


def test_nccl_exchange_path_world1():
    """The NCCL all-gather path (dlopen'ed libnccl, communicator from a unique id,
    96-B result slots) end to end on a 1-rank NCCL group: every batch goes
    through the collective, and the search behaves as without it."""
    import os
    import socket

    import torch.distributed as dist
    if dist.is_initialized():
        pytest.skip("a process group is already initialised")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev())
    try:
        m, n, k = 96, 80, 72
        x, w, yo, ao = gemm_case(1, m, n, k, "uniform", 21)
        xd, wd = to_dev(x, w)
        y = torch.empty(1, m, n, device=dev())
        t = Tuner("dense", {"m": m, "n": n, "k": k}, spaces=[(0, sketch_space(0))], x=xd, w=wd, y=y, seed=4,
                  group=dist.group.WORLD, max_batch=16)
        smp = t.sample(40)
        rep = t.droplet(t.best().point, 20)
        st = t.stats()
        # one all-gather per non-empty batch (world 1: no tier or calibration collectives)
        assert st["collectives"] == st["batches"] >= 3 + 1
        assert len(smp) == 40 and all(s.status == "ok" and s.rank == 0 for s in smp)
        assert all(np.isfinite(s.cost_ns) for s in t.history())
        t.run(rep["best"], xd, wd, y)
        torch.cuda.synchronize()
        assert on.max_rel_err(y.cpu().numpy().reshape(yo.shape), yo, ao) <= on.TOL_F32
        t.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sk,case", [(7, (1, 75, 53, 200)), (7, (3, 33, 40, 130)), (8, CONV_CASES[1]), (8, CONV_CASES[4]),
                                     (8, (1, 14, 14, 64, 64, 3, 3, (1, 1), (1, 1), (1, 1)))])
def test_pipe_cluster_splitk_vs_oracle(sk, case):
    """RED = 1: the SPLIT_K CTAs of a tile form a thread-block cluster and reduce their partial
    tiles through distributed shared memory (no zeroing kernel, no atomics): every such valid
    schedule (sampled) equals the oracle, and on integer inputs bit for bit, also from a
    replayed CUDA graph."""
    space = sketch_space(sk)
    ired = knob_names(sk).index("RED")
    if sk == 7:
        b, m, n, k = case
        x, w = tensors([(b, m, k), (b, n, k)], sum(case), "int")
        yo, _ = oc.bmm(x, w)
        op, shape = ("dense" if b == 1 else "batch_matmul"), {"b": b, "m": m, "n": n, "k": k}
    else:
        nn, h, wd_, c, kk, r, s, st, pd, dl = case
        x, w = tensors([(nn, h, wd_, c), (kk, r, s, c)], sum(case[:7]), "int")
        yo, _ = oc.conv2d(x, w, st, pd, dl)
        op, shape = "conv2d", {"N": nn, "H": h, "W": wd_, "C": c, "K": kk, "R": r, "S": s, "stride": st, "pad": pd,
                               "dil": dl}
    xd, wdd = to_dev(x, w)
    y = torch.empty(yo.shape, device=dev())
    t = Tuner(op, shape, spaces=[(sk, space)], x=xd, w=wdd, y=y)
    pts = [p for p in all_points(sk) if p[1][ired] == 1 and t.valid(p)]
    assert len(pts) > 20
    for p, yv in run_points(t, random.Random(8).sample(pts, min(250, len(pts))), xd, wdd, y):
        np.testing.assert_array_equal(yv.reshape(yo.shape), yo.astype(np.float32), err_msg=str(t.values(p)))
    p = pts[0]
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(3):
                t.run(p, xd, wdd, y, stream=s)
    y.fill_(float("nan"))
    g.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy().reshape(yo.shape), yo.astype(np.float32))
    res = t.measure(pts[:16])
    assert all(r.status == "ok" for r in res), [(t.values(r.point), r.status) for r in res if r.status != "ok"]


def test_batched_costs_mixed_launch_shapes():
    """The timing-graph executable cache (cudaGraphExecUpdate) never carries one candidate's
    launch shape over to another: a batch interleaving split-K schedules reduced by atomics
    (zeroing node + programmatic edge), by a thread-block cluster (RED = 1, cluster dims), and
    plain launches of the same sketch gives every candidate its one-at-a-time cost."""
    n, h, wd_, c, k = 1, 28, 28, 128, 128
    x, w = tensors([(n, h, wd_, c), (k, 3, 3, c)], 41)
    xd, wdd = to_dev(x, w)
    y = torch.empty(n, h, wd_, k, device=dev())
    shape = {"N": n, "H": h, "W": wd_, "C": c, "K": k, "R": 3, "S": 3, "stride": (1, 1), "pad": (1, 1)}
    sp = sketch_space(8)
    pick = lambda vals: (8, tuple(sp[d].index(v) for d, v in enumerate(vals)))  # noqa: E731
    pts = [pick([32, 64, 32, 4, 1, 4, 2, 6, 0, 1]), pick([16, 64, 32, 4, 1, 4, 2, 1, 0, 0]),
           pick([32, 64, 32, 4, 1, 4, 2, 6, 0, 0]), pick([64, 64, 16, 4, 1, 4, 2, 4, 0, 1]),
           pick([16, 128, 32, 4, 2, 4, 3, 1, 0, 0]), pick([64, 64, 16, 4, 1, 4, 2, 4, 0, 0])]
    single = {}
    for p in pts:
        t1 = Tuner("conv2d", shape, spaces=[(8, sp)], x=xd, w=wdd, y=y, seed=1)
        assert t1.valid(p), t1.values(p)
        single[p] = t1.measure([p])[0].cost_ns
        t1.close()
    t = Tuner("conv2d", shape, spaces=[(8, sp)], x=xd, w=wdd, y=y, seed=2)
    for p, r in zip(pts, t.measure(pts)):
        assert r.status == "ok"
        assert 0.7 < r.cost_ns / single[p] < 1.4, (t.values(p), r.cost_ns, single[p])
