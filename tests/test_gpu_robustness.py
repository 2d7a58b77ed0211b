"""GPU robustness of the measurement path:

* stream-K / k-chunked tcgen05 schedules (SCHED 1, 2) whose static persistent grid used to
  exceed the co-resident CTA count (heads spin on tails that never get an SM): every such
  schedule of a BERT-like dense layer (tiles mod groups in [capacity, groups/2], S >= 2)
  now completes and matches the oracle -- under the harness's watchdog, so a regression
  fails instead of hanging;
* the stream-K workspace belongs to the handle: two handles running stream-K schedules
  concurrently on two streams both stay correct; a first stream-K launch inside a stream
  capture is refused (ESTATE) instead of allocating inside the capture.
"""
import itertools

import numpy as np
import pytest
import torch

from oracle import contractions as oc
from oracle import numerics as on
from paper_2406_20037_b200 import Tuner, TunerError, sketch_space
from synth import tensors

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def bf16_dense(m, n, k, seed):
    x, w = tensors([(m, k), (n, k)], seed)
    x, w = on.round_bf16(x), on.round_bf16(w)
    yo, ao = oc.dense(x, w)
    return (torch.from_numpy(x).to(DEV).to(torch.bfloat16), torch.from_numpy(w).to(DEV).to(torch.bfloat16), yo, ao)


def sched_points(t, sched_vals):
    sp = sketch_space(2)
    pts = [(2, idx) for idx in itertools.product(*[range(len(v)) for v in sp])]
    return [p for p in pts if t.valid(p) and sp[5][p[1][5]] in sched_vals]


def test_stream_k_schedules_complete_and_match_oracle():
    m, n, k = 2048, 768, 768  # 16 x 12 = 192 tiles of 128 x 64: more tiles than resident groups
    xd, wd, yo, ao = bf16_dense(m, n, k, 31)
    y = torch.empty(m, n, device=DEV)
    t = Tuner("dense", {"m": m, "n": n, "k": k}, dtype="bf16", spaces=[(2, sketch_space(2))], x=xd, w=wd, y=y,
              repeats=2, warmup=1, timeout_ms=2000.0)
    pts = sched_points(t, (1, 2))
    assert len(pts) > 20
    res = t.measure(pts)
    bad = [(t.values(r.point), r.status, r.max_err) for r in res if r.status != "ok" or r.max_err > 1e-5]
    assert not bad, bad[:5]
    for p in pts[:: max(1, len(pts) // 8)]:
        y.fill_(float("nan"))
        t.run(p, xd, wd, y)
        torch.cuda.synchronize()
        assert on.max_rel_err(y.cpu().numpy(), yo, ao) <= 1e-5, t.values(p)


def test_stream_k_workspace_is_per_handle():
    m, n, k = 1024, 768, 1536
    xd, wd, yo, ao = bf16_dense(m, n, k, 32)
    ya = torch.empty(m, n, device=DEV)
    yb = torch.empty(m, n, device=DEV)
    ta = Tuner("dense", {"m": m, "n": n, "k": k}, dtype="bf16", spaces=[(2, sketch_space(2))], x=xd, w=wd, y=ya)
    tb = Tuner("dense", {"m": m, "n": n, "k": k}, dtype="bf16", spaces=[(2, sketch_space(2))], x=xd, w=wd, y=yb)
    pa = sched_points(ta, (1,))[0]
    pb = sched_points(tb, (2,))[-1]
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    ta.run(pa, xd, wd, ya, stream=sa)  # first launches outside any capture: workspaces allocated
    tb.run(pb, xd, wd, yb, stream=sb)
    torch.cuda.synchronize()
    for _ in range(3):
        ya.fill_(float("nan"))
        yb.fill_(float("nan"))
        torch.cuda.synchronize()
        for _ in range(10):  # interleaved, concurrent on two streams
            ta.run(pa, xd, wd, ya, stream=sa)
            tb.run(pb, xd, wd, yb, stream=sb)
        torch.cuda.synchronize()
        assert on.max_rel_err(ya.cpu().numpy(), yo, ao) <= 1e-5
        assert on.max_rel_err(yb.cpu().numpy(), yo, ao) <= 1e-5


def test_first_stream_k_launch_inside_capture_is_refused():
    m, n, k = 512, 256, 512
    xd, wd, yo, ao = bf16_dense(m, n, k, 33)
    y = torch.empty(m, n, device=DEV)
    t = Tuner("dense", {"m": m, "n": n, "k": k}, dtype="bf16", spaces=[(2, sketch_space(2))], x=xd, w=wd, y=y)
    p = sched_points(t, (1,))[0]
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with pytest.raises(TunerError, match="ESTATE"):
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                t.run(p, xd, wd, y, stream=s)
    torch.cuda.synchronize()
    t2 = Tuner("dense", {"m": m, "n": n, "k": k}, dtype="bf16", spaces=[(2, sketch_space(2))], x=xd, w=wd, y=y)
    t2.run(p, xd, wd, y)  # allocates its workspace
    torch.cuda.synchronize()
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g2, stream=s):
            t2.run(p, xd, wd, y, stream=s)
    y.fill_(float("nan"))
    g2.replay()
    torch.cuda.synchronize()
    assert on.max_rel_err(y.cpu().numpy(), yo, ao) <= 1e-5
