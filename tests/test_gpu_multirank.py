"""Measured-mode SPMD at world 2 on ONE B200 (P:276-277 -- the parallelism the
build re-introduces): two processes share cuda:0 over a gloo group, each
measures batch items j = rank (mod 2) of every batch with the real harness (verify + timing +
early-cut and precise tiers), and the results are all-gathered.

Asserted: both ranks end with the identical history (points, costs bit for bit, statuses,
measuring ranks), trajectory and best; both ranks measured candidates; every candidate was
verified against the library's reference; the tiers used the all-gathered references
(collectives beyond one per batch); every accepted point -- each Droplet step and the
best-of-N start -- carries a rank-0 cost (a winner timed on rank 1 is re-timed on rank 0
before acceptance); and the chosen schedule computes the layer (oracle)."""
import json
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPE = {"N": 1, "H": 28, "W": 28, "C": 64, "K": 64, "R": 3, "S": 3, "stride": (1, 1), "pad": (1, 1)}


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    from paper_2406_20037_b200 import Tuner
    from synth import tensors
    x, w = tensors([(1, 28, 28, 64), (64, 3, 3, 64)], 77)
    xd = torch.from_numpy(x).cuda()
    wd = torch.from_numpy(w).cuda()
    y = torch.empty(1, 28, 28, 64, device="cuda")
    t = Tuner("conv2d", SHAPE, x=xd, w=wd, y=y, seed=5, group=dist.group.WORLD, early_cut=4.0, max_batch=64)
    smp = t.sample(128)
    b = t.best()
    rep = t.droplet(b.point, 60)
    t.run(rep["best"], xd, wd, y)
    torch.cuda.synchronize()
    hist = [[s.point[0], list(s.point[1]), s.cost_ns.hex(), s.status, s.rank, s.max_err] for s in t.history()]
    out = {"n_sample": len(smp), "start": [b.point[0], list(b.point[1])],
           "traj": [[p[0], list(p[1])] for p in rep["traj"]],
           "best": [rep["best"][0], list(rep["best"][1])], "best_cost": rep["best_cost"].hex(),
           "history": hist, "stats": t.stats(), "y": y.cpu().numpy().ravel()[::7].tolist()}
    with open(os.path.join(outdir, f"r{rank}.json"), "w") as f:
        json.dump(out, f)
    t.close()
    dist.destroy_process_group()


def test_measured_mode_world2_on_one_gpu(tmp_path):
    mp.spawn(worker, args=(2, free_port(), str(tmp_path)), nprocs=2, join=True)
    r0 = json.load(open(tmp_path / "r0.json"))
    r1 = json.load(open(tmp_path / "r1.json"))
    for key in ("n_sample", "start", "traj", "best", "best_cost", "history"):
        assert r0[key] == r1[key], key
    hist = r0["history"]
    assert r0["n_sample"] == 128
    assert {h[4] for h in hist} == {0, 1}, "both ranks measured candidates"
    bad = [h for h in hist if not (h[3] == "ok" and h[5] <= 1e-4)]
    assert not bad, ("every candidate verified ok", bad[:8])
    rank_of = {(h[0], tuple(h[1])): h[4] for h in hist}
    for p in r0["traj"]:
        assert rank_of[(p[0], tuple(p[1]))] == 0, ("accepted point not re-timed on rank 0", p)
    st = r0["stats"]
    assert st["collectives"] > st["batches"], "the tiers' all-gathered references"
    print("world-2 measured:", len(hist), "candidates,", st["calibrations"], "calibrations,",
          st["early_cut"], "cut,", st["precise"], "precise; stats r1:", r1["stats"])
    from oracle import contractions as oc
    from oracle import numerics as on
    from synth import tensors
    x, w = tensors([(1, 28, 28, 64), (64, 3, 3, 64)], 77)
    yo, ao = oc.conv2d(x, w, (1, 1), (1, 1))
    sel = slice(None, None, 7)
    err = np.max(np.abs(np.array(r0["y"]) - yo.ravel()[sel]) / np.maximum(ao.ravel()[sel], 1e-30))
    assert err <= on.TOL_F32
