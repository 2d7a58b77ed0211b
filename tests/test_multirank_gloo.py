"""Candidate sharding across ranks: with world = 2 over gloo
(CPU), batch item j is measured by rank j mod 2 and the results are
all-gathered, so every rank holds the identical history and takes the same
descent steps; trajectories equal the world = 1 run and the oracle."""
import json
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    from tests.test_costtable_parity import make_case, run_product
    from synth import landscape
    res = []
    for seed, fam, pol in [(0, "rugged", "grow"), (3, "correlated_valley", "plain"), (4, "plateau", "grow")]:
        sk = make_case(seed * 7 + 1)
        table = landscape([[len(v) for v in s] for s in sk], fam, seed, 0.1)
        out, t = run_product(sk, table, seed, pol, 40, 100, 9, group=dist.group.WORLD)
        ranks = [s.rank for s in t.history()]
        out["stats"] = t.stats()
        out["ranks"] = ranks
        res.append(out)
        t.close()
    with open(os.path.join(outdir, f"r{rank}.json"), "w") as f:
        json.dump(res, f)
    dist.destroy_process_group()


def test_two_rank_gloo_matches_single_rank(tmp_path):
    port = free_port()
    mp.spawn(worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0 = json.load(open(tmp_path / "r0.json"))
    r1 = json.load(open(tmp_path / "r1.json"))
    from tests.test_costtable_parity import make_case, run_oracle
    from synth import landscape
    for i, (seed, fam, pol) in enumerate([(0, "rugged", "grow"), (3, "correlated_valley", "plain"),
                                          (4, "plateau", "grow")]):
        a, b = r0[i], r1[i]
        assert a["stats"]["collectives"] > 0
        for key in ("sample", "best", "droplet", "history"):
            assert a[key] == b[key], key
        sk = make_case(seed * 7 + 1)
        table = landscape([[len(v) for v in s] for s in sk], fam, seed, 0.1)
        o, _ = run_oracle(sk, table, seed, pol, 40, 100, 9)
        o = json.loads(json.dumps(o))  # tuples -> lists like the workers' JSON
        for key in ("sample", "best", "droplet", "history"):
            assert a[key] == o[key], key
        assert set(a["ranks"]) == {0, 1}
