"""Cost-table mode (R-T1): the C++ driver behind the C ABI must reproduce the
oracle's sampled set, history order, best-of-N and Droplet trajectory bit for
bit ("Search trajectories ... under cost-table mode must match
the oracle bit-exactly").  CPU only: no device is touched in this mode."""
import math
import random

import numpy as np
import pytest

from oracle.search import OracleTuner, Space, random_baseline, table_cost
from paper_2406_20037_b200 import Tuner, TunerError
from synth import FAMILIES, landscape

LABEL0 = 40  # sketch ids are free labels in cost-table mode


def make_case(seed, nsk=None):
    rng = random.Random(seed)
    nsk = nsk or rng.randint(1, 3)
    sketches = []
    for _ in range(nsk):
        d = rng.randint(1, 5)
        sketches.append([sorted(rng.sample(range(1, 300), rng.randint(1, 8))) for _ in range(d)])
    return sketches


def run_oracle(sketches, table, seed, policy, n_sample, budget, max_batch):
    sp = Space(sketches)
    cost, valid = table_cost(sp, table)
    t = OracleTuner(sp, cost, valid, seed)
    smp = t.sample(n_sample, max_batch)
    out = {"sample": [(LABEL0 + p[0], p[1], c) for p, c in smp]}
    if not t.history:
        return out, t
    bp, bc = t.best()
    out["best"] = (LABEL0 + bp[0], bp[1], bc)
    rep = t.droplet(bp, budget, policy)
    out["droplet"] = {k: rep[k] for k in ("best_cost", "trials_used", "rounds", "converged")}
    out["droplet"]["best"] = (LABEL0 + rep["best"][0], rep["best"][1])
    out["droplet"]["traj"] = [(LABEL0 + p[0], p[1]) for p in rep["traj"]]
    out["history"] = [(LABEL0 + p[0], p[1], c) for p, c in t.history]
    return out, t


def run_product(sketches, table, seed, policy, n_sample, budget, max_batch, group=None):
    spaces = [(LABEL0 + i, v) for i, v in enumerate(sketches)]
    t = Tuner("dense", {"m": 1, "n": 1, "k": 1}, spaces=spaces, cost_table=table, seed=seed, policy=policy,
              max_batch=max_batch, group=group)
    smp = t.sample(n_sample)
    out = {"sample": [(s.point[0], s.point[1], s.cost_ns) for s in smp]}
    if not smp:
        return out, t
    b = t.best()
    out["best"] = (b.point[0], b.point[1], b.cost_ns)
    rep = t.droplet(b.point, budget)
    out["droplet"] = {k: rep[k] for k in ("best_cost", "trials_used", "rounds", "converged")}
    out["droplet"]["best"] = rep["best"]
    out["droplet"]["traj"] = rep["traj"]
    out["history"] = [(s.point[0], s.point[1], s.cost_ns) for s in t.history()]
    return out, t


CASES = [(fam, seed, pol) for fam in FAMILIES for seed in range(6) for pol in ("plain", "grow", "radius")]


@pytest.mark.parametrize("family,seed,policy", CASES)
def test_trajectory_bit_exact(family, seed, policy):
    sketches = make_case(seed * 31 + len(family))
    cards = [[len(v) for v in s] for s in sketches]
    table = landscape(cards, family, seed, invalid_fraction=0.1 if seed % 2 else 0.0)
    n_sample = [1, 5, 30, 300][seed % 4]
    budget = [100, 7, 1, 100, 25, 100][seed]
    a, _ = run_oracle(sketches, table, seed, policy, n_sample, budget, 13)
    b, t = run_product(sketches, table, seed, policy, n_sample, budget, 13)
    assert a == b
    t.close()


def test_paper_example_through_abi():
    # Example 2.3 space, f(i,j) = (i-3)^2 + 2(j-2)^2 + 1, start (0,0) (tests/golden)
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "droplet_example_2_3.json")))
    table = [float((i - 3) ** 2 + 2 * (j - 2) ** 2 + 1) for i in range(5) for j in range(5)]
    for policy in ("plain", "grow"):
        t = Tuner("dense", {"m": 1, "n": 1, "k": 1}, spaces=[(7, g["values"])], cost_table=table, policy=policy)
        rep = t.droplet((7, (0, 0)), 100)
        exp = g[policy]
        assert [list(p[1]) for p in rep["traj"]] == exp["traj"]
        assert (rep["trials_used"], rep["rounds"], rep["converged"]) == (exp["trials_used"], exp["rounds"], exp["converged"])
        assert rep["best_cost"] == exp["best_cost"]


def test_random_baseline_and_exhaustive_match():
    sketches = make_case(5, 2)
    cards = [[len(v) for v in s] for s in sketches]
    table = landscape(cards, "rugged", 3, 0.1)
    sp = Space(sketches)
    cost, valid = table_cost(sp, table)
    o = OracleTuner(sp, cost, valid, 9)
    random_baseline(o, k=10000)
    t = Tuner("dense", {"m": 1, "n": 1, "k": 1}, spaces=[(LABEL0 + i, v) for i, v in enumerate(sketches)],
              cost_table=table, seed=9)
    allpts = [(LABEL0 + p[0], p[1]) for p in sp.enumerate()]
    res = t.measure(allpts)
    assert sum(r.status == "ok" for r in res) == len(o.history)
    assert t.best().cost_ns == o.best()[1]


def test_errors():
    table = [1.0, 2.0, math.inf, 0.5]
    sp = [(3, [[1, 2], [5, 6]])]
    t = Tuner("dense", {"m": 1, "n": 1, "k": 1}, spaces=sp, cost_table=table)
    with pytest.raises(TunerError, match="ESTATE"):
        t.best()
    with pytest.raises(TunerError, match="EINVAL"):
        t.droplet((3, (0, 0)), 0)
    with pytest.raises(TunerError, match="EDIM"):
        t.droplet((3, (0,)), 10)
    with pytest.raises(TunerError, match="ERANGE"):
        t.droplet((3, (0, 2)), 10)
    with pytest.raises(TunerError, match="ERANGE"):
        t.droplet((3, (1, 0)), 10)  # +inf = invalid start
    with pytest.raises(TunerError, match="ERANGE"):
        t.droplet((4, (0, 0)), 10)  # unknown sketch
    with pytest.raises(TunerError, match="EINVAL"):
        Tuner("dense", {"m": 1, "n": 1, "k": 1}, spaces=sp, cost_table=[1.0, float("nan"), 1.0, 1.0])
    with pytest.raises(TunerError, match="EINVAL"):
        Tuner("dense", {"m": 1, "n": 1, "k": 1}, spaces=sp, cost_table=[1.0, 2.0])
    with pytest.raises(TunerError, match="EINVAL"):
        Tuner("dense", {"m": 1, "n": 1, "k": 1}, spaces=[(3, [[2, 1]])], cost_table=[1.0, 2.0])
    with pytest.raises(TunerError, match="ESTATE"):
        t.run((3, (0, 0)), None, None, None)
    rep = t.droplet((3, (0, 0)), 100)
    # (1,1) = 0.5 is not a neighbour of (0,0); (1,0) is invalid: a local minimum
    assert rep["best"] == (3, (0, 0)) and rep["converged"] and rep["trials_used"] == 2
    r = t.measure([(3, (1, 0)), (3, (0, 0)), (3, (1, 1))])
    assert r[0].status == "invalid" and r[1].status == "ok" and r[2].cost_ns == 0.5
    assert t.stats()["candidates"] == 3 and t.best().point == (3, (1, 1))


def test_sample_exhausts_gracefully():
    table = np.arange(6, dtype=np.float64)
    t = Tuner("dense", {"m": 1, "n": 1, "k": 1}, spaces=[(1, [[1, 2, 3], [1, 2]])], cost_table=table, seed=1)
    got = t.sample(100)
    assert len(got) == 6 and len({s.point for s in got}) == 6
    assert t.sample(5) == []


def test_sampler_hand_trace_product():
    # tests/test_oracle_pins_r2.py::test_sampler_hand_traced_with_rejected_draw through tuner_sample:
    # draw 1 (1,(1,)) is invalid and rejected, draws 2-3 give (0,(1,)), (0,(0,)) (published outputs #1-#6)
    t = Tuner("dense", {"m": 1, "n": 1, "k": 1}, spaces=[(0, [[10, 20]]), (1, [[1, 2, 3]])],
              cost_table=[1.0, 2.0, 3.0, math.inf, 5.0], seed=0)
    assert [s.point for s in t.sample(2)] == [(0, (1,)), (0, (0,))]


@pytest.mark.parametrize("seed", range(4))
def test_per_sketch_droplet_bit_exact(seed):
    # R-D17: after exploration, Droplet from each sketch's best point (tuner_best_of_sketch): the
    # starts, trajectories and final best match the oracle bit for bit in cost-table mode
    rng = random.Random(seed + 40)
    sk = [[list(range(rng.randint(2, 5))) for _ in range(rng.randint(2, 4))] for _ in range(3)]
    table = landscape([[len(v) for v in s] for s in sk], "rugged", seed, 0.1)
    sp = Space(sk)
    c, v = table_cost(sp, table)
    o = OracleTuner(sp, c, v, seed)
    o.sample(20)
    t = Tuner("dense", {"m": 1, "n": 1, "k": 1}, spaces=[(i, s) for i, s in enumerate(sk)], cost_table=table,
              seed=seed)
    t.sample(20)
    for s_ in range(3):
        ob = o.best_of_sketch(s_)
        tb = t.best_of_sketch(s_)
        assert (ob is None) == (tb is None)
        if ob is None:
            continue
        assert (ob[0][0], ob[0][1], ob[1]) == (tb.point[0], tb.point[1], tb.cost_ns)
        orep = o.droplet(ob[0], 40, "grow")
        trep = t.droplet(tb.point, 40)
        assert [p[1] for p in orep["traj"]] == [p[1] for p in trep["traj"]]
        assert (orep["trials_used"], orep["rounds"]) == (trep["trials_used"], trep["rounds"])
    assert o.best()[1] == t.best().cost_ns
