"""Statistical convergence (alpha > 0): with per-point repeat timings
in cost-table mode, the C++ Droplet moves only on significant improvements and
reproduces the oracle's trajectory bit for bit; the library's rank-sum test
agrees with the oracle's enumeration."""
import random

import numpy as np
import pytest

from oracle.search import OracleTuner, Space, table_cost
from oracle.stats import wilcoxon_p
from paper_2406_20037_b200 import Tuner
from synth import FAMILIES, landscape


def noisy(table, nsamp, seed, rel):
    rng = np.random.Generator(np.random.PCG64(seed))
    t = np.asarray(table, np.float64)
    fin = np.isfinite(t)
    smp = np.zeros((t.size, nsamp))
    smp[fin] = t[fin, None] * (1.0 + rel * rng.standard_normal((fin.sum(), nsamp)))
    smp = smp.astype(np.float32).astype(np.float64)  # the library keeps float32 timings
    cost = np.where(fin, smp.mean(1), np.inf)
    return cost, smp


@pytest.mark.parametrize("family,seed", [(f, s) for f in FAMILIES for s in range(3)])
@pytest.mark.parametrize("alpha", [0.05, 0.3])
def test_statistical_droplet_bit_exact(family, seed, alpha):
    rng = random.Random(seed + 100)
    sk = [[list(range(rng.randint(2, 6))) for _ in range(rng.randint(2, 4))]]
    base = landscape([[len(v) for v in s] for s in sk], family, seed, 0.1)
    nsamp = [3, 5, 6][seed]
    cost, smp = noisy(base, nsamp, seed, 0.15)
    sp = Space(sk)
    c, valid = table_cost(sp, cost)
    o = OracleTuner(sp, c, valid, seed, samples=lambda p: list(smp[sp.linear(p)]))
    o.sample(8)
    start = o.best()[0]
    for pol in ("plain", "grow"):
        orep = o.droplet(start, 60, pol, alpha=alpha)
        t = Tuner("dense", {"m": 1, "n": 1, "k": 1}, spaces=[(5, sk[0])], cost_table=cost, cost_samples=smp,
                  seed=seed, policy=pol, alpha=alpha)
        t.sample(8)
        tb = t.best()
        assert tb.point[1] == start[1]
        trep = t.droplet(tb.point, 60)
        assert [p[1] for p in orep["traj"]] == [p[1] for p in trep["traj"]]
        assert (orep["trials_used"], orep["rounds"], orep["converged"]) == (trep["trials_used"], trep["rounds"],
                                                                            trep["converged"])
        assert list(map(float, t.timings(tb.point))) == list(smp[sp.linear(start)])
        # re-arm the oracle for the second policy
        o = OracleTuner(sp, c, valid, seed, samples=lambda p: list(smp[sp.linear(p)]))
        o.sample(8)


def test_significance_stops_earlier_than_strict_compare():
    # identical-in-distribution neighbours: alpha > 0 refuses noise-driven moves
    sk = [[list(range(8)), list(range(8))]]
    base = np.ones(64)
    cost, smp = noisy(base, 5, 1, 0.2)
    strict = Tuner("dense", {"m": 1, "n": 1, "k": 1}, spaces=[(1, sk[0])], cost_table=cost, cost_samples=smp,
                   policy="plain")
    stat = Tuner("dense", {"m": 1, "n": 1, "k": 1}, spaces=[(1, sk[0])], cost_table=cost, cost_samples=smp,
                 policy="plain", alpha=0.05)
    r1 = strict.droplet((1, (0, 0)), 100)
    r2 = stat.droplet((1, (0, 0)), 100)
    assert r2["trials_used"] <= r1["trials_used"]
    assert len(r2["traj"]) <= len(r1["traj"])


@pytest.mark.parametrize("alpha,moves", [(0.0, True), (0.05, False), (0.1, False), (0.15, True)])
def test_alpha_gate_spec_example_product(alpha, moves):
    # SPEC S:228 ({1,2,3} vs {4,5,6}: p = 0.1; "tie when p >= alpha") through the C++ Droplet
    cost = np.array([5.0, 2.0])
    smp = np.array([[4.0, 5.0, 6.0], [1.0, 2.0, 3.0]])
    t = Tuner("dense", {"m": 1, "n": 1, "k": 1}, spaces=[(0, [[0, 1]])], cost_table=cost, cost_samples=smp,
              policy="plain", alpha=alpha)
    rep = t.droplet((0, (0,)), 100)
    assert rep["best"] == ((0, (1,)) if moves else (0, (0,))) and rep["converged"] and rep["trials_used"] == 2
