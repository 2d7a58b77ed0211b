"""Pins for oracle/search.py against values the paper prints, closed forms,
brute force and invariants (never against the oracle's own formulas)."""
import itertools
import json
import math
import os
import random

import pytest

from oracle.search import (OracleTuner, SplitMix64, Space, brute_force, is_local_min,
                           random_baseline, table_cost)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- PRNG
def test_splitmix64_published_vector():
    g = load("splitmix64.json")
    r = SplitMix64(g["seed"])
    assert [f"{r.next():016x}" for _ in g["outputs_hex"]] == g["outputs_hex"]
    r = SplitMix64(g["seed"])
    assert [r.uniform(5) for _ in g["uniform5_first4"]] == g["uniform5_first4"]


def test_uniform_chi_squared():
    r = SplitMix64(12345)
    m, n = 7, 70000
    counts = [0] * m
    for _ in range(n):
        counts[r.uniform(m)] += 1
    exp = n / m
    chi2 = sum((c - exp) ** 2 / exp for c in counts)
    assert chi2 < 22.5  # df = 6, p ~ 0.001


# ---------------------------------------------------------------- space / ring
def test_example_2_3_neighbourhood_and_size():
    g = load("droplet_example_2_3.json")
    sp = Space([g["values"]])
    assert sp.size(0) == g["space_size"] == 25
    vals = g["values"]
    pv = g["paper_neighbours"]["point_values"]
    p = (0, (vals[0].index(pv[0]), vals[1].index(pv[1])))
    got = [sp.values(q) for q in sp.ring(p)]
    assert got == g["paper_neighbours"]["neighbour_values"]  # order as printed


def test_ring_corner_and_single_point():
    sp = Space([[[1, 2], [1, 2]]])
    assert [sp.values(q) for q in sp.ring((0, (0, 0)))] == [[2, 1], [1, 2]]
    sp1 = Space([[[1]]])
    assert sp1.ring((0, (0,))) == []


def test_ring_cardinality_symmetry_and_enumerate():
    sp = Space([[[1, 2, 3], [4, 5], [6, 7, 8, 9]], [[1, 2], [3]]])
    pts = sp.enumerate()
    assert len(pts) == len(set(pts)) == sp.total == 3 * 2 * 4 + 2
    assert pts[:3] == [(0, (0, 0, 0)), (0, (0, 0, 1)), (0, (0, 0, 2))]  # row-major
    for p in pts:
        cards = sp.cards(p[0])
        b = sum(1 for d, i in enumerate(p[1]) if i == 0) + sum(1 for d, i in enumerate(p[1]) if i == cards[d] - 1)
        assert len(sp.ring(p)) == 2 * len(cards) - b
        for q in sp.ring(p):
            assert p in sp.ring(q)
            assert sum(abs(a - c) for a, c in zip(p[1], q[1])) == 1
        assert sp.point(sp.linear(p)) == p


# ---------------------------------------------------------------- Droplet golden
def example_tuner(seed=0):
    g = load("droplet_example_2_3.json")
    sp = Space([g["values"]])
    cost = lambda p: float((p[1][0] - 3) ** 2 + 2 * (p[1][1] - 2) ** 2 + 1)
    return g, sp, OracleTuner(sp, cost, lambda p: True, seed)


@pytest.mark.parametrize("policy", ["plain", "grow"])
def test_droplet_example_golden(policy):
    g, sp, t = example_tuner()
    rep = t.droplet((0, tuple(g["start"])), budget=100, policy=policy)
    exp = g[policy]
    assert [list(p[1]) for p in rep["traj"]] == exp["traj"]
    assert rep["best_cost"] == exp["best_cost"]
    assert rep["trials_used"] == exp["trials_used"]
    assert rep["rounds"] == exp["rounds"]
    assert rep["converged"] == exp["converged"]
    if "best_values" in exp:
        assert sp.values(rep["best"]) == exp["best_values"]


@pytest.mark.parametrize("policy", ["plain", "grow", "radius"])
def test_droplet_separable_convex_closed_form(policy):
    # cost sum (v_i - 3)^2 on {0..9}^4 from (0,0,0,0) -> (3,3,3,3)
    sp = Space([[list(range(10))] * 4])
    cost = lambda p: float(sum((v - 3) ** 2 for v in p[1]))
    t = OracleTuner(sp, cost, lambda p: True)
    rep = t.droplet((0, (0, 0, 0, 0)), budget=10 ** 6, policy=policy)
    assert rep["best"] == (0, (3, 3, 3, 3)) and rep["best_cost"] == 0.0 and rep["converged"]
    assert rep["trials_used"] <= 10 ** 4


def random_table(rng, dims, inv=0.1):
    cards = [rng.randint(1, 5) for _ in range(dims)]
    n = math.prod(cards)
    tab = [rng.choice([rng.random(), float(rng.randint(0, 4))]) for _ in range(n)]
    for i in range(n):
        if rng.random() < inv:
            tab[i] = math.inf
    return cards, tab


@pytest.mark.parametrize("policy", ["plain", "grow", "radius"])
def test_droplet_invariants_vs_brute_force(policy):
    rng = random.Random(7)
    checked = 0
    for trial in range(600):
        cards, tab = random_table(rng, rng.randint(1, 4))
        sp = Space([[list(range(c)) for c in cards]])
        cost, valid = table_cost(sp, tab)
        starts = [p for p in sp.enumerate() if valid(p)]
        if not starts:
            continue
        start = rng.choice(starts)
        budget = rng.randint(1, 40)
        t = OracleTuner(sp, cost, valid)
        rep = t.droplet(start, budget, policy)
        assert rep["trials_used"] <= budget
        assert rep["trials_used"] == len(t.history)
        costs = [cost(p) for p in rep["traj"]]
        assert all(b < a for a, b in zip(costs, costs[1:])), "accepted costs strictly decrease"
        assert len(set(t.history)) == len(t.history), "no point measured twice"
        if rep["converged"]:
            assert all(q in t.memo for q in sp.ring(rep["best"]) if valid(q))
            assert is_local_min(sp, rep["best"], cost, valid)
            checked += 1
        if policy == "plain":
            for a, b in zip(rep["traj"], rep["traj"][1:]):
                assert b in sp.ring(a)
        if policy == "radius":
            # every move is along one axis; a converged result is optimal along every axis
            # line through it (R-D16): brute force over each line
            for a, b in zip(rep["traj"], rep["traj"][1:]):
                assert sum(i != j for i, j in zip(a[1], b[1])) == 1
            if rep["converged"]:
                c0 = cost(rep["best"])
                for d in range(len(cards)):
                    for i in range(cards[d]):
                        q = (0, rep["best"][1][:d] + (i,) + rep["best"][1][d + 1:])
                        assert not valid(q) or cost(q) >= c0
    assert checked > 200


@pytest.mark.parametrize("policy", ["plain", "grow", "radius"])
def test_droplet_unimodal_reaches_global(policy):
    rng = random.Random(3)
    for _ in range(60):
        d = rng.randint(1, 5)
        cards = [rng.randint(2, 10) for _ in range(d)]
        w = [rng.uniform(0.5, 2) for _ in range(d)]
        m = [rng.uniform(0, c - 1) for c in cards]
        sp = Space([[list(range(c)) for c in cards]])
        cost = lambda p, w=w, m=m: sum(wi * (i - mi) ** 2 for wi, i, mi in zip(w, p[1], m))
        bp, bc = brute_force(sp, cost, lambda p: True)
        start = (0, tuple(rng.randrange(c) for c in cards))
        t = OracleTuner(sp, cost, lambda p: True)
        rep = t.droplet(start, 10 ** 5, policy)
        assert rep["best"] == bp and rep["converged"]


def test_radius_escapes_a_ring_trap_hand_traced():
    # 1-D table [5, 4, 6, 1, 7] from index 0 (R-D16).  PLAIN: ring {1}: 4 < 5 -> move; ring
    # {0, 2} = {5, 6}: no move -> converged at 1 (cost 4), 3 trials, 2 rounds.  RADIUS: at 1, ring
    # r=2 = {3} (index -1 out of range): 1 < 4 -> move to 3, r = 1; ring {2, 4} = {6, 7} (2
    # memoised): no; r=2 {1} memoised: no; r=3 {0} memoised: no; r=4: nothing in range ->
    # converged at 3 (cost 1): trials 1 + 1 + 1 + 1 + 1 = 5 (0, 1, 2, 3, 4), rounds 2 + 1 + 3 = 6
    tab = [5.0, 4.0, 6.0, 1.0, 7.0]
    sp = Space([[list(range(5))]])
    cost, valid = table_cost(sp, tab)
    t = OracleTuner(sp, cost, valid)
    rp = t.droplet((0, (0,)), 100, "plain")
    assert rp["best"] == (0, (1,)) and rp["trials_used"] == 3 and rp["rounds"] == 2 and rp["converged"]
    t = OracleTuner(sp, cost, valid)
    rr = t.droplet((0, (0,)), 100, "radius")
    assert [p[1][0] for p in rr["traj"]] == [0, 1, 3]
    assert rr["best_cost"] == 1.0 and rr["trials_used"] == 5 and rr["rounds"] == 6 and rr["converged"]


def test_radius_equals_plain_when_plain_ends_axis_optimal():
    # the radius-1 phase is PLAIN verbatim: whenever PLAIN's converged point is already optimal
    # along every axis line, RADIUS takes the same trajectory and only adds the outer rings
    rng = random.Random(13)
    same = 0
    for _ in range(400):
        cards, tab = random_table(rng, rng.randint(1, 3), inv=0.0)
        sp = Space([[list(range(c)) for c in cards]])
        cost, valid = table_cost(sp, tab)
        start = (0, tuple(rng.randrange(c) for c in cards))
        rp = OracleTuner(sp, cost, valid).droplet(start, 10 ** 4, "plain")
        rr = OracleTuner(sp, cost, valid).droplet(start, 10 ** 4, "radius")
        c0 = cost(rp["best"])
        axis_opt = all(cost((0, rp["best"][1][:d] + (i,) + rp["best"][1][d + 1:])) >= c0
                       for d in range(len(cards)) for i in range(cards[d]))
        if axis_opt:
            assert rr["traj"] == rp["traj"] and rr["trials_used"] >= rp["trials_used"]
            same += 1
        else:
            assert rr["best_cost"] < rp["best_cost"]  # it escaped PLAIN's ring trap
    assert same > 100


def test_grow_within_100_trials_on_convex():
    # GROW needs <= 77 trials on weighted separable-convex tables (dims <= 5, <= 10 values)
    rng = random.Random(11)
    for _ in range(100):
        d = rng.randint(1, 5)
        cards = [rng.randint(2, 10) for _ in range(d)]
        w = [rng.uniform(0.5, 2) for _ in range(d)]
        m = [rng.uniform(0, c - 1) for c in cards]
        sp = Space([[list(range(c)) for c in cards]])
        cost = lambda p, w=w, m=m: sum(wi * (i - mi) ** 2 for wi, i, mi in zip(w, p[1], m))
        bp, _ = brute_force(sp, cost, lambda p: True)
        t = OracleTuner(sp, cost, lambda p: True)
        rep = t.droplet((0, tuple(rng.randrange(c) for c in cards)), 100, "grow")
        assert rep["best"] == bp


def test_droplet_budget_truncation_and_memo():
    g, sp, t = example_tuner()
    rep = t.droplet((0, (0, 0)), budget=4, policy="plain")
    assert rep["trials_used"] == 4 and not rep["converged"]
    # a second call starting at the incumbent re-uses the memo: nothing re-measured
    n0 = len(t.history)
    rep2 = t.droplet(rep["best"], budget=100, policy="plain")
    assert len(t.history) - n0 == rep2["trials_used"]
    assert rep2["best_cost"] == 1.0 and rep2["converged"]


def test_droplet_rejects_bad_args():
    g, sp, t = example_tuner()
    with pytest.raises(ValueError):
        t.droplet((0, (0, 0)), budget=0)
    sp2 = Space([[[1, 2]]])
    t2 = OracleTuner(sp2, lambda p: 1.0, lambda p: p[1][0] == 1)
    with pytest.raises(ValueError):
        t2.droplet((0, (0,)), 10)


# ---------------------------------------------------------------- sampler / best / baseline
def test_sampler_distinct_valid_and_capped():
    sp = Space([[list(range(4)), list(range(3))], [list(range(5))]])
    valid = lambda p: sum(p[1]) % 3 != 1
    t = OracleTuner(sp, lambda p: float(sp.linear(p)), valid, seed=5)
    got = t.sample(10)
    pts = [p for p, _ in got]
    assert len(pts) == len(set(pts)) == 10 and all(valid(p) for p in pts)
    nvalid = sum(valid(p) for p in sp.enumerate())
    more = t.sample(1000)  # cannot exceed the remaining valid points; stops at 64n attempts
    assert len(more) <= nvalid - 10
    assert len(set(p for p, _ in t.history)) == len(t.history)


def test_sampler_first_draw_by_hand():
    # seed 0, one sketch of 5x5: draws are sketch=uniform(1), then uniform(5) twice
    sp = Space([[list(range(5)), list(range(5))]])
    t = OracleTuner(sp, lambda p: 0.0, lambda p: True, seed=0)
    p = t.draw(1)[0]
    g = load("splitmix64.json")
    # outputs #1 -> sketch 0 (uniform(1)), #2 -> uniform(5)=2, #3 -> uniform(5)=0
    assert p == (0, (g["uniform5_first4"][1], g["uniform5_first4"][2]))


def test_best_first_argmin():
    sp = Space([[list(range(6))]])
    tab = [3.0, 1.0, 2.0, 1.0, math.inf, 5.0]
    cost, valid = table_cost(sp, tab)
    t = OracleTuner(sp, cost, valid)
    t.measure([(0, (0,)), (0, (3,)), (0, (1,)), (0, (2,))])
    assert t.best() == ((0, (3,)), 1.0)  # earliest of the tied minima
    with pytest.raises(LookupError):
        OracleTuner(sp, cost, valid).best()


def test_random_baseline_exhaustive_when_small():
    sp = Space([[list(range(4)), list(range(4))]])
    tab = [float((i * 7) % 5) for i in range(16)]
    tab[3] = math.inf
    cost, valid = table_cost(sp, tab)
    t = OracleTuner(sp, cost, valid)
    random_baseline(t, k=10000)
    assert len(t.history) == 15
    bp, bc = brute_force(sp, cost, valid)
    assert t.best()[1] == bc
