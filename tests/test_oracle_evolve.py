"""Pins for the oracle's evolutionary explorer (reading R-E1):
structural invariants that a dropped step, a wrong index or a swapped operand
would break, plus its determinism and its relation to the plain sampler."""
import math
import random

from oracle.search import OracleTuner, Space, table_cost
from synth import landscape


def make(seed, fam="rugged"):
    rng = random.Random(seed)
    sketches = [[list(range(rng.randint(2, 6))) for _ in range(rng.randint(2, 5))] for _ in range(rng.randint(1, 3))]
    cards = [[len(v) for v in s] for s in sketches]
    table = landscape(cards, fam, seed, 0.1)
    sp = Space(sketches)
    return sp, table


def test_generation0_is_the_sampler():
    sp, table = make(1)
    cost, valid = table_cost(sp, table)
    a = OracleTuner(sp, cost, valid, seed=9)
    b = OracleTuner(sp, cost, valid, seed=9)
    ev = a.evolve(40, pop=16, elite=4)
    dr = b.draw(16)
    assert [p for p, _ in ev[:16]] == dr


def test_children_come_from_elite_parents_with_one_mutation():
    for seed in range(20):
        sp, table = make(seed)
        cost, valid = table_cost(sp, table)
        t = OracleTuner(sp, cost, valid, seed=seed)
        pop, elite = 12, 5
        res = t.evolve(100, pop=pop, elite=elite, max_batch=7)
        pts = [p for p, _ in res]
        assert len(pts) == len(set(pts)) <= 100
        assert all(valid(p) for p in pts)
        # each generation's parents are the elite of everything measured before it, and
        # each child agrees with two of those parents on all but <= 1 knob
        hist = pts[:min(pop, 100)]
        assert sum(len(ch) for _, ch in t.generations) + len(hist) == len(pts)
        for parents_rec, gen in t.generations:
            ranked = sorted(((cost(p), k, p) for k, p in enumerate(hist) if math.isfinite(cost(p))))
            parents = [p for _, _, p in ranked[:elite]]
            assert parents == parents_rec
            for c in gen:
                ok = False
                for a in parents:
                    for b in parents:
                        if a[0] != c[0] or b[0] != c[0]:
                            continue
                        diff = sum(1 for d in range(len(c[1])) if c[1][d] not in (a[1][d], b[1][d]))
                        ok |= diff <= 1
                assert ok, (c, parents)
            hist += gen


def test_evolution_beats_its_first_generation_on_convex_tables():
    wins = 0
    for seed in range(30):
        sp, table = make(seed, "separable_convex")
        cost, valid = table_cost(sp, table)
        t = OracleTuner(sp, cost, valid, seed=seed)
        res = t.evolve(120, pop=20, elite=5)
        g0 = min(c for _, c in res[:20])
        best = min(c for _, c in res)
        assert best <= g0
        wins += best < g0
    assert wins >= 15


def test_evolve_exhausts_small_spaces_gracefully():
    sp = Space([[[1, 2], [1, 2, 3]]])
    cost, valid = table_cost(sp, [1.0, 2.0, 3.0, 4.0, 5.0, 6.0])
    t = OracleTuner(sp, cost, valid, seed=0)
    res = t.evolve(100, pop=4, elite=2)
    assert len(res) == len({p for p, _ in res}) <= 6
    assert t.best()[1] == 1.0
