"""Multi-layer budget scheduler: pins for the
oracle (the paper's min(K/L, 64) quota examples, single layer, symmetry, the
heavy layer gets more) and bit-exact parity of tuner_schedule in cost-table mode."""
import random

import numpy as np
import pytest

from oracle.schedule import initial_quota, schedule as oschedule
from oracle.search import OracleTuner, Space, table_cost
from paper_2406_20037_b200 import Tuner, schedule
from synth import landscape


def test_initial_quota_examples():
    assert initial_quota(10000, 13) == 64     # AlexNet, 13 layers
    assert initial_quota(10000, 113) == 64    # DenseNet-201, 113 layers: floor(88.5) -> 64
    assert initial_quota(20, 40) == 1         # clamped to at least 1
    assert initial_quota(300, 13) == 23


def layers(seed, L, scale=None):
    rng = random.Random(seed)
    out = []
    for i in range(L):
        sk = [[list(range(rng.randint(3, 7))) for _ in range(rng.randint(2, 4))]]
        tab = landscape([[len(v) for v in sk[0]]], "rugged", seed * 10 + i, 0.05)
        if scale is not None:
            tab = tab * scale[i]
        out.append((sk, tab))
    return out


def oracle_tuners(ls, seed):
    ts = []
    for i, (sk, tab) in enumerate(ls):
        sp = Space(sk)
        c, v = table_cost(sp, tab)
        ts.append(OracleTuner(sp, c, v, seed + i))
    return ts


def product_tuners(ls, seed):
    return [Tuner("dense", {"m": 1, "n": 1, "k": 1}, spaces=[(0, sk[0])], cost_table=tab, seed=seed + i)
            for i, (sk, tab) in enumerate(ls)]


@pytest.mark.parametrize("seed,L,K", [(0, 1, 50), (1, 3, 200), (2, 5, 120), (3, 4, 7), (4, 6, 400)])
def test_schedule_bit_exact(seed, L, K):
    ls = layers(seed, L)
    w = [1.0 + (i % 3) for i in range(L)]
    ot = oracle_tuners(ls, seed)
    pt = product_tuners(ls, seed)
    a = oschedule(ot, w, K, increment=16, drop_frac=0.01, pop=16, elite=4)
    b = schedule(pt, w, K, increment=16, drop_frac=0.01, pop=16, elite=4)
    assert a == b
    assert sum(a) <= K
    for o, p in zip(ot, pt):
        assert [(q[1], c) for q, c in o.history] == [(s.point[1], s.cost_ns) for s in p.history()]


def test_single_layer_gets_the_budget_and_heavy_layer_gets_more():
    sk = [[list(range(8))] * 4]  # 4096 points: room for the whole budget
    ot = oracle_tuners([(sk, landscape([[8] * 4], "rugged", 7, 0.0))], 7)
    assert oschedule(ot, [1.0], 60, pop=8, elite=4) == [60]
    ls3 = layers(8, 3, scale=[10.0, 1.0, 1.0])
    ot3 = oracle_tuners(ls3, 8)
    used = oschedule(ot3, [1.0, 1.0, 1.0], 300, pop=8, elite=4)
    assert used[0] > used[1] and used[0] > used[2]


@pytest.mark.parametrize("c2,w2,expect", [(0.1, 1.0, [4, 4, 30]), (10.0, 1.0, [4, 4, 64]), (0.1, 100.0, [4, 4, 64])])
def test_drop_rule_hand_derived_product(c2, w2, expect):
    # the hand-derived drop cases of tests/test_oracle_pins_r2.py::test_drop_rule_hand_derived
    # through tuner_schedule in cost-table mode
    ts = [Tuner("dense", {"m": 1, "n": 1, "k": 1}, spaces=[(0, [list(range(n))])], cost_table=np.full(n, c),
                seed=n) for n, c in ((4, 100.0), (4, 50.0), (64, c2))]
    assert schedule(ts, [1.0, 1.0, w2], 90, increment=16, drop_frac=0.01, pop=16, elite=4) == expect
