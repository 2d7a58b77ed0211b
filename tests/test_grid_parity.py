"""Grid search (tuner_grid, the RQ4 exploitation alternative of P:550-563):
oracle pins -- successive calls enumerate every valid point exactly once, in
Space.enumerate() order, skipping measured ones -- and bit-exact parity of the
C++ cursor with the oracle in cost-table mode (several sketches, invalid points,
interleaved with sampling)."""
import math
import random

import pytest

from oracle.search import OracleTuner, Space, table_cost
from paper_2406_20037_b200 import Tuner
from synth import landscape


def case(seed):
    rng = random.Random(seed)
    return [[sorted(rng.sample(range(1, 100), rng.randint(1, 5))) for _ in range(rng.randint(1, 4))]
            for _ in range(rng.randint(1, 3))]


def test_oracle_grid_covers_valid_space_once_in_order():
    sk = case(3)
    sp = Space(sk)
    table = landscape([[len(v) for v in s] for s in sk], "rugged", 3, 0.2)
    cost, valid = table_cost(sp, table)
    o = OracleTuner(sp, cost, valid, 0)
    pre = [p for p, _ in o.sample(5)]
    got = []
    while True:
        chunk = o.grid(7)
        if not chunk:
            break
        got += [p for p, _ in chunk]
    allv = [p for p in sp.enumerate() if valid(p)]
    assert sorted(got + pre, key=sp.linear) == allv               # every valid point exactly once
    assert got == [p for p in allv if p not in set(pre)]          # in enumeration order, measured ones skipped
    assert all(math.isfinite(cost(p)) for p in got)


@pytest.mark.parametrize("seed", range(6))
def test_grid_bit_exact(seed):
    sk = case(seed * 5 + 1)
    table = landscape([[len(v) for v in s] for s in sk], "plateau" if seed % 2 else "rugged", seed, 0.15)
    sp = Space(sk)
    cost, valid = table_cost(sp, table)
    o = OracleTuner(sp, cost, valid, seed)
    t = Tuner("dense", {"m": 1, "n": 1, "k": 1}, spaces=[(20 + i, v) for i, v in enumerate(sk)],
              cost_table=table, seed=seed, max_batch=9)
    steps = [("sample", 4), ("grid", 5), ("grid", 11), ("sample", 3), ("grid", 1000)]
    for what, n in steps:
        a = getattr(o, what)(n)
        b = getattr(t, what)(n)
        assert [(20 + p[0], p[1], c) for p, c in a] == [(s.point[0], s.point[1], s.cost_ns) for s in b]
    assert t.grid(10) == [] and o.grid(10) == []
