"""The C++ evolutionary explorer (tuner_evolve) reproduces the oracle's
generations bit for bit in cost-table mode, then feeds Droplet identically."""
import random

import pytest

from oracle.search import OracleTuner, Space, table_cost
from paper_2406_20037_b200 import Tuner
from synth import FAMILIES, landscape

LABEL0 = 11


def case(seed):
    rng = random.Random(seed)
    sketches = [[sorted(rng.sample(range(1, 200), rng.randint(1, 7))) for _ in range(rng.randint(1, 5))]
                for _ in range(rng.randint(1, 3))]
    return sketches


@pytest.mark.parametrize("family,seed", [(f, s) for f in FAMILIES for s in range(5)])
def test_evolve_then_droplet_bit_exact(family, seed):
    sk = case(seed * 13 + 7)
    table = landscape([[len(v) for v in s] for s in sk], family, seed, 0.1 if seed % 2 else 0.0)
    n, pop, elite = [10, 40, 120, 300, 64][seed], [8, 16, 32, 64, 5][seed], [2, 4, 8, 16, 1][seed]
    sp = Space(sk)
    cost, valid = table_cost(sp, table)
    o = OracleTuner(sp, cost, valid, seed)
    oev = o.evolve(n, pop, elite, max_batch=17)
    t = Tuner("dense", {"m": 1, "n": 1, "k": 1}, spaces=[(LABEL0 + i, v) for i, v in enumerate(sk)],
              cost_table=table, seed=seed, max_batch=17)
    tev = t.evolve(n, pop, elite)
    assert [(LABEL0 + p[0], p[1], c) for p, c in oev] == [(s.point[0], s.point[1], s.cost_ns) for s in tev]
    if not oev:
        return
    ob = o.best()
    tb = t.best()
    assert (LABEL0 + ob[0][0], ob[0][1], ob[1]) == (tb.point[0], tb.point[1], tb.cost_ns)
    orep = o.droplet(ob[0], 100, "grow")
    trep = t.droplet(tb.point, 100)
    assert [(LABEL0 + p[0], p[1]) for p in orep["traj"]] == trep["traj"]
    assert (orep["trials_used"], orep["rounds"], orep["converged"]) == (trep["trials_used"], trep["rounds"],
                                                                        trep["converged"])
