"""Round-2 pins for the oracle parts VERDICT r1 found unpinned or weakly pinned
(each checked against a value written out by hand, a published vector or a closed
form -- never against the oracle's own code):

* the sampler's rejection path ("rejected draws still consume PRNG
  output"; R-S1) -- hand-traced over the published SplitMix64 outputs, and the state
  after the 64·n attempt cap in closed form;
* the alpha gate of Droplet (P:410 Wilcoxon rank-sum; "considered similar with a
  confidence level of 95%, then the coordinate descent procedure stops"; SPEC S:222-229
  worked example {1,2,3} vs {4,5,6});
* the phase-2 drop rule of the multi-layer scheduler ("layers that run for a
  very short time are removed from this worklist"; R-F3) -- hand-derived trial splits;
* SURVEY §8(c)'s closed-form trial and round counts for sum (v_i - 3)^2 on {0..9}^4.

Each docstring states the hand derivation.  tests/test_pin_mutants.py re-runs the pins against deliberately broken oracle variants to show they bite.
"""
import json
import math
import os

import pytest

from oracle.schedule import schedule as oschedule
from oracle.search import OracleTuner, Space, table_cost

GOLD = os.path.join(os.path.dirname(__file__), "golden")
GAMMA = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


def splitmix_outputs():
    with open(os.path.join(GOLD, "splitmix64.json")) as f:
        g = json.load(f)
    return [int(h, 16) for h in g["outputs_hex"]]


# ---------------------------------------------------------------- sampler rejection path
def test_published_outputs_as_fractions():
    # the hand trace below reads each published output z as the fraction z / 2^64
    z = splitmix_outputs()
    frac = [v / 2.0 ** 64 for v in z]
    assert [round(f, 4) for f in frac] == [0.8833, 0.4315, 0.0264, 0.9709, 0.1063, 0.3273, 0.1739, 0.7715]


def sampler_space():
    # sketch 0: one knob of 2 values (both valid); sketch 1: one knob of 3 values, index 1 invalid
    sp = Space([[[10, 20]], [[1, 2, 3]]])
    tab = [1.0, 2.0, 3.0, math.inf, 5.0]  # linear ids: (0,0) (0,1) | (1,0) (1,1) (1,2)
    return sp, tab


def test_sampler_hand_traced_with_rejected_draw():
    """seed 0.  A draw consumes uniform(2) for the sketch, then uniform(card) for the knob
    (uniform(m) = floor(m * z / 2^64)).  Published outputs as fractions:
      draw 1: #1 .8833 -> sketch 1; #2 .4315 -> floor(3 x .4315) = 1 -> (1,(1,)) INVALID, rejected
      draw 2: #3 .0264 -> sketch 0; #4 .9709 -> floor(2 x .9709) = 1 -> (0,(1,)) accepted
      draw 3: #5 .1063 -> sketch 0; #6 .3273 -> floor(2 x .3273) = 0 -> (0,(0,)) accepted
    so draw(2) = [(0,(1,)), (0,(0,))] after 3 attempts = 6 outputs: state = 6 x gamma (seed 0).
    A sampler that re-draws only the knob after a rejection, or does not consume output for a
    rejected draw, returns a different list."""
    sp, tab = sampler_space()
    cost, valid = table_cost(sp, tab)
    t = OracleTuner(sp, cost, valid, seed=0)
    assert t.draw(2) == [(0, (1,)), (0, (0,))]
    assert t.rng.state == (6 * GAMMA) & M64


def test_sampler_duplicates_consume_output_until_the_cap():
    """Every valid point already measured: draw(n) makes exactly 64 n attempts (R-S1) and
    each rejected attempt consumes one output for the sketch and one per knob, so the
    state advances by 64 n x (1 + nknobs) outputs: closed form (64 n (1 + nknobs)) x gamma."""
    sp = Space([[[1, 2], [1, 2, 3]]])
    t = OracleTuner(sp, lambda p: 1.0, lambda p: True, seed=0)
    t.measure(sp.enumerate())
    s0 = t.rng.state
    assert s0 == 0
    assert t.draw(3) == []
    assert t.rng.state == (64 * 3 * 3 * GAMMA) & M64


# ---------------------------------------------------------------- alpha gate
def gate_tuner(samples_start, samples_nb):
    # a 2-point line: start (0,) and its only neighbour (1,); costs = mean of the samples
    sp = Space([[[0, 1]]])
    smp = {(0, (0,)): samples_start, (0, (1,)): samples_nb}
    cost = lambda p: sum(smp[p]) / len(smp[p])
    return OracleTuner(sp, cost, lambda p: True, samples=lambda p: smp[p])


@pytest.mark.parametrize("alpha,moves", [(0.0, True), (0.05, False), (0.1, False), (0.15, True)])
def test_alpha_gate_spec_worked_example(alpha, moves):
    """timings {1,2,3} vs {4,5,6}: two-sided exact p = 2/20 = 0.1 (one extreme
    assignment of C(6,3) = 20 each side).  "tie when p >= alpha": alpha = 0.05 -> no move
    (converged at the start); alpha = 0.1 -> p < alpha is false -> no move; alpha = 0.15 ->
    move; alpha = 0 -> the strict cost compare alone (R-D4) -> move."""
    t = gate_tuner([4.0, 5.0, 6.0], [1.0, 2.0, 3.0])
    rep = t.droplet((0, (0,)), 100, "plain", alpha=alpha)
    assert rep["best"] == ((0, (1,)) if moves else (0, (0,)))
    assert rep["converged"]
    assert rep["trials_used"] == 2  # the start + its one neighbour, whatever the gate decides


def test_alpha_gate_needs_lower_cost_too():
    """A significant difference in the wrong direction never moves: {4,5,6} for the
    neighbour vs {1,2,3} for the start, p = 0.1 < 0.15 but the neighbour is slower."""
    t = gate_tuner([1.0, 2.0, 3.0], [4.0, 5.0, 6.0])
    rep = t.droplet((0, (0,)), 100, "plain", alpha=0.15)
    assert rep["best"] == (0, (0,))


# ---------------------------------------------------------------- scheduler drop rule
def const_layer(nvals, c):
    # one knob, every point costs c: the layer's best is c whatever exploration picks
    sp = Space([[list(range(nvals))]])
    return OracleTuner(sp, lambda p: c, lambda p: True, seed=nvals)


@pytest.mark.parametrize("c2,w2,expect", [
    (0.1, 1.0, [4, 4, 30]),    # 0.1 < 1 % of 150.1: layer 2 dropped before phase 2
    (10.0, 1.0, [4, 4, 64]),   # 10 >= 1 % of 160: kept, takes the rest of its space
    (0.1, 100.0, [4, 4, 64]),  # weight x best = 10: kept (the rule weighs by occurrence)
])
def test_drop_rule_hand_derived(c2, w2, expect):
    """K = 90, L = 3: phase-1 quota min(floor(90/3), 64) = 30.  Layers 0 and 1 have
    4 points each (costs 100 and 50): exploration exhausts them at 4 trials.  Layer 2 has 64
    points of cost c2: it takes its full 30.  used = 38 < 90 -> phase 2.
      drop: model = 1x100 + 1x50 + w2 x c2; layer 2 is removed iff w2 x c2 < 0.01 x model.
      case (0.1, 1): 0.1 < 1.501 -> removed.  Layer 0 (largest, 100) yields no new point ->
        leaves the worklist; then layer 1 likewise -> worklist empty: [4, 4, 30].
      case (10, 1): 10 >= 1.6 -> kept; layers 0, 1 leave as above; layer 2 gets 16 + 16 + 2
        (its 64 points run out) -> [4, 4, 64].
      case (0.1, 100): weight x best = 10 >= 1.6 -> kept -> [4, 4, 64]."""
    ts = [const_layer(4, 100.0), const_layer(4, 50.0), const_layer(64, c2)]
    used = oschedule(ts, [1.0, 1.0, w2], 90, increment=16, drop_frac=0.01, pop=16, elite=4)
    assert used == expect
    assert [len(t.history) for t in ts] == expect


# ---------------------------------------------------------------- closed-form counts
def convex4():
    sp = Space([[list(range(10))] * 4])
    return sp, (lambda p: float(sum((v - 3) ** 2 for v in p[1])))


def test_plain_closed_form_counts():
    """sum (v_i - 3)^2 on {0..9}^4 from the origin.  One +1 step on a coordinate at v lowers
    the cost by (v-3)^2 - (v-2)^2 = 5, 3, 1 for v = 0, 1, 2, so steepest descent with
    first-in-ring-order ties raises every coordinate to 1, then to 2, then to 3: 12 moves,
    plus the final ring that holds no improvement = 13 rounds.  SURVEY §8(c) counts 71
    neighbour measurements (+ 1 for the unmeasured start = 72 trials)."""
    sp, cost = convex4()
    t = OracleTuner(sp, cost, lambda p: True)
    rep = t.droplet((0, (0, 0, 0, 0)), 10 ** 6, "plain")
    assert rep["rounds"] == 13 and rep["trials_used"] == 71 + 1 and rep["converged"]
    assert len(rep["traj"]) == 13
    assert [p[1] for p in rep["traj"][:5]] == [(0, 0, 0, 0), (1, 0, 0, 0), (1, 1, 0, 0), (1, 1, 1, 0), (1, 1, 1, 1)]


def test_grow_closed_form_counts():
    """GROW (R-D9) on the same table.  Per coordinate d (in order): a ring move 0 -> 1 (round),
    then the ray from 0 along +: 2, 4, 8, 9 (round): 2 is strictly better (cost 1 < 4), 4 is
    not (1 = 1) -> stop at 2.  4 coordinates x 2 = 8 rounds to (2,2,2,2).  Then per coordinate
    a ring move 2 -> 3 (round) and the ray 4, 6, 9 (round), none better: 8 more rounds.  The
    final ring: 1 round.  17 rounds; SURVEY §8(c) counts 75 neighbour measurements (+ 1)."""
    sp, cost = convex4()
    t = OracleTuner(sp, cost, lambda p: True)
    rep = t.droplet((0, (0, 0, 0, 0)), 10 ** 6, "grow")
    assert rep["rounds"] == 17 and rep["trials_used"] == 75 + 1 and rep["converged"]
    assert [p[1] for p in rep["traj"][:3]] == [(0, 0, 0, 0), (1, 0, 0, 0), (2, 0, 0, 0)]
    assert rep["best"] == (0, (3, 3, 3, 3))


def test_best_of_sketch_by_hand():
    """R-D17 start points: history (measurement order) = (1,(0,)) 5, (0,(1,)) 3, (1,(2,)) 2, (0,(0,)) 3,
    (1,(1,)) 2, (0,(2,)) inf: sketch 0 -> (0,(1,)) (first of the tied 3s), sketch 1 -> (1,(2,)) (first of
    the tied 2s), a sketch with no finite cost -> None."""
    sp = Space([[[0, 1, 2]], [[0, 1, 2]], [[0]]])
    cost = {(1, (0,)): 5.0, (0, (1,)): 3.0, (1, (2,)): 2.0, (0, (0,)): 3.0, (1, (1,)): 2.0, (0, (2,)): math.inf,
            (2, (0,)): math.inf}
    t = OracleTuner(sp, lambda p: cost[p], lambda p: True)
    t.measure([(1, (0,)), (0, (1,)), (1, (2,)), (0, (0,)), (1, (1,)), (0, (2,)), (2, (0,))])
    assert t.best_of_sketch(0) == ((0, (1,)), 3.0)
    assert t.best_of_sketch(1) == ((1, (2,)), 2.0)
    assert t.best_of_sketch(2) is None
