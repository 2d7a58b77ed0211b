"""ORACLE — TEST INFRASTRUCTURE ONLY.  The multi-layer trial-budget scheduler
(Ansor's task scheduler as the paper describes it).

P:244-248: "an initial round of trials is partitioned among these layers.
Layers are grouped into a worklist, and receive a quota of trials in
round-robin fashion.  After an initial round of optimizations, layers that run
for a very short time are removed from this worklist."
P:393-396: "this initial fraction is min(K/L, 64) ... After an initial round of
optimizations, Ansor applies the remaining trials onto kernels that run for the
longest time."

Reading R-F3 (the constants are not in the paper; SPEC S:418-436 defaults):
  phase 1: every layer explores q = max(1, min(floor(K/L), 64)) trials, in order;
  phase 2: while trials remain and the worklist is non-empty: drop every layer
           whose weight x best cost is < drop_frac (1 %) of the model total
           sum_l weight_l x best_l; give min(increment (16), K - used) more
           exploration trials to the layer with the largest weight x best cost
           (ties: the lowest index); a layer whose exploration yields no new
           point leaves the worklist.
Exploration = OracleTuner.evolve(n, pop, elite) (R-E1), which continues from a
layer's elite once it has measurements.
"""
from __future__ import annotations

import math
from typing import List, Sequence


def initial_quota(K: int, L: int) -> int:
    """min(K/L, 64), floored, at least 1."""
    return max(1, min(K // L, 64))


def schedule(tuners: Sequence, weights: Sequence[float], K: int, increment: int = 16,
             drop_frac: float = 0.01, pop: int = 64, elite: int = 16) -> List[int]:
    L = len(tuners)
    used = [0] * L
    q = initial_quota(K, L)
    total = 0
    for i, t in enumerate(tuners):
        n = min(q, K - total)
        if n <= 0:
            break
        got = len(t.evolve(n, pop, elite))
        used[i] += got
        total += got
    work = list(range(L))

    def wbest(i):
        return weights[i] * tuners[i].best()[1] if tuners[i].history else math.inf

    while total < K and work:
        model = sum(wbest(i) for i in range(L) if math.isfinite(wbest(i)))
        work = [i for i in work if not (math.isfinite(wbest(i)) and wbest(i) < drop_frac * model)]
        if not work:
            break
        pick = work[0]
        for i in work[1:]:
            if wbest(i) > wbest(pick):
                pick = i
        got = len(tuners[pick].evolve(min(increment, K - total), pop, elite))
        if got == 0:
            work.remove(pick)
            continue
        used[pick] += got
        total += got
    return used
