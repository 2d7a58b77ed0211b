"""ORACLE — TEST INFRASTRUCTURE ONLY.  The Wilcoxon rank-sum test ("the
p-value (produced via the non-parametric Wilcoxon rank-sum test) for the
difference between the two populations"; neighbours "similar with a
confidence level of 95%" stop the descent).

Reading R-W1: two-sided exact test on midranks.  W = sum of the (mid)ranks of
sample a in the pooled sample; under H0 every choice of len(a) positions among
the pooled ranks is equally likely; p = min(1, 2 * min(P(W' <= W), P(W' >= W))).
Written as the plain enumeration of all C(n, n1) subsets.
"""
from __future__ import annotations

from itertools import combinations
from typing import Sequence


def midranks(values: Sequence[float]):
    """Ranks 1..n of the values, ties sharing the mean of their positions (x2: integers)."""
    order = sorted(range(len(values)), key=lambda i: values[i])
    r2 = [0] * len(values)
    i = 0
    while i < len(order):
        j = i
        while j + 1 < len(order) and values[order[j + 1]] == values[order[i]]:
            j += 1
        for k in range(i, j + 1):
            r2[order[k]] = (i + 1) + (j + 1)  # twice the mean rank of positions i+1..j+1
        i = j + 1
    return r2


def wilcoxon_p(a: Sequence[float], b: Sequence[float]) -> float:
    n1, n2 = len(a), len(b)
    if n1 == 0 or n2 == 0:
        return 1.0
    r2 = midranks(list(a) + list(b))
    w = sum(r2[:n1])
    le = ge = total = 0
    for sub in combinations(range(n1 + n2), n1):
        s = sum(r2[i] for i in sub)
        total += 1
        le += s <= w
        ge += s >= w
    return min(1.0, 2.0 * min(le, ge) / total)
