"""Seeded synthetic cost landscapes (cost tables) for cost-table-mode parity.

Families follow SPEC.md's landscape description, used only
as test inputs:
  separable_convex   sum_i w_i (v_i - m_i)^2
  correlated_valley  separable_convex + sum_{i<j} c_ij (v_i - m_i)(v_j - m_j)
  rugged             separable_convex * (1 + 0.35 * seeded per-point noise)
  plateau            separable_convex quantised into steps (many equal costs)
``invalid_fraction`` of the points (never the global optimum) are +inf.
Output: one float64 array per sketch, flattened row-major (last knob fastest),
concatenated in sketch order (DESIGN.md R-T1).
"""
from __future__ import annotations

import numpy as np

FAMILIES = ("separable_convex", "correlated_valley", "rugged", "plateau")


def _one(cards, family, rng, invalid_fraction):
    grids = np.indices(cards).reshape(len(cards), -1).astype(np.float64)
    d = len(cards)
    w = rng.uniform(0.5, 2.0, size=d)
    m = np.array([rng.uniform(0, c - 1) for c in cards])
    dev = grids - m[:, None]
    cost = 1.0 + (w[:, None] * dev ** 2).sum(0)
    if family == "correlated_valley":
        for i in range(d):
            for j in range(i + 1, d):
                cij = rng.uniform(-0.9, 0.9) * np.sqrt(w[i] * w[j])
                cost = cost + cij * dev[i] * dev[j]
        cost = cost - cost.min() + 1.0
    elif family == "rugged":
        cost = cost * (1.0 + 0.35 * rng.uniform(0.0, 1.0, size=cost.size))
    elif family == "plateau":
        cost = np.floor(cost / 2.0) + 1.0
    elif family != "separable_convex":
        raise ValueError(family)
    n_inv = int(np.floor(invalid_fraction * cost.size))
    if n_inv:
        opt = int(np.argmin(cost))
        order = [i for i in rng.permutation(cost.size) if i != opt]
        cost[np.array(order[:n_inv], dtype=np.int64)] = np.inf
    return cost


def landscape(sketch_cards, family: str, seed: int, invalid_fraction: float = 0.0):
    """Cost table for the union of sketches with knob cardinalities ``sketch_cards``."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.concatenate([_one(list(c), family, rng, invalid_fraction) for c in sketch_cards])
