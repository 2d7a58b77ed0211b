"""ORACLE — TEST INFRASTRUCTURE ONLY.  The search side of the method, step by step.

Follows PAPER.md in the paper's order and notation; where the paper is silent
the reading taken is named (R-xx = DESIGN.md §3 readings table, which mirrors
SURVEY.md §8(c)).  Plain Python, no cleverness: lists, dicts, loops.

Space (Def. 2.1; Example 2.3)
    A sketch's search space has one dimension per annotation parameter; a point
    ("coordinate") is an index vector into each parameter's ordered value list.
    Points are (sketch_position, idx_tuple).  Linear ids are mixed-radix,
    row-major, last knob fastest; sketches are concatenated in order (R-T1).
Neighbourhood
    "the neighbors of (unrolling=3, tiling=8) would be (2,8), (4,8), (3,4) and
    (3,16)": one index step along one coordinate, no diagonals (R-D5, R-D7),
    out-of-range indices skipped, no wrap (R-D6); order dimension-major, minus
    before plus (R-D3).
Sampler (R-S1; Fig. 6's distributions are lost)
    SplitMix64, uniform(m) = (z*m) >> 64; per draw the sketch then each knob
    index uniformly; reject invalid or already-visited draws; stop at n accepted
    or 64*n attempts.
Droplet Search — see ``droplet``.
Best-of-N ("Give the best schedule found with N trials"): first argmin
    over history in measurement order (R-B1).
"""
from __future__ import annotations

import math
from typing import Callable, Dict, List, Optional, Sequence, Tuple

from .stats import wilcoxon_p

Point = Tuple[int, Tuple[int, ...]]

MASK64 = (1 << 64) - 1


# ----------------------------------------------------------------------------- PRNG
class SplitMix64:
    """Vigna's SplitMix64 (public-domain reference algorithm), state = seed."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self, m: int) -> int:
        """An integer in [0, m): the high 64 bits of the 128-bit product z*m."""
        return (self.next() * m) >> 64


# ----------------------------------------------------------------------------- space
class Space:
    """Union of sketch spaces.  ``sketches[s]`` = list of value lists, one per knob."""

    def __init__(self, sketches: Sequence[Sequence[Sequence[int]]]):
        self.sketches = [[list(v) for v in knobs] for knobs in sketches]
        for knobs in self.sketches:
            for vals in knobs:
                assert len(vals) >= 1 and all(a < b for a, b in zip(vals, vals[1:])), \
                    "values must be non-empty and strictly increasing"
        self.offsets = []
        off = 0
        for s in range(len(self.sketches)):
            self.offsets.append(off)
            off += self.size(s)
        self.total = off

    @property
    def nsketch(self) -> int:
        return len(self.sketches)

    def cards(self, s: int) -> List[int]:
        return [len(v) for v in self.sketches[s]]

    def size(self, s: int) -> int:
        """Product of the knob cardinalities (Example 2.3: 5 x 5 = 25)."""
        n = 1
        for c in self.cards(s):
            n *= c
        return n

    def values(self, p: Point) -> List[int]:
        s, idx = p
        return [self.sketches[s][d][i] for d, i in enumerate(idx)]

    def linear(self, p: Point) -> int:
        s, idx = p
        lin = 0
        for d, c in enumerate(self.cards(s)):
            lin = lin * c + idx[d]
        return self.offsets[s] + lin

    def point(self, gid: int) -> Point:
        s = max(i for i in range(self.nsketch) if self.offsets[i] <= gid)
        lin = gid - self.offsets[s]
        idx = []
        for c in reversed(self.cards(s)):
            idx.append(lin % c)
            lin //= c
        return (s, tuple(reversed(idx)))

    def enumerate(self) -> List[Point]:
        """Every point once: sketches in order, each row-major (last knob fastest)."""
        return [self.point(g) for g in range(self.total)]

    def ring(self, p: Point, r: int = 1) -> List[Point]:
        """The neighbourhood of P:292-294: +-1 index along each coordinate.  With r > 1 the
        axis-aligned ring at index distance r (the expanding-radius reading, R-D16)."""
        s, idx = p
        cards = self.cards(s)
        out = []
        for d in range(len(idx)):
            for delta in (-r, +r):
                i = idx[d] + delta
                if 0 <= i < cards[d]:
                    out.append((s, idx[:d] + (i,) + idx[d + 1:]))
        return out


# ----------------------------------------------------------------------------- tuner state
class OracleTuner:
    """History + memo + sampler state for one layer, measured through ``cost``.

    ``cost(p)`` returns the cost of an executed point (+inf for a runtime failure);
    ``valid(p)`` is the static validity predicate: invalid points are never
    executed and never count as trials (R-T2; "each trial consists of the
    observation of the execution of an actual schedule").
    """

    def __init__(self, space: Space, cost: Callable[[Point], float],
                 valid: Callable[[Point], bool], seed: int = 0,
                 samples: Optional[Callable[[Point], List[float]]] = None):
        self.space = space
        self._cost = cost
        self.valid = valid
        self.rng = SplitMix64(seed)
        self.history: List[Tuple[Point, float]] = []
        self.memo: Dict[Point, float] = {}
        self._samples = samples                      # per-point repeat timings (statistical mode)
        self.smemo: Dict[Point, List[float]] = {}
        self.batches: List[List[Point]] = []
        self.generations: List[Tuple[List[Point], List[Point]]] = []  # evolve(): (parents, children)

    # one measured batch, in batch order (sharding changes nothing, R-M1)
    def measure(self, batch: List[Point]) -> None:
        self.batches.append(list(batch))
        for p in batch:
            c = self._cost(p)
            self.memo[p] = c
            if self._samples is not None:
                self.smemo[p] = list(self._samples(p))
            self.history.append((p, c))

    # Ansor-style proposal (R-S1)
    def draw(self, n: int) -> List[Point]:
        out: List[Point] = []
        taken = set(self.memo)
        attempts = 0
        while len(out) < n and attempts < 64 * n:
            attempts += 1
            s = self.rng.uniform(self.space.nsketch)
            idx = tuple(self.rng.uniform(c) for c in self.space.cards(s))
            p = (s, idx)
            if not self.valid(p) or p in taken:
                continue
            taken.add(p)
            out.append(p)
        return out

    def sample(self, n: int, max_batch: int = 512) -> List[Tuple[Point, float]]:
        pts = self.draw(n)
        for i in range(0, len(pts), max_batch):
            self.measure(pts[i:i + max_batch])
        return [(p, self.memo[p]) for p in pts]

    # ------------------------------------------------------------------ grid search (RQ4)
    def grid(self, n: int, max_batch: int = 512) -> List[Tuple[Point, float]]:
        """AutoTVM's grid search as an exploitation alternative (RQ4): the next n
        valid, unmeasured points of ``Space.enumerate()`` order, from a cursor kept across calls."""
        cur = getattr(self, "_grid_cursor", 0)
        pts: List[Point] = []
        while len(pts) < n and cur < self.space.total:
            p = self.space.point(cur)
            cur += 1
            if p in self.memo or not self.valid(p):
                continue
            pts.append(p)
        self._grid_cursor = cur
        for i in range(0, len(pts), max_batch):
            self.measure(pts[i:i + max_batch])
        return [(p, self.memo[p]) for p in pts]

    # ------------------------------------------------------------------ evolutionary exploration
    def evolve(self, n: int, pop: int = 64, elite: int = 16, max_batch: int = 512) -> List[Tuple[Point, float]]:
        """Ansor-style evolution of the annotated population (R-E1), without
        the learned cost model: every child is measured.

        Generation 0 is ``draw(min(pop, n))`` (the sampler, R-S1) -- only on a tuner with no
        finite measurement yet; otherwise the call continues from its elite.  Each later generation
        takes the ``elite`` best measured points of the whole history (cost, then
        measurement order; finite costs only) as parents and produces up to
        min(pop, n - used) new children, each:
          a = parents[uniform(E)]; op = uniform(2)
          op == 1: b = parents[uniform(E)]; if b is of a's sketch, for every knob d
                   child[d] = (a[d], b[d])[uniform(2)], else child = a
          op == 0: child = a
          mutation: d = uniform(nknobs); child[d] = uniform(card_d)
        A child is kept iff valid, unmeasured and new in this generation; at most 64*pop
        attempts per generation; an empty generation ends the run.
        """
        out: List[Point] = []
        first: List[Point] = []
        if not any(math.isfinite(c) for _, c in self.history):  # a fresh tuner: generation 0
            first = self.draw(min(pop, n))                          # (else: continue from the elite)
            for i in range(0, len(first), max_batch):
                self.measure(first[i:i + max_batch])
        out += first
        used = len(first)
        while used < n:
            ranked = sorted(((c, k, p) for k, (p, c) in enumerate(self.history) if math.isfinite(c)))
            parents = [p for _, _, p in ranked[:elite]]
            if not parents:
                break
            want = min(pop, n - used)
            children: List[Point] = []
            taken = set()
            attempts = 0
            while len(children) < want and attempts < 64 * pop:
                attempts += 1
                a = parents[self.rng.uniform(len(parents))]
                child = list(a[1])
                if self.rng.uniform(2) == 1:
                    b = parents[self.rng.uniform(len(parents))]
                    if b[0] == a[0]:
                        for d in range(len(child)):
                            if self.rng.uniform(2) == 1:
                                child[d] = b[1][d]
                cards = self.space.cards(a[0])
                if cards:
                    d = self.rng.uniform(len(cards))
                    child[d] = self.rng.uniform(cards[d])
                c = (a[0], tuple(child))
                if not self.valid(c) or c in self.memo or c in taken:
                    continue
                taken.add(c)
                children.append(c)
            if not children:
                break
            self.generations.append((list(parents), list(children)))
            for i in range(0, len(children), max_batch):
                self.measure(children[i:i + max_batch])
            out += children
            used += len(children)
        return [(p, self.memo[p]) for p in out]

    def best(self) -> Tuple[Point, float]:
        """First argmin of cost over history, in measurement order (R-B1)."""
        if not self.history:
            raise LookupError("best() before any measurement")
        bp, bc = self.history[0]
        for p, c in self.history[1:]:
            if c < bc:
                bp, bc = p, c
        return bp, bc

    def best_of_sketch(self, s: int) -> Optional[Tuple[Point, float]]:
        """First argmin over the history points of sketch s with a finite cost (R-B1 restricted to
        one sketch: the start of that sketch's Droplet run, R-D17); None if there is none."""
        found = None
        for p, c in self.history:
            if p[0] == s and math.isfinite(c) and (found is None or c < found[1]):
                found = (p, c)
        return found

    # ------------------------------------------------------------------ Droplet Search
    def droplet(self, start: Point, budget: int = 100, policy: str = "plain", alpha: float = 0.0) -> dict:
        """Droplet Search, PAPER.md P:297-304:

          1. "At iteration zero, let the best current candidate be" the start.
          2. "Let (c_1..c_n) be the best set of parameters discovered up to
             iteration i.
             (a) If there exists c_i' ... such that (c_1..c_i'..c_n) yields a
                 faster kernel ..., then update the current best candidate to
                 use c_i' instead of c_i.
             (b) If there is no such c_i', then the search terminates."

        Readings: the whole neighbourhood is measured as one batch and the best
        improving neighbour is taken (R-D2), first in ring order on ties (R-D3),
        only strictly faster moves (R-D4); at most ``budget`` new measurements,
        counting the start iff it was unmeasured (R-D14, P:474 cap 100); a
        truncated batch keeps its prefix in ring order and ends the search
        unconverged (R-D13).  policy "grow" (R-D9, north_star "grows its step")
        after each ring move along u also probes x_prev + 2^j u (j = 1, 2, ...,
        clamped, until the clamp repeats) as one batch and accepts its points
        in order while each is strictly better than the incumbent.  policy "radius" (R-D16,
        the original Droplet's speculation that P:276-277 says was removed): when the ring
        holds no improving point, the axis-aligned ring at index distance r = 2, 3, ... is
        measured instead (one batch and one round each) until a strictly better point is
        found -- the search moves there and r returns to 1 -- or no ring point is in range
        any more (converged: x is optimal along every axis line of its sketch).
        """
        if budget < 1:
            raise ValueError("budget must be >= 1")
        if not self.valid(start):
            raise ValueError("start is statically invalid")
        used = 0
        if start not in self.memo:
            self.measure([start])
            used += 1
        x = start
        c = self.memo[x]
        traj = [x]
        rounds = 0

        def better(p: Point, q: Point) -> bool:
            """p yields a faster kernel than q: strictly lower cost (R-D4) and, with
            alpha > 0, a significant difference (Wilcoxon rank-sum p < alpha, R-W1)."""
            if not (self.memo[p] < self.memo[q]):
                return False
            return alpha <= 0 or wilcoxon_p(self.smemo[p], self.smemo[q]) < alpha

        def new_batch(cands: List[Point]) -> Tuple[List[Point], bool]:
            q = [p for p in cands if p not in self.memo and self.valid(p)]
            room = budget - used
            return q[:room], len(q) > room

        r = 1
        while True:
            ring = self.space.ring(x, r)
            if r > 1 and not ring:  # R-D16: every axis line of x has been examined
                return self._report(x, c, used, rounds, True, traj)
            q, trunc = new_batch(ring)
            if q:
                self.measure(q)
            used += len(q)
            rounds += 1
            best_p, best_c = None, None
            for p in ring:
                if p in self.memo and self.valid(p):
                    if best_p is None or self.memo[p] < best_c:
                        best_p, best_c = p, self.memo[p]
            if best_p is None or not better(best_p, x):
                if policy == "radius" and not trunc:
                    r += 1
                    continue
                return self._report(x, c, used, rounds, not trunc, traj)
            r = 1
            prev = x
            x, c = best_p, best_c
            traj.append(x)
            if used == budget:
                return self._report(x, c, used, rounds, False, traj)
            if policy == "grow":
                d = next(i for i in range(len(x[1])) if x[1][i] != prev[1][i])
                step = x[1][d] - prev[1][d]          # +1 or -1
                card = self.space.cards(x[0])[d]
                ray: List[Point] = []
                last = x
                j = 1
                while True:
                    i = min(max(prev[1][d] + step * (2 ** j), 0), card - 1)
                    qj = (x[0], x[1][:d] + (i,) + x[1][d + 1:])
                    if qj == last:
                        break
                    ray.append(qj)
                    last = qj
                    j += 1
                q, trunc = new_batch(ray)
                if q:
                    self.measure(q)
                used += len(q)
                rounds += 1
                for p in ray:
                    if p in self.memo and self.valid(p) and better(p, x):
                        x, c = p, self.memo[p]
                        traj.append(x)
                    else:
                        break
                if trunc:
                    return self._report(x, c, used, rounds, False, traj)

    @staticmethod
    def _report(x, c, used, rounds, converged, traj) -> dict:
        return {"best": x, "best_cost": c, "trials_used": used, "rounds": rounds,
                "converged": bool(converged), "traj": list(traj)}


# ----------------------------------------------------------------------------- helpers
def table_cost(space: Space, table: Sequence[float]):
    """Cost-table mode (R-T1): cost(p) = table[linear(p)], valid <=> finite."""
    def cost(p: Point) -> float:
        return float(table[space.linear(p)])

    def valid(p: Point) -> bool:
        return math.isfinite(float(table[space.linear(p)]))
    return cost, valid


def brute_force(space: Space, cost, valid) -> Tuple[Optional[Point], float]:
    """Exhaustive grid search: first argmin over enumerate order."""
    bp, bc = None, math.inf
    for p in space.enumerate():
        if valid(p):
            c = cost(p)
            if bp is None or c < bc:
                bp, bc = p, c
    return bp, bc


def is_local_min(space: Space, p: Point, cost, valid) -> bool:
    """No valid ring point is strictly cheaper (the paper's neighbourhood)."""
    c = cost(p)
    return all(not (cost(q) < c) for q in space.ring(p) if valid(q))


def random_baseline(tuner: OracleTuner, k: int = 10000, max_batch: int = 512):
    """AutoTVM random search without replacement (R-B2): k sampled
    points, or exhaustive enumeration when the valid space holds <= k points."""
    valid_pts = [p for p in tuner.space.enumerate() if tuner.valid(p) and p not in tuner.memo]
    if len(valid_pts) <= k:
        for i in range(0, len(valid_pts), max_batch):
            tuner.measure(valid_pts[i:i + max_batch])
        return
    tuner.sample(k, max_batch)
