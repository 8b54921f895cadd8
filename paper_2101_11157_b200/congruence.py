"""Congruence derivation and search (section 2).

Host-side planning tool, not on the hot path: it produces new instantiated
congruences  L X == sum_j a_j S(x_j, y_j) (mod p)  for the residue kernels.

Objects are instantiated at the index the search needs:
    W: X = B_{p-3}, S(x,y) = sum_{xp<s<yp} s^{-3}   (l = p-4: d^l == d^-3, (-1)^l = -1)
    V: X = E_{p-3}, S(x,y) = sum_{xp<s<yp} s^{-2}   (l = p-3: d^l == d^-2, (-1)^l = +1)
so every coefficient is a rational number independent of p (Fermat).

Proposition 1 on such sums:
    separation   S(x,z) = S(x,y) + S(y,z)              (yp not an integer)
    reflection   S(x,y) = (-1)^l S(1-y, 1-x)
    subdivision  S(x,y) = d^l sum_{i<d} S((x+i)/d, (y+i)/d)     (p does not divide d)
The right side is kept canonical as a piecewise-constant coefficient function c(z)
on (0, 1/2]: pieces above 1/2 are reflected down, overlapping pieces merge
(separation), zero pieces vanish.  Cost = p * sum of the lengths of the nonzero
pieces.

Seeds (k at the Wolstenholme / Vandiver index):
    eqnSV        21 B == S(1/6, 1/4)                         (C_k(3,4,6) == 21)
    eqnVandiver  14 B == S(1/6, 1/5) + S(1/3, 2/5)            (C_k(2,5,6) == 14)
    eqnE1        -4 E == S(0, 1/4)                           (sign reading R1)
    eqnEMac2    -40 E == S(0, 1/12) - S(5/12, 1/2)            (P:L897-903 at k = 1: -4^0 (9+1) E, 2^-2)

Searches: exhaustive over subdivision sequences (section 2.1) and the
greedy heuristic (section 2.2): repeatedly apply the lambda-step
sequence of subdivisions (d <= D) that minimises the cost.
"""
from __future__ import annotations

import bisect
import math
from dataclasses import dataclass, field
from fractions import Fraction as Fr

HALF = Fr(1, 2)


@dataclass
class Congruence:
    """L * X == sum_j c_j S(x_j, y_j) (mod p) with pieces on (0, 1/2], rational c_j."""
    kind: str                                   # "B" (e = 3) or "E" (e = 2)
    left: Fr
    bps: list = field(default_factory=list)     # breakpoints z_0 < z_1 < ... (Fractions)
    vals: list = field(default_factory=list)    # vals[i] = coefficient on (z_i, z_{i+1})
    min_p: int = 11
    history: list = field(default_factory=list)

    # ------------------------------------------------------------ construction
    @property
    def e(self):
        return 3 if self.kind == "B" else 2

    @property
    def refl_sign(self):
        return -1 if self.kind == "B" else 1

    @classmethod
    def from_terms(cls, kind, left, terms, min_p=11):
        c = cls(kind, Fr(left), [Fr(0), HALF], [Fr(0)], min_p)
        for a, x, y in terms:
            c._add(Fr(x), Fr(y), Fr(a))
        return c

    def copy(self):
        return Congruence(self.kind, self.left, list(self.bps), list(self.vals), self.min_p, list(self.history))

    def _split(self, z):
        """Ensure z is a breakpoint; return its index."""
        i = bisect.bisect_left(self.bps, z)
        if i < len(self.bps) and self.bps[i] == z:
            return i
        self.bps.insert(i, z)
        self.vals.insert(i, self.vals[i - 1])
        return i

    def _add_raw(self, x, y, a):
        """c += a on (x, y), 0 <= x < y <= 1/2."""
        i, j = self._split(x), self._split(y)
        for k in range(i, j):
            self.vals[k] += a

    def _add(self, x, y, a):
        """c += a on (x, y) for 0 <= x < y <= 1, reflecting the part above 1/2 (Prop. 1(b))."""
        if y <= HALF:
            self._add_raw(x, y, a)
        elif x >= HALF:
            self._add_raw(1 - y, 1 - x, a * self.refl_sign)
        else:                                    # separation at 1/2 (p/2 is never an integer)
            self._add_raw(x, HALF, a)
            self._add_raw(1 - y, HALF, a * self.refl_sign)

    def normalize(self):
        """Merge equal neighbours (separation) so pieces are maximal."""
        bps, vals = [self.bps[0]], []
        for k, v in enumerate(self.vals):
            if vals and vals[-1] == v:
                bps[-1] = self.bps[k + 1]
            else:
                vals.append(v)
                bps.append(self.bps[k + 1])
        self.bps, self.vals = bps, vals
        return self

    # ------------------------------------------------------------ queries
    def pieces(self):
        """[(x, y, c)] nonzero maximal pieces."""
        self.normalize()
        return [(self.bps[k], self.bps[k + 1], v) for k, v in enumerate(self.vals) if v != 0]

    def cost(self):
        """Cost / p = sum of lengths of nonzero pieces."""
        return sum((self.bps[k + 1] - self.bps[k] for k, v in enumerate(self.vals) if v != 0), Fr(0))

    def m(self):
        return len(self.pieces())

    # ------------------------------------------------------------ Proposition 1(c)
    def subdivide(self, x, y, d):
        """Replace the term c S(x,y) (a maximal nonzero piece) by c d^-e sum_i S((x+i)/d, (y+i)/d)."""
        k = self.bps.index(x)
        assert self.bps[k + 1] == y
        c = self.vals[k]
        out = self.copy()
        out._add_raw(x, y, -c)
        f = c / Fr(d) ** self.e
        for i in range(d):
            out._add((x + i) / d, (y + i) / d, f)
        out.history.append((d, x, y))
        # denominators of breakpoints gain the prime factors of d: p must not divide them
        out.min_p = max(self.min_p, _max_prime(d) + 1)
        return out.normalize()

    # ------------------------------------------------------------ integer form
    def integer_form(self):
        """(L, [(a, xn, xd, yn, yd)]) with integer L, a_j: the rational form times the lcm of denominators."""
        ps = self.pieces()
        den = self.left.denominator
        for _, _, c in ps:
            den = den * c.denominator // math.gcd(den, c.denominator)
        L = self.left * den
        terms = [(int(c * den), x.numerator, x.denominator, y.numerator, y.denominator) for x, y, c in ps]
        g = abs(int(L))
        for t in terms:
            g = math.gcd(g, abs(t[0]))
        return int(L) // g, [(a // g, xn, xd, yn, yd) for a, xn, xd, yn, yd in terms]

    def residue(self, p):
        """X mod p by direct evaluation (slow; validation only)."""
        L, terms = self.integer_form()
        tot = 0
        for a, xn, xd, yn, yd in terms:
            first = (xn * p) // xd + 1
            last = -((-yn * p) // yd) - 1
            for s in range(first, last + 1):
                tot += a * pow(s, -self.e, p)
        return tot * pow(L % p, -1, p) % p


def _max_prime(d):
    q, best, f = d, 1, 2
    while f * f <= q:
        while q % f == 0:
            best, q = f, q // f
        f += 1
    return max(best, q) if q > 1 else best


# ---------------------------------------------------------------- seeds
def seed(name):
    if name == "SV":            # eqnSV at k = (p-3)/2  (== eqnBB1)
        return Congruence.from_terms("B", 21, [(1, Fr(1, 6), Fr(1, 4))], min_p=11)
    if name == "Vandiver":      # eqnVandiver at k = (p-3)/2
        return Congruence.from_terms("B", 14, [(1, Fr(1, 6), Fr(1, 5)), (1, Fr(1, 3), Fr(2, 5))], min_p=11)
    if name == "E1":            # eqnE1 at k = 1, reading R1
        return Congruence.from_terms("E", -4, [(1, Fr(0), Fr(1, 4))], min_p=7)
    if name == "EMac2":         # eqnEMac2 at k = 1
        return Congruence.from_terms("E", -40, [(1, Fr(0), Fr(1, 12)), (-1, Fr(5, 12), HALF)], min_p=7)
    if name.startswith("table:"):   # a congruence of the library's table (e.g. "table:BB30", eqnBB30)
        from . import _wv
        for c in _wv.congruences():
            if c["name"] == name[6:]:
                return Congruence.from_terms("B" if c["e"] == 3 else "E", c["L"],
                                             [(a, Fr(xn, xd), Fr(yn, yd)) for a, xn, xd, yn, yd in c["terms"]],
                                             min_p=max(11, c["min_p"]))
    raise KeyError(name)


# ---------------------------------------------------------------- searches
def _value(c, z):
    """Coefficient on the elementary interval starting at z (z in [0, 1/2))."""
    k = bisect.bisect_right(c.bps, z) - 1
    return c.vals[k]


def delta_cost(c, k, d):
    """Exact change of cost/p if piece k is subdivided with d, without building the result."""
    x, y, a = c.bps[k], c.bps[k + 1], c.vals[k]
    f = a / Fr(d) ** c.e
    mods = [(x, y, -a)]
    for i in range(d):
        u, v = (x + i) / d, (y + i) / d
        if v <= HALF:
            mods.append((u, v, f))
        elif u >= HALF:
            mods.append((1 - v, 1 - u, f * c.refl_sign))
        else:
            mods.append((u, HALF, f))
            mods.append((1 - v, HALF, f * c.refl_sign))
    pts = set()
    for u, v, _ in mods:
        pts.add(u)
        pts.add(v)
        i, j = bisect.bisect_right(c.bps, u), bisect.bisect_left(c.bps, v)
        pts.update(c.bps[i:j])
    pts = sorted(pts)
    dc = Fr(0)
    for u, v in zip(pts, pts[1:]):
        add = sum((m for lo, hi, m in mods if lo <= u and v <= hi), Fr(0))
        if add == 0:
            continue
        old = _value(c, u)
        new = old + add
        if (new != 0) != (old != 0):
            dc += (v - u) if new != 0 else -(v - u)
    return dc


def best_move(c, D):
    """(delta cost, d, piece index) of the best single subdivision with 2 <= d <= D."""
    c.normalize()
    best = None
    for k, v in enumerate(c.vals):
        if v == 0:
            continue
        for d in range(2, D + 1):
            dc = delta_cost(c, k, d)
            if best is None or dc < best[0]:
                best = (dc, d, k)
    return best


def greedy_fast(c, rounds, D=8, verbose=False, stop_at=None, on_round=None):
    """Section 2.2 heuristic with lambda = 1: apply the best single subdivision while it lowers the cost."""
    cur = c.normalize()
    for r in range(rounds):
        if on_round is not None:
            on_round(r, cur)
        mv = best_move(cur, D)
        if mv is None or mv[0] >= 0:
            break
        dc, d, k = mv
        cur = cur.subdivide(cur.bps[k], cur.bps[k + 1], d)
        if verbose and r % 10 == 0:
            print(f"round {r}: cost p/{float(1 / cur.cost()):.3f}, {cur.m()} sums", flush=True)
        if stop_at is not None and cur.m() >= stop_at:
            break
    return cur


def _moves(c, D):
    for x, y, _ in c.pieces():
        for d in range(2, D + 1):
            yield d, x, y


def greedy(c, rounds, D=8, lam=1, verbose=False):
    """Section 2.2 heuristic: each round applies the lam-step subdivision sequence of least cost."""
    cur = c.normalize()
    for r in range(rounds):
        best = None
        frontier = [cur]
        for _ in range(lam):
            nxt = []
            for g in frontier:
                for d, x, y in _moves(g, D):
                    h = g.subdivide(x, y, d)
                    nxt.append(h)
                    if best is None or h.cost() < best.cost() or (h.cost() == best.cost() and h.m() < best.m()):
                        best = h
            frontier = nxt if lam > 1 else []
        if best is None or best.cost() >= cur.cost():
            break
        cur = best
        if verbose:
            print(f"round {r}: cost {cur.cost()} = p/{float(1 / cur.cost()):.3f}, {cur.m()} sums", flush=True)
    return cur


def replay(c, steps):
    """Apply a recorded list of (d, x, y) subdivisions."""
    for d, x, y in steps:
        c = c.subdivide(Fr(x), Fr(y), d)
    return c
