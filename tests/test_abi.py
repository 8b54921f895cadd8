"""CPU-side checks of the C-ABI library (no compute calls; no GPU needed).

* libwv.so loads and exports every function include/wv.h declares, and the
  binding's SIGNATURES cover exactly that set;
* the congruence table the kernels use (read back through the ABI) reproduces
  the paper's printed costs and, evaluated naively here in Python (test code,
  not a product path), gives the oracle's residue for every prime in range.
"""
import os
import re
from fractions import Fraction

import pytest
import sympy

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pkg():
    import __graft_entry__ as g
    g.build()
    import paper_2101_11157_b200 as p
    return p


def _declared():
    src = open(os.path.join(ROOT, "include", "wv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(wv_\w+)\s*\(", src)) - {"wv_hit", "wv_residue"}


def test_library_exports_every_declared_symbol(pkg):
    lib = pkg.lib()
    decl = _declared()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(lib, name), name
    assert set(pkg._wv.SIGNATURES) == decl
    assert "sm_100a" in pkg.version()


def test_host_utilities(pkg):
    # splitmix64 finaliser of p ^ rotl(rw,21) ^ rotl(rv,42) (reading R6)
    def mix(z):
        m = (1 << 64) - 1
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
        return z ^ (z >> 31)

    def rotl(x, r):
        return ((x << r) | (x >> (64 - r))) & ((1 << 64) - 1)

    for p, rw, rv in [(5, 1, 1), (16843, 0, 777), (1062232319, (1 << 64) - 1, 0)]:
        assert pkg.checksum_term(p, rw, rv) == mix(p ^ rotl(rw, 21) ^ rotl(rv, 42))
    # default schedule (include/wv.h)
    names = {c["id"]: c["name"] for c in pkg.congruences()}
    assert names[pkg.schedule(5, pkg.MODE_W)] == "BB1"
    assert names[pkg.schedule(7, pkg.MODE_W)] == "VOR12"
    assert names[pkg.schedule(10 ** 5, pkg.MODE_W)] == "BB30"
    assert names[pkg.schedule(5, pkg.MODE_V)] == "EE3"
    assert names[pkg.schedule(10 ** 5, pkg.MODE_V)] == "EE33"
    assert names[pkg.schedule(10 ** 6, pkg.MODE_W)] == "BG_SML" and names[pkg.schedule(10 ** 6, pkg.MODE_V)] == "EG_SML"
    # generated many-sum congruences (NEXT-2) for large p (BIG from 2^24)
    assert names[pkg.schedule(10 ** 7, pkg.MODE_W)] == "BG_SML" and names[pkg.schedule(10 ** 7, pkg.MODE_V)] == "EG_MID"
    assert names[pkg.schedule(10 ** 9, pkg.MODE_W)] == "BG_XL" and names[pkg.schedule(10 ** 9, pkg.MODE_V)] == "EG_XL"
    assert names[pkg.schedule(5 * 10 ** 10, pkg.MODE_W)] == "BG_BIG"
    assert names[pkg.schedule(5 * 10 ** 10, pkg.MODE_V)] == "EG_BIG"
    with pytest.raises(pkg.WVError):
        pkg.set_schedule_override(99, -1)


# costs printed in the paper: p * sum (y_i - x_i)
PAPER_COSTS = {
    "VOR12": Fraction(1, 12),            # P:L244-250 (cost p/12 like eqnSV)
    "BB1": Fraction(1, 12),
    "BB2": Fraction(1, 15),
    "BB6": Fraction(1, 1) / Fraction(96, 5),   # p/19.2
    "BB9": Fraction(1, 20),
    "BB16": Fraction(1, 24),
    "BB22": Fraction(3, 80),
    "BB30": Fraction(227, 6480),
    "EE3": Fraction(3, 16), "EE5": Fraction(9, 64), "EE9": Fraction(43, 384),   # section 4 costs
    "EE16": Fraction(205, 2304), "EE24": Fraction(115, 1536), "EE33": Fraction(27, 512),
}


def test_congruence_costs_match_paper(pkg):
    table = pkg.congruences()[: len(PAPER_COSTS)]
    assert [c["name"] for c in table] == list(PAPER_COSTS)
    for c in table:
        cost = sum(Fraction(yn, yd) - Fraction(xn, xd) for _, xn, xd, yn, yd in c["terms"])
        assert cost == PAPER_COSTS[c["name"]], c["name"]
        for _, xn, xd, yn, yd in c["terms"]:
            assert Fraction(xn, xd) < Fraction(yn, yd) <= Fraction(1, 2)


def _naive(c, p):
    """L^{-1} * sum_j a_j * sum_{x_j p < s < y_j p} s^{-e} mod p, by direct modular inverses."""
    tot = 0
    for a, xn, xd, yn, yd in c["terms"]:
        x, y = Fraction(xn, xd) * p, Fraction(yn, yd) * p
        s = int(x) + 1
        while s < y:
            tot += a * pow(s, -c["e"], p)
            s += 1
    return tot * pow(c["L"] % p, -1, p) % p


def test_congruence_table_against_oracle(pkg):
    """Each transcribed congruence, evaluated naively, equals the oracle's residue for
    every prime in its validity range below 700 and a few larger seeded primes."""
    import random
    rng = random.Random(11157)
    extra = [int(sympy.nextprime(rng.randrange(2000, 20000))) for _ in range(4)]
    for c in pkg.congruences():
        for p in list(sympy.primerange(max(5, c["min_p"]), 700)) + extra:
            if p == c["excluded_p"]:
                continue
            want = oracle.residue_B(p) if c["e"] == 3 else oracle.residue_E(p)
            assert _naive(c, p) == want, (c["name"], p)


def test_left_factor_vanishes_exactly_where_excluded(pkg):
    """Validity reading R5: L == 0 mod p exactly for the primes the table excludes."""
    for c in pkg.congruences():
        for p in sympy.primerange(5, 50):
            vanishes = c["L"] % p == 0
            valid = p >= c["min_p"] and p != c["excluded_p"]
            if valid:
                assert not vanishes, (c["name"], p)
    names = {c["name"]: c for c in pkg.congruences()}
    assert names["BB1"]["L"] % 7 == 0 and names["VOR12"]["L"] % 5 == 0 and names["EE33"]["L"] % 5 == 0


def test_schedule_tier_boundaries(pkg):
    """The default schedule takes, for each p, the tier with the largest threshold <= p (include/wv.h),
    at every boundary (BG_MID is built but in no default range)."""
    names = {c["id"]: c["name"] for c in pkg.congruences()}
    W, V = pkg.MODE_W, pkg.MODE_V
    want = [(W, 4095, "BB1"), (W, 4096, "BB30"), (W, (1 << 17) - 1, "BB30"), (W, 1 << 17, "BG_SML"),
            (W, (1 << 24) - 1, "BG_SML"), (W, 1 << 24, "BG_XL"), (W, 1 << 29, "BG_XL"), (W, (1 << 30) - 1, "BG_XL"),
            (W, 1 << 30, "BG_BIG"), (W, 1 << 44, "BG_BIG"),
            (V, 4095, "EE3"), (V, 4096, "EE33"), (V, 1 << 17, "EG_SML"), (V, (1 << 21) - 1, "EG_SML"),
            (V, 1 << 21, "EG_MID"), (V, 1 << 24, "EG_XL"), (V, (1 << 30) - 1, "EG_XL"), (V, 1 << 30, "EG_BIG")]
    for test, p, name in want:
        assert names[pkg.schedule(p, test)] == name, (test, p)
