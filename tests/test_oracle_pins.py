"""Pins for the CPU oracle (oracle/), independent of the oracle's own code.

Every oracle tier is checked against something other than itself:
exact rationals from sympy / an independent integer algorithm, values and
lists the paper prints (tests/golden/, each with its citation), textbook
prime counts, and cross-tier agreement between formulas that share no
arithmetic.  None of these tests touch the GPU path.
"""
import csv
import json
import os
import random

import pytest
import sympy

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _primes(lo, hi):
    return list(sympy.primerange(lo, hi))


def _modq(fr, p):
    """Rational -> residue mod p (denominator invertible)."""
    num, den = sympy.fraction(sympy.Rational(fr))
    return int(num) * pow(int(den), -1, p) % p


def _secant_numbers(nmax):
    """E_0, E_2, ..., E_{2 nmax} of sec z, by Seidel's boustrophedon
    (Entringer triangle) -- integer additions only, an algorithm unrelated to
    the oracle's sec*cos recurrence.  sec z has all-positive even coefficients
    (the zigzag numbers), so E_2 = 1, E_4 = 5, E_10 = 50521."""
    zig = [1]
    row = [1]
    for n in range(1, 2 * nmax + 1):
        new = [0]
        for k in range(n):
            new.append(new[-1] + row[n - 1 - k])
        row = new
        zig.append(row[-1])
    return [zig[2 * i] for i in range(nmax + 1)]


# ---------------------------------------------------------------- tier A
def test_bernoulli_values_exact():
    """Small B_n against exact rationals (generating function z/(e^z-1))."""
    p = 1000003
    B = oracle.bernoulli_mod_p(p, 40)
    for n in range(0, 41):
        ref = sympy.bernoulli(n)
        if n == 1:
            ref = sympy.Rational(-1, 2)  # z/(e^z-1) convention; sympy>=1.12 returns +1/2
        assert B[n] == _modq(ref, p), n
    assert B[3] == 0 and B[5] == 0  # B_{2k+1} = 0


def test_37_divides_B32():
    """37 is the smallest irregular prime; B_32 = -7709321041217/510, 37 | numerator."""
    assert oracle.bernoulli_mod_p(37, 32)[32] == 0
    for p in _primes(5, 37):
        B = oracle.bernoulli_mod_p(p, p - 3)
        assert all(B[k] != 0 for k in range(2, p - 2, 2)), p  # regular primes < 37


def test_euler_values_exact():
    """E_{2n}, secant convention: 1, 1, 5, 61, 1385, 50521, ..."""
    sec = _secant_numbers(20)
    assert sec[:6] == [1, 1, 5, 61, 1385, 50521]
    p = 1000003
    E = oracle.euler_mod_p(p, 40)
    assert E == [v % p for v in sec]
    # sympy uses sech (footnote P:L74): E^sec_{2n} = (-1)^n E^sech_{2n}
    for n in range(0, 21):
        assert (-1) ** n * int(sympy.euler(2 * n)) == sec[n]


def test_19_divides_E10():
    """the smallest E-irregular prime is 19, as 19 | E_10."""
    assert oracle.euler_mod_p(19, 10)[5] == 0
    assert 50521 % 19 == 0
    for p in _primes(5, 19):
        E = oracle.euler_mod_p(p, p - 3)
        assert all(e != 0 for e in E[1:]), p


def test_tier_A_against_exact_rationals():
    """B_{p-3}, E_{p-3} mod p from the oracle's recurrences equal the exact
    rational / integer values reduced mod p, for every prime 5 <= p < 400."""
    plist = _primes(5, 400)
    sec = _secant_numbers(200)
    for p in plist:
        assert oracle.B_recurrence(p) == _modq(sympy.bernoulli(p - 3), p), p
        assert oracle.E_recurrence(p) == sec[(p - 3) // 2] % p, p


SMALL_VECTORS = {  # SURVEY.md section 4 "Exact small-p vectors" (p: (B_{p-3}, E_{p-3}) mod p)
    5: (1, 1), 7: (3, 5), 11: (4, 10), 13: (5, 3), 17: (4, 9), 19: (15, 7), 23: (15, 22),
    29: (27, 3), 31: (14, 22), 37: (2, 4), 41: (31, 4), 43: (15, 4), 47: (24, 14), 53: (49, 46),
    59: (31, 12), 61: (38, 16), 67: (31, 25), 71: (54, 49), 73: (53, 25), 79: (22, 75),
    83: (7, 60), 89: (4, 56), 97: (50, 42), 101: (76, 86), 103: (100, 57), 107: (8, 89),
    109: (59, 23),
}


def test_small_vectors():
    # p=5: B_2 = 1/6 == 1 (mod 5); p=7: B_4 = -1/30 == 3 (mod 7); E_2 = 1, E_4 = 5.
    for p, (b, e) in SMALL_VECTORS.items():
        assert (oracle.residue_B(p), oracle.residue_E(p)) == (b, e), p
        assert _modq(sympy.bernoulli(p - 3), p) == b


# ---------------------------------------------------------------- tier B / C agreement
def test_tier_B_W_matches_tier_A():
    """Harmonic mod p^2 (eqnWolst + Glaisher) == Bernoulli recurrence, all 5 <= p < 1500,
    and the printed binomial form eqnGlaisher agrees too."""
    for p in _primes(5, 1500):
        a = oracle.B_recurrence(p)
        assert oracle.B_harmonic(p) == a, p
        assert oracle.B_glaisher(p) == a, p


def test_tier_B_V_matches_tier_A():
    """Quarter sum with reading R1 (-4 E_{p-3} == sum_{s<p/4} s^-2) == secant recurrence,
    all 5 <= p < 1500 -- both residue classes mod 4, so a sign error in R1 fails here."""
    n3 = 0
    for p in _primes(5, 1500):
        assert oracle.E_quarter(p) == oracle.E_recurrence(p), p
        n3 += p % 4 == 3
    assert n3 > 100


def test_printed_glaisher_E1_sign_reading():
    """eqnE1 as printed at k=1 carries (-1)^{(p-1)/2-1}; it disagrees with the secant
    convention exactly when p == 3 mod 4 (R1) -- the reading is forced."""
    for p in _primes(7, 400):
        e = oracle.E_recurrence(p)
        q = oracle.quarter_sum(p)
        printed = ((-1) ** ((p - 1) // 2 - 1) * 4 * e) % p
        if p % 4 == 1:
            assert printed == q
        else:
            assert printed == (-q) % p and q != 0


def test_p2_long_multiplication_exact():
    """The wide tier's base-p digit product (a0 + a1 p)(b0 + b1 p) mod p^2 equals Python's exact integer
    a*b mod p^2 for seeded random operands and moduli up to 2^62 (both digit columns, carries > 2^64)."""
    rng = random.Random(1157)
    for bits in (20, 33, 36, 45, 61):
        for _ in range(40):
            p = rng.randrange(1 << (bits - 1), 1 << bits) | 1
            a, b = rng.randrange(p * p), rng.randrange(p * p)
            assert oracle.p2_mul(a, b, p) == a * b % (p * p), (p, a, b)
        p = (1 << bits) - 1
        assert oracle.p2_mul(p * p - 1, p * p - 1, p) == 1          # (-1)^2


def test_wide_harmonic_matches_narrow_and_definition():
    """Tier B in base-p digits (the W oracle for p >= 2^32) == the one-word tier B and the Bernoulli
    recurrence (tier A) wherever those apply; H2 itself (not only its p-quotient) is compared."""
    for p in _primes(5, 700):
        assert oracle.B_harmonic_wide(p) == oracle.B_recurrence(p), p
    rng = random.Random(3)
    for _ in range(6):
        p = int(sympy.nextprime(rng.randrange(10 ** 5, 2 * 10 ** 6)))
        assert oracle.wolstenholme_h2_wide(p) == oracle.wolstenholme_h2(p), p
        assert oracle.B_harmonic_wide(p) == oracle.B_harmonic(p), p
    for p in _known()["wolstenholme_below_6e10"]:
        assert oracle.B_harmonic_wide(p) == 0, p                  # H2 == 0 mod p^3


def test_table2_rows_above_2_32_from_definition():
    """Table 2: the rows with p > 2^32, computed by oracle tier B in base-p digits
    (sum k^-2 mod p^2 -- the definition-level W oracle of every C4/C5 prime) by the committed script
    scripts/gen_wide_goldens.py, equal the printed symmetric residues, sign included."""
    path = os.path.join(GOLD, "oracle_table2_wide.json")
    if not os.path.exists(path):
        pytest.skip("oracle_table2_wide.json not generated yet (scripts/gen_wide_goldens.py)")
    with open(path) as f:
        got = {int(p): r for p, r in json.load(f)["res_w"].items()}
    rows = {int(r["p"]): int(r["symres_B"]) for r in _table("paper_table2_bernoulli.csv")}
    above = [p for p in rows if p > (1 << 32)]
    assert len(above) == 14 and set(got) == set(above)
    for p in above:
        assert oracle.symres(got[p], p) == rows[p], p


def test_tier_B_and_C_agree_random():
    """Stafford-Vandiver (eqnSV, tier C; pin only) == harmonic (tier B) on seeded random primes."""
    rng = random.Random(2101_11157)
    for _ in range(12):
        p = int(sympy.nextprime(rng.randrange(10 ** 4, 3 * 10 ** 6)))
        assert oracle.B_stafford_vandiver(p) == oracle.B_harmonic(p), p


def test_tier_A_larger_random():
    rng = random.Random(7)
    for _ in range(3):
        p = int(sympy.nextprime(rng.randrange(2000, 5000)))
        assert oracle.B_harmonic(p) == oracle.B_recurrence(p)
        assert oracle.E_quarter(p) == oracle.E_recurrence(p)


# ---------------------------------------------------------------- paper-printed pins
def _known():
    with open(os.path.join(GOLD, "paper_known_primes.json")) as f:
        return json.load(f)


def test_wolstenholme_primes():
    """Theorem 1: 16843 and 2124679 are Wolstenholme primes."""
    k = _known()
    for p in k["wolstenholme_below_6e10"]:
        assert oracle.B_harmonic(p) == 0
    # eqnWolst third form: C(2p-1, p-1) == 1 mod p^4 at 16843 (and 2124679 via h2)
    assert oracle.binom_2p_1_mod_p4(16843) == 1
    assert oracle.B_glaisher(16843) == 0
    assert oracle.wolstenholme_h2(2124679) == 0
    # and a non-example: 2946901 is a Vandiver but not a Wolstenholme prime
    assert oracle.B_harmonic(2946901) == 299776


@pytest.mark.slow
def test_vandiver_primes():
    """Theorem 1 with reading R3: E_{p-3} == 0 at all eight Vandiver primes below 4*10^10."""
    k = _known()
    for p in k["vandiver_below_4e10"]:
        assert oracle.residue_E(p) == 0, p
    p = k["not_vandiver_printed_in_theorem1"]
    assert oracle.symres(oracle.residue_E(p), p) == -85724
    c = k["composite_in_baseline_json"]
    assert c == 4547 * 228457


def test_vandiver_small_by_definition():
    """149 | E_146 and 241 | E_238 from the secant recurrence itself (tier A)."""
    assert oracle.E_recurrence(149) == 0
    assert oracle.E_recurrence(241) == 0
    assert oracle.B_recurrence(149) != 0


def _table(name):
    with open(os.path.join(GOLD, name)) as f:
        return list(csv.DictReader(r for r in f if not r.startswith("#")))


@pytest.mark.slow
def test_table2_rows_near_1e9():
    """Table 2: 1025793739 -> -9, 1029113299 -> -7 (tier C, eqnSV)."""
    rows = {int(r["p"]): int(r["symres_B"]) for r in _table("paper_table2_bernoulli.csv")}
    for p in (1025793739, 1029113299):
        assert oracle.symres(oracle.B_stafford_vandiver(p), p) == rows[p]


@pytest.mark.slow
def test_table3_rows_near_1e9():
    """Table 3: 1062232319 -> 0 (exact) and 1348936931 -> |17| (R2)."""
    rows = {int(r["p"]): (int(r["symres_E"]), int(r["sign_exact"])) for r in _table("paper_table3_euler.csv")}
    p = 1348936931
    v = oracle.symres(oracle.E_quarter(p), p)
    assert abs(v) == abs(rows[p][0]) and rows[p][1] == 0
    assert v == -17  # secant convention (R2): the printed +17 has the sech sign


# ---------------------------------------------------------------- primes
def test_prime_counts():
    with open(os.path.join(GOLD, "paper_prime_counts.json")) as f:
        counts = json.load(f)["counts"]
    for c in counts:
        if c["hi"] <= 10 ** 7:
            assert oracle.prime_count(c["lo"], c["hi"]) == c["n"], c
    assert oracle.primes(0, 30) == [2, 3, 5, 7, 11, 13, 17, 19, 23, 29]
    assert oracle.primes(10 ** 9, 10 ** 9 + 2000) == _primes(10 ** 9, 10 ** 9 + 2000)


def test_c4_golden_samples_are_the_stated_sample():
    """tests/golden/oracle_c4.npz holds all 64 samples floor(j*N/64) of the C4 window's primes (the oracle's
    sieve), each W residue written by scripts/gen_wide_goldens.py from oracle tier B; the duplicates computed
    on two hosts agree (scripts/data/oracle_wide_cache*.jsonl)."""
    import glob
    import numpy as np
    from paper_2101_11157_b200.workloads import CONFIGS, sample_indices
    z = np.load(os.path.join(GOLD, "oracle_c4.npz"))
    meta = json.loads(str(z["meta"]))
    assert meta["complete"] and meta["samples_present"] == 64
    w = CONFIGS["c4"]
    ps = oracle.primes(w.lo, w.hi)
    assert z["p"].tolist() == [ps[i] for i in sample_indices(len(ps), 64)]
    vals = {}
    for path in glob.glob(os.path.join(os.path.dirname(GOLD), "..", "scripts", "data", "oracle_wide_cache*.jsonl")):
        for line in open(path):
            d = json.loads(line)
            vals.setdefault((d["p"], d["test"]), set()).add(d["res"])
    assert all(len(v) == 1 for v in vals.values())
    assert [vals[(int(p), "W")].pop() for p in z["p"]] == z["res_w"].tolist()
