"""NEXT-3: general-index residues B_{2k}, E_{2k} mod p (the irregular-pair census).

CPU: the oracle's all-index arrays (tier A) are pinned against exact rationals (sympy), the
secant numbers by Seidel's triangle, and the counts the paper prints (37 | B_32, P:L71;
19 | E_10; the E-irregularity index 5 of p = 5783).
GPU (through the C ABI): every (p, 2k) of all primes < 1500 bit-exact against the oracle,
closed forms for small indices and the hot path's B_{p-3} / E_{p-3} at large p, the paper's
census facts, checksums and edge cases."""
import random

import numpy as np
import pytest
import sympy

import oracle

M64 = (1 << 64) - 1


def _modq(fr, p):
    num, den = sympy.fraction(sympy.Rational(fr))
    return int(num) * pow(int(den), -1, p) % p


def _mix64(z):
    """splitmix64 finaliser (no increment), as include/wv.h states"""
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _rotl(x, r):
    return ((x << r) | (x >> (64 - r))) & M64


def _chk_term(p, index, kind, res):
    """include/wv.h wv_census_checksum_term, retyped from the header's definition."""
    return _mix64(p ^ (index << 32) ^ _rotl(res, 17) ^ (kind << 62))


def _secant(nmax):
    """E_0, E_2, ..., E_{2 nmax} of sec z by Seidel's boustrophedon (integer additions only)."""
    zig, row = [1], [1]
    for n in range(1, 2 * nmax + 1):
        new = [0]
        for k in range(n):
            new.append(new[-1] + row[n - 1 - k])
        row = new
        zig.append(row[-1])
    return [zig[2 * i] for i in range(nmax + 1)]


# ---------------------------------------------------------------- oracle pins (CPU)
def test_oracle_index_residues_exact_small_p():
    """Every index of every prime 5 <= p < 200 against exact B_n (sympy) and secant numbers."""
    sec = _secant(100)
    for p in sympy.primerange(5, 200):
        for i, b, e in oracle.index_residues(p):
            assert b == _modq(sympy.bernoulli(i), p), (p, i)
            assert e == sec[i // 2] % p, (p, i)


def test_oracle_paper_census_facts():
    """37 | B_32 and 19 | E_10 are the only (E-)irregular pairs of those primes
    (sympy: 37 is the first irregular prime); p = 5783 has E-irregularity index 5."""
    ib, ie = oracle.irregular_pairs(37)
    assert ib == [32]
    ib, ie = oracle.irregular_pairs(19)
    assert ie == [10]
    _, ie = oracle.irregular_pairs(5783)
    assert len(ie) == 5


# ---------------------------------------------------------------- GPU parity
def _by_p(recs):
    out = {}
    for r in recs:
        out.setdefault(int(r["p"]), []).append((int(r["index"]), int(r["res_b"]), int(r["res_e"])))
    return out


@pytest.mark.gpu
def test_census_residues_match_oracle_all_small(wv):
    """Every (p, 2k) for all primes 5 <= p < 1500, both kinds, bit-exact; the window includes
    (p, k) with C_k(3,4,6) == 0 (mod p), i.e. the fix-up congruences are exercised."""
    recs = wv.census_residues(5, 1500, wv.MODE_BOTH)
    got = _by_p(recs)
    ps = list(sympy.primerange(5, 1500))
    assert sorted(got) == ps
    want = oracle.index_residues_many(ps)
    for p in ps:
        assert got[p] == want[p], p
    fix = [(p, 2 * k) for p in ps for k in range(1, (p - 3) // 2 + 1)
           if (pow(3, p - 2 * k, p) + pow(4, p - 2 * k, p) - pow(6, p - 2 * k, p) - 1) % p == 0]
    assert len(fix) > 50
    # single-kind modes give the same values
    rb = _by_p(wv.census_residues(5, 300, wv.MODE_W))
    re_ = _by_p(wv.census_residues(5, 300, wv.MODE_V))
    for p in sympy.primerange(5, 300):
        assert [(i, b) for i, b, _ in rb[p]] == [(i, b) for i, b, _ in want[p]]
        assert [(i, e) for i, _, e in re_[p]] == [(i, e) for i, _, e in want[p]]
        assert all(e == wv.RES_NONE for _, _, e in rb[p]) and all(b == wv.RES_NONE for _, b, _ in re_[p])


@pytest.mark.gpu
def test_census_residues_match_oracle_multisegment(wv):
    """Two primes above 16384 (walks of > 8192 steps: several segments per index) vs the oracle."""
    lo, hi = 20011, 20022                          # 20011, 20021
    got = _by_p(wv.census_residues(lo, hi, wv.MODE_BOTH))
    want = oracle.index_residues_many(list(sympy.primerange(lo, hi)))
    assert sorted(got) == sorted(want) == [20011, 20021]
    for p in want:
        assert got[p] == want[p], p


@pytest.mark.gpu
def test_census_closed_forms_and_hot_path_at_large_p(wv):
    """Primes in [10^5, 10^5 + 600): small indices against exact values (B_2 = 1/6, B_4 = -1/30,
    B_6 = 1/42, E_2 = 1, E_4 = 5, E_6 = 61) and index p-3 against the hot path (wv_search),
    itself bit-exact against the oracle -- two unrelated methods."""
    lo, hi = 100000, 100600
    got = _by_p(wv.census_residues(lo, hi, wv.MODE_BOTH))
    hits, res = wv.search(lo, hi, wv.MODE_BOTH)
    hot = {int(r["p"]): (int(r["res_w"]), int(r["res_v"])) for r in res}
    assert sorted(got) == sorted(hot)
    exact_b = {2: sympy.Rational(1, 6), 4: sympy.Rational(-1, 30), 6: sympy.Rational(1, 42)}
    exact_e = {2: 1, 4: 5, 6: 61}
    for p, rows in got.items():
        d = {i: (b, e) for i, b, e in rows}
        for i in (2, 4, 6):
            assert d[i][0] == _modq(exact_b[i], p) and d[i][1] == exact_e[i] % p, (p, i)
        assert d[p - 3] == hot[p], p


@pytest.mark.gpu
def test_census_pairs_and_checksum_small(wv):
    """Pairs of [5, 1500) = the oracle's zero set; checksum = sum of the header's terms over the
    oracle residues; a ragged split of the window gives the same pairs and checksums that add."""
    pairs, npr, chk = wv.census(5, 1500, wv.MODE_BOTH)
    ps = list(sympy.primerange(5, 1500))
    assert npr == len(ps)
    want = oracle.index_residues_many(ps)
    wp, wc = [], 0
    for p in ps:
        for i, b, e in want[p]:
            if b == 0:
                wp.append((p, i, 1))
            wc = (wc + _chk_term(p, i, 1, b)) & M64
        for i, b, e in want[p]:
            if e == 0:
                wp.append((p, i, 2))
            wc = (wc + _chk_term(p, i, 2, e)) & M64
    assert [(int(x["p"]), int(x["index"]), int(x["kind"])) for x in pairs] == wp
    assert chk == wc
    assert wv.census_checksum_term(37, 32, 1, 0) == _chk_term(37, 32, 1, 0)
    a = wv.census(5, 777, wv.MODE_BOTH)
    b = wv.census(777, 1500, wv.MODE_BOTH)
    assert list(a[0]) + list(b[0]) == list(pairs)
    assert (a[2] + b[2]) & M64 == chk


@pytest.mark.gpu
def test_census_paper_facts(wv):
    """[5, 10^4): the maximum E-irregularity index is 5, attained by p = 5783 alone (Ernvall and
    Metsankyla).  [5, 30000): 16843 is the only prime with (p, p-3) an irregular pair
    (P:L91-94); the E-pairs (p, p-3) are exactly the Vandiver primes 149, 241."""
    pairs, npr, _ = wv.census(5, 10 ** 4, wv.MODE_V)
    assert npr == 1227                      # pi(10^4) = 1229 minus 2 and 3
    cnt = {}
    for x in pairs:
        assert int(x["kind"]) == 2
        cnt[int(x["p"])] = cnt.get(int(x["p"]), 0) + 1
    m = max(cnt.values())
    assert m == 5 and [p for p, c in cnt.items() if c == m] == [5783]
    pairs, npr, _ = wv.census(5, 30000, wv.MODE_BOTH)
    top = [(int(x["p"]), int(x["kind"])) for x in pairs if int(x["index"]) == int(x["p"]) - 3]
    assert top == [(149, 2), (241, 2), (16843, 1)]
    # 37 is the smallest irregular prime and (37, 32) its only pair
    first = [(int(x["p"]), int(x["index"])) for x in pairs if int(x["kind"]) == 1][:1]
    assert first == [(37, 32)]


@pytest.mark.gpu
def test_census_edges(wv):
    """p = 5, 7 (one / two indices), empty windows, and invalid arguments."""
    r = wv.census_residues(5, 8, wv.MODE_BOTH)
    assert [(int(x["p"]), int(x["index"]), int(x["res_b"]), int(x["res_e"])) for x in r] == \
        [(5, 2, 1, 1), (7, 2, 6, 1), (7, 4, 3, 5)]          # B_2 = 1/6, B_4 = -1/30, E_2 = 1, E_4 = 5
    assert len(wv.census_residues(0, 5, wv.MODE_BOTH)) == 0
    assert len(wv.census_residues(24, 29, wv.MODE_BOTH)) == 0
    p, n, c = wv.census(24, 29, wv.MODE_BOTH)
    assert len(p) == 0 and n == 0 and c == 0
    for args in ((10, 10, 3), (10, 5, 3), (5, 100, 0), (5, 100, 4), (5, (1 << 26) + 1, 3)):
        with pytest.raises(wv.WVError):
            wv.census(*args)
