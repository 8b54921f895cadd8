"""NEXT-2: the congruence derivation engine (Prop. 1) reproduces the paper's printed
congruences from the paper's own recipes, and greedy-derived congruences agree with the oracle.
CPU only; the engine is host-side planning code."""
from fractions import Fraction as F

import sympy

import oracle
from paper_2101_11157_b200.congruence import greedy_fast, replay, seed


def _norm(L, terms):
    terms = [tuple(t) for t in terms]
    if L < 0:
        L, terms = -L, [(-t[0],) + t[1:] for t in terms]
    return L, terms


def _table():
    import __graft_entry__ as g
    g.build()
    import paper_2101_11157_b200 as wv
    return {c["name"]: (c["L"], c["terms"]) for c in wv.congruences()}


def test_recipes_reproduce_printed_congruences():
    tab = _table()
    # eqnB2: d=2 on S(1/3, 2/5) of eqnVandiver
    b2 = replay(seed("Vandiver"), [(2, F(1, 3), F(2, 5))])
    assert _norm(*b2.integer_form()) == _norm(*tab["BB2"]) and b2.cost() == F(1, 15)
    # eqnB6: four d=2 subdivisions of eqnB2
    b6 = replay(b2, [(2, F(3, 10), F(1, 3)), (2, F(1, 3), F(7, 20)), (2, F(13, 40), F(1, 3)), (2, F(1, 3), F(27, 80))])
    assert _norm(*b6.integer_form()) == _norm(*tab["BB6"]) and b6.cost() == F(5, 96)
    # intermediate steps give the m = 4 and m = 5 entries of Table 1: 7p/120, 13p/240
    assert replay(b2, [(2, F(3, 10), F(1, 3)), (2, F(1, 3), F(7, 20))]).cost() == F(7, 120)
    # eqnE3, eqnE5; eqnE9 with reading R8 (subdivide S(0,1/64), the garbled "S(0,1/128)")
    e3 = replay(seed("E1"), [(2, F(0), F(1, 4)), (2, F(0), F(1, 8))])
    assert _norm(*e3.integer_form()) == _norm(*tab["EE3"])
    e5 = replay(e3, [(2, F(0), F(1, 16)), (2, F(0), F(1, 32))])
    assert _norm(*e5.integer_form()) == _norm(*tab["EE5"])
    e9 = replay(e5, [(2, F(0), F(1, 64)), (3, F(3, 8), F(7, 16))])
    assert _norm(*e9.integer_form()) == _norm(*tab["EE9"])


def test_emac2_seed_and_greedy_agree_with_oracle():
    """eqnEMac2 at k=1 (-40 E == S(0,1/12) - S(5/12,1/2)) and a few greedy rounds from each seed
    evaluate to the oracle's residues for every prime in range."""
    for name, rounds in [("EMac2", 0), ("EMac2", 12), ("Vandiver", 12)]:
        c = greedy_fast(seed(name), rounds, D=8)
        L, _ = c.integer_form()
        for p in sympy.primerange(max(c.min_p, 11), 700):
            if L % p == 0:
                continue
            want = oracle.residue_B(p) if c.kind == "B" else oracle.residue_E(p)
            assert c.residue(p) == want, (name, rounds, p)
