#!/usr/bin/env python3
"""Derive low-cost congruences with the section-2.2 greedy heuristic (NEXT-2) and record them.

    python scripts/gen_congruences.py SEED ROUNDS D OUT.json

Writes the subdivision history (replayable with congruence.replay from the seed),
cost, number of sums and the integer form (L, terms) to OUT.json.  Every congruence
is validated by direct evaluation against the oracle for all primes in
[min_p, 2000) before it is written.
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_11157_b200.congruence import seed, greedy_fast


def validate(c, pmax=2000):
    import oracle
    import sympy
    bad = []
    for p in sympy.primerange(max(c.min_p, 11), pmax):
        L, _ = c.integer_form()
        if L % p == 0:
            continue
        want = oracle.residue_B(p) if c.kind == "B" else oracle.residue_E(p)
        if c.residue(p) != want:
            bad.append(p)
    return bad


def main():
    name, rounds, D, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    resume = sys.argv[5] if len(sys.argv) > 5 else None     # history JSON to continue from
    t0 = time.time()

    def dump(r, cur):          # checkpoint the history every 10 rounds (replayable)
        if r % 10 == 0 and r:
            json.dump(dict(seed=name, D=D, rounds=r, history=[(d, str(x), str(y)) for d, x, y in cur.history],
                           r=float(1 / cur.cost()), m=cur.m()), open(out + ".partial", "w"))

    start = seed(name)
    if resume:
        from fractions import Fraction as Fr
        from paper_2101_11157_b200.congruence import replay
        start = replay(start, [(d, Fr(x), Fr(y)) for d, x, y in json.load(open(resume))["history"]])
    c = greedy_fast(start, rounds, D=D, verbose=True, on_round=dump)
    L, terms = c.integer_form()
    bad = validate(c)
    rec = dict(seed=name, rounds=rounds, D=D, cost=str(c.cost()), r=float(1 / c.cost()), m=c.m(), min_p=c.min_p,
               history=[(d, str(x), str(y)) for d, x, y in c.history], L=str(L),
               terms=[(str(a), xn, xd, yn, yd) for a, xn, xd, yn, yd in terms], bits=max(abs(int(a)).bit_length()
               for a, *_ in terms), L_bits=abs(L).bit_length(), validated_primes_below=2000, bad=bad,
               seconds=time.time() - t0)
    json.dump(rec, open(out, "w"), indent=0)
    print(name, "cost p/%.3f" % rec["r"], "m", rec["m"], "bits", rec["bits"], "bad", bad, flush=True)


if __name__ == "__main__":
    main()
