"""One census call for ncu (scripts/profile_census.py LO HI): the walk kernel dominates."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_11157_b200 as wv
lo, hi = (int(float(x)) for x in sys.argv[1:3]) if len(sys.argv) > 2 else (90000, 100000)
pairs, n, chk = wv.census(lo, hi, wv.MODE_BOTH)
print(n, len(pairs), f"{chk:016x}")
