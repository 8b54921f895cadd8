#!/usr/bin/env python3
"""Write oracle residues to tests/golden/ -- calls only oracle/ (and workloads).

Usage: python scripts/gen_oracle_goldens.py [c1] [c2] [c3] [c4] [c5] [pin_v] [--workers N]

Outputs (np.savez_compressed): tests/golden/oracle_<name>.npz with arrays
  p (uint64), res_w (uint64; 2^64-1 = not requested), res_v (uint64), and a
  json 'meta' string (window, mode, sampling rule, oracle tiers, timing).
Full windows for c1/c2; for c3..c5/pin_v the deterministic sample
floor(j*N/k) of the window's primes (k = 64 for c3/pin_v, 8 for c4/c5).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2101_11157_b200.workloads import CONFIGS, sample_indices  # noqa: E402

NONE = (1 << 64) - 1
SAMPLES = {"c3": 64, "c4": 8, "c5": 8, "pin_v": 64}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["c1", "c2"])
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    a = ap.parse_args()
    for name in a.names:
        w = CONFIGS[name]
        t0 = time.time()
        ps = oracle.primes(max(w.lo, 5), w.hi)
        n_all = len(ps)
        if name in SAMPLES:
            ps = [ps[i] for i in sample_indices(len(ps), SAMPLES[name])]
            if name == "pin_v" and 1062232319 not in ps:
                ps = sorted(ps + [1062232319])
        # big primes first so the pool stays busy
        order = sorted(range(len(ps)), key=lambda i: -ps[i])
        out = oracle.residues([ps[i] for i in order], w.mode, workers=a.workers)
        res = {p: (rw, rv) for p, rw, rv in out}
        p_arr = np.array(ps, dtype=np.uint64)
        rw = np.array([NONE if res[p][0] is None else res[p][0] for p in ps], dtype=np.uint64)
        rv = np.array([NONE if res[p][1] is None else res[p][1] for p in ps], dtype=np.uint64)
        meta = dict(window=[w.lo, w.hi], mode=w.mode, name=name, primes_in_window=n_all,
                    sampled=name in SAMPLES, sample_k=SAMPLES.get(name), seconds=time.time() - t0,
                    workers=a.workers, generator="scripts/gen_oracle_goldens.py (oracle/ only)")
        path = os.path.join(ROOT, "tests", "golden", f"oracle_{name}.npz")
        np.savez_compressed(path, p=p_arr, res_w=rw, res_v=rv, meta=json.dumps(meta))
        print(name, len(ps), "primes", f"{time.time() - t0:.1f}s", path, flush=True)


if __name__ == "__main__":
    main()
