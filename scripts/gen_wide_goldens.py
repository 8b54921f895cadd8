#!/usr/bin/env python3
"""Oracle goldens for p >= 2^32 (C4, C5 samples; Table 2 rows) -- calls only oracle/.

W for p >= 2^32 is the definition-level tier B of the oracle: sum_{0<k<p} k^-2 mod p^2 in base-p
digit arithmetic (eqnWolst + Glaisher), ~1000 s per prime near 6e10 on one core, so the
work runs as a resumable pool: every finished (p, test) is appended to a JSONL cache
(scripts/data/oracle_wide_cache.jsonl) and skipped on the next start.

Tasks, in this order so that a partial run still covers evenly spaced primes:
  table2  -- the Table 2 rows with p > 2^32 (pins the oracle, not the GPU);
  c4, c5  -- the deterministic samples floor(j*N/64) of the windows' primes,
             dealt in bit-reversed j order, W (and V for C5).

Usage:
  python scripts/gen_wide_goldens.py run [--workers N]     # compute (resumable)
  python scripts/gen_wide_goldens.py assemble [--partial]  # cache -> tests/golden/*.npz / *.json
"""
import argparse
import csv
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor, as_completed
import multiprocessing

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2101_11157_b200.workloads import CONFIGS, sample_indices  # noqa: E402

CACHE = os.path.join(ROOT, "scripts", "data", "oracle_wide_cache.jsonl")
CACHE_GLOB = os.path.join(ROOT, "scripts", "data", "oracle_wide_cache*.jsonl")   # + other hosts' shares
GOLD = os.path.join(ROOT, "tests", "golden")
NONE = (1 << 64) - 1
K = 64


def _bitrev_order(k):
    bits = (k - 1).bit_length()
    return sorted(range(k), key=lambda j: int(format(j, f"0{bits}b")[::-1], 2))


def _table2_primes():
    with open(os.path.join(GOLD, "paper_table2_bernoulli.csv")) as f:
        rows = list(csv.DictReader(r for r in f if not r.startswith("#")))
    return [int(r["p"]) for r in rows if int(r["p"]) >= (1 << 32)]


def _samples(name):
    w = CONFIGS[name]
    ps = oracle.primes(max(w.lo, 5), w.hi)
    return w, len(ps), [ps[i] for i in sample_indices(len(ps), K)]


def _tasks():
    out = [("table2", p, "W") for p in _table2_primes()]
    s4 = _samples("c4")[2]
    s5 = _samples("c5")[2]
    for j in _bitrev_order(K):
        out.append(("c4", s4[j], "W"))
        out.append(("c5", s5[j], "V"))
        out.append(("c5", s5[j], "W"))
    return out


def _work(task):
    tag, p, test = task
    t0 = time.time()
    r = oracle.residue_B(p) if test == "W" else oracle.residue_E(p)
    return tag, p, test, r, time.time() - t0


def _cache():
    import glob
    done = {}
    for path in sorted(glob.glob(CACHE_GLOB)):
        with open(path) as f:
            for line in f:
                if line.strip():
                    d = json.loads(line)
                    done[(d["p"], d["test"])] = d
    return done


def run(workers, reverse=False, limit=None, out=CACHE, deadline=None):
    """Compute the missing tasks (in order, or from the end with reverse -- a second host's share);
    limit: at most that many tasks; deadline: seconds after which no further task starts."""
    done = _cache()
    todo = [t for t in _tasks() if (t[1], t[2]) not in done]
    if reverse:
        todo = todo[::-1]
    if limit is not None:
        todo = todo[:limit]
    print(f"{len(done)} cached, {len(todo)} to do, {workers} workers", flush=True)
    t_start = time.time()
    ctx = multiprocessing.get_context("spawn")
    with ProcessPoolExecutor(max_workers=workers, mp_context=ctx) as ex, open(out, "a") as f:
        futs = []
        pending = list(todo)
        while pending and len(futs) < workers:
            futs.append(ex.submit(_work, pending.pop(0)))
        while futs:
            fu = next(as_completed(futs))
            futs.remove(fu)
            if pending and (deadline is None or time.time() - t_start < deadline):
                futs.append(ex.submit(_work, pending.pop(0)))
            tag, p, test, r, dt = fu.result()
            f.write(json.dumps(dict(tag=tag, p=p, test=test, res=r, seconds=round(dt, 1),
                                    tier="B (sum k^-2 mod p^2, base-p digits)" if test == "W"
                                    else "B (quarter sum, R1)")) + "\n")
            f.flush()
            print(tag, p, test, r, f"{dt:.0f}s", flush=True)


def assemble(partial):
    done = _cache()
    t2 = {p: done[(p, "W")]["res"] for p in _table2_primes() if (p, "W") in done}
    with open(os.path.join(GOLD, "oracle_table2_wide.json"), "w") as f:
        json.dump(dict(generator="scripts/gen_wide_goldens.py (oracle/ only)",
                       note="oracle tier B residues B_{p-3} mod p for the Table 2 rows with p > 2^32 "
                            "(PAPER.md L695-729); the test compares them with the printed values",
                       res_w={str(p): r for p, r in sorted(t2.items())}), f, indent=1)
    print("table2", len(t2), "rows")
    for name in ("c4", "c5"):
        w, n_all, ps = _samples(name)
        keep = []
        for p in ps:
            need = [t for t, bit in (("W", 1), ("V", 2)) if w.mode & bit]
            if all((p, t) in done for t in need):
                keep.append(p)
        if len(keep) < len(ps) and not partial:
            print(name, f"{len(keep)}/{len(ps)} samples done; not written (use --partial)")
            continue
        rw = [done[(p, "W")]["res"] if w.mode & 1 else NONE for p in keep]
        rv = [done[(p, "V")]["res"] if w.mode & 2 else NONE for p in keep]
        meta = dict(window=[w.lo, w.hi], mode=w.mode, name=name, primes_in_window=n_all, sampled=True,
                    sample_k=K, samples_present=len(keep), complete=len(keep) == len(ps),
                    oracle_tiers="W: tier B sum_{k<p} k^-2 mod p^2 (base-p digits); V: tier B quarter sum",
                    generator="scripts/gen_wide_goldens.py (oracle/ only)")
        np.savez_compressed(os.path.join(GOLD, f"oracle_{name}.npz"), p=np.array(keep, dtype=np.uint64),
                            res_w=np.array(rw, dtype=np.uint64), res_v=np.array(rv, dtype=np.uint64),
                            meta=json.dumps(meta))
        print(name, f"{len(keep)}/{len(ps)} samples written")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cmd", choices=["run", "assemble"])
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    ap.add_argument("--partial", action="store_true")
    ap.add_argument("--reverse", action="store_true")
    ap.add_argument("--limit", type=int, default=None)
    ap.add_argument("--deadline", type=float, default=None)
    ap.add_argument("--out", default=CACHE)
    a = ap.parse_args()
    if a.cmd == "run":
        run(a.workers, a.reverse, a.limit, a.out, a.deadline)
    else:
        assemble(a.partial)


if __name__ == "__main__":
    main()
