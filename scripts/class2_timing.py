#!/usr/bin/env python3
"""Class-2 (p >= 2^44, 64-bit Montgomery) engines: terms/s of each kernel variant on the first primes
above 2^44 (or --base), W+V, and bit-identity of their residues.   python scripts/class2_timing.py [n] [--base B]"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_11157_b200 as wv

ap = argparse.ArgumentParser()
ap.add_argument("n", type=int, nargs="?", default=8)
ap.add_argument("--base", type=int, default=1 << 44)
ap.add_argument("--cls", type=int, default=2)
ap.add_argument("--variants", default="")
a = ap.parse_args()
ps = [int(x) for x in wv.sieve_device(a.base, a.base + 400 * a.n)[: a.n]]
ids = {name: vid for vid, name, cls in wv.kernel_variants() if cls == a.cls}
names = [v for v in a.variants.split(",") if v] or list(ids)
out, ref = {}, None
for name in names:
    wv.set_kernel_variant(a.cls, ids[name])
    wv.residues_of(ps[:1], 3)
    torch.cuda.synchronize()
    wv.stats_reset(); wv.stats_enable(True)
    t0 = time.perf_counter()
    rw, rv = wv.residues_of(ps, 3)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st = wv.stats(); wv.stats_enable(False)
    same = None if ref is None else (rw.tolist() == ref[0].tolist() and rv.tolist() == ref[1].tolist())
    ref = ref or (rw, rv)
    out[name] = dict(seconds=round(dt, 3), kernel_ms=round(st["residue_ms"], 1), terms=st["terms"],
                     terms_per_s=st["terms"] / (st["residue_ms"] / 1e3) if st["residue_ms"] else None,
                     identical_to_first=same)
    print(name, json.dumps(out[name]), flush=True)
wv.set_kernel_variant(a.cls, -1)
print(json.dumps({"primes": ps, "base": a.base, "results": out}))
