"""Per-rank step time of the C2 bench window when split over N ranks (interleaved blocks), measured
one shard at a time on one GPU: what each rank of an N-GPU run does.  Not a bench line."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_11157_b200 as wv
from paper_2101_11157_b200.workloads import CONFIGS

w = CONFIGS["c2"]
ns = [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]
for n in ns:
    worst = 0.0
    for shard in range(n):
        ds = wv.DeviceSearch(w.lo, w.hi, w.mode, shard, n)
        for _ in range(3):
            ds.run(hit_count=False, prime_count=False)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(5):
            ds.run(hit_count=False, prime_count=False)
        e.record()
        torch.cuda.synchronize()
        worst = max(worst, s.elapsed_time(e) / 5)
    print(f"N={n}: max per-rank step {worst:.3f} ms -> {216814 / (worst / 1e3):.3e} primes/s aggregate, "
          f"efficiency vs N=1 (if N=1 is {n}x) printed by the caller", flush=True)
