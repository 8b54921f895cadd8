"""Per-rank step time and residue-kernel time of the C2 bench window split over N ranks (interleaved
blocks), one shard at a time on one GPU.  Diagnostic for strong scaling; not a bench line."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_11157_b200 as wv
from paper_2101_11157_b200.workloads import CONFIGS

w = CONFIGS["c2"]
blocks = [int(b) for b in os.environ.get("BLOCKS", "0").split(",")]
for blk in blocks:
    for n in [int(x) for x in os.environ.get("NS", "1,8").split(",")]:
        rows = []
        for shard in range(n):
            ds = wv.DeviceSearch(w.lo, w.hi, w.mode, shard, n, block=blk) if blk else wv.DeviceSearch(w.lo, w.hi, w.mode, shard, n)
            for _ in range(3):
                ds.run()
            torch.cuda.synchronize()
            wv.stats_reset(); wv.stats_enable(True)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(5):
                ds.run()
            e.record()
            torch.cuda.synchronize()
            wv.stats_enable(False)
            st = wv.stats()
            rows.append((shard, ds.n_primes, s.elapsed_time(e) / 5, st["residue_ms"] / 5, st["terms"] / 5))
        worst = max(r[2] for r in rows)
        print(f"block={blk} N={n}: worst step {worst:.3f} ms", flush=True)
        for r in rows:
            print(f"  shard {r[0]}: primes {r[1]} step {r[2]:.3f} ms residue {r[3]:.3f} ms "
                  f"other {r[2]-r[3]:.3f} ms terms {r[4]:.3e}", flush=True)
