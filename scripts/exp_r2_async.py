import sys; sys.path.insert(0, '.')
import torch, paper_2101_11157_b200 as wv
from paper_2101_11157_b200.workloads import CONFIGS
w = CONFIGS["c2"]
for n in (4, 8):
  for sync in (False, True):
    worst = 0
    for s in range(n):
        ds = wv.DeviceSearch(w.lo, w.hi, w.mode, s, n)
        for _ in range(3): ds.run(hit_count=sync, prime_count=sync)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        for _ in range(5): ds.run(hit_count=sync, prime_count=sync)
        b.record(); torch.cuda.synchronize()
        t = a.elapsed_time(b) / 5; worst = max(worst, t)
        print(f"N={n} sync={sync} shard {s}: {t:.3f}", flush=True)
    print(f"N={n} sync={sync} worst {worst:.3f}", flush=True)
