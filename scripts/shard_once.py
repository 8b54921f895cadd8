"""One step of shard S of N of the C2 window (for an ncu launch list of a per-rank step)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_11157_b200 as wv
from paper_2101_11157_b200.workloads import CONFIGS

w = CONFIGS["c2"]
s, n = int(sys.argv[1]), int(sys.argv[2])
ds = wv.DeviceSearch(w.lo, w.hi, w.mode, s, n)
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
    ds.run()
torch.cuda.synchronize()
