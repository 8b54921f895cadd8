"""Small, fixed targets for ncu captures (each runs the path twice; profile the 2nd launch).
   c2   : DeviceSearch over configs[1] (class-0 Mont32 kernel dominates)
   c4s  : residues of the oracle's 8-prime C4 sample (class-1 FP64 kernel)
   c5s  : residues of the oracle's C5 sample, both tests
   c2big: the two smallest primes above 2^44, W (class-2 Mont64 eight-term kernel)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2101_11157_b200 as wv
from paper_2101_11157_b200.workloads import CONFIGS

what = sys.argv[1] if len(sys.argv) > 1 else "c2"
if what == "c2":
    w = CONFIGS["c2"]
    ds = wv.DeviceSearch(w.lo, w.hi, w.mode)
    for _ in range(2):
        ds.run()
elif what == "c2big":
    for _ in range(2):
        wv.residues_of([17592186044423, 17592186044437], 1)
else:
    z = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", f"oracle_{what[:2]}.npz"))
    for _ in range(2):
        wv.residues_of(z["p"][:8].tolist(), CONFIGS[what[:2]].mode)   # 8 samples: ncu replays the launch ~40x
torch.cuda.synchronize()
print("ok", what)
