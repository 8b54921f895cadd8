"""Time each residue-kernel variant on windows of its prime class (CUDA events; not a bench line)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_11157_b200 as wv
from paper_2101_11157_b200.workloads import CONFIGS, SUBWINDOWS

WIN = {0: sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2", "c3_slice", "c3_slice_both"],
       1: sys.argv[2].split(",") if len(sys.argv) > 2 else ["c4_head", "c5_head"],
       2: ["c2_probe"]}
ONLY = set(int(x) for x in sys.argv[3].split(",")) if len(sys.argv) > 3 else None
for vid, name, cls in wv.kernel_variants():
    if cls not in WIN or (ONLY is not None and vid not in ONLY):
        continue
    wv.set_kernel_variant(cls, vid)
    for wname in WIN[cls]:
        w = CONFIGS.get(wname) or SUBWINDOWS.get(wname)
        if w is None:
            continue
        ds = wv.DeviceSearch(w.lo, w.hi, w.mode)
        ds.run()
        wv.stats_reset(); wv.stats_enable(True)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); ds.run(); e.record(); torch.cuda.synchronize()
        wv.stats_enable(False); st = wv.stats()
        print(f"[{vid}] {name:12s} {wname:14s} {s.elapsed_time(e):9.2f} ms  residue {st['residue_ms']:9.2f} ms  "
              f"{st['terms'] / st['residue_ms'] * 1e3:.3e} terms/s  chk {ds.checksum_int():016x}", flush=True)
    wv.set_kernel_variant(cls, -1)
