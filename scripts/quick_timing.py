"""Scratch timing of wv_search_device on BASELINE windows (CUDA events; not a bench line)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_11157_b200 as wv
from paper_2101_11157_b200.workloads import CONFIGS, SUBWINDOWS

names = sys.argv[1:] or ["c1", "c2"]
for name in names:
    w = CONFIGS.get(name) or SUBWINDOWS[name]
    ds = wv.DeviceSearch(w.lo, w.hi, w.mode)
    ds.run()
    reps = int(os.environ.get("REPS", 3 if name in ("c1", "c2") else 1))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        ds.run()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    wv.stats_reset(); wv.stats_enable(True); ds.run(); wv.stats_enable(False); st = wv.stats()
    tps = st["terms"] / (st["residue_ms"] / 1e3) if st["residue_ms"] else 0
    print(f"{name}: {ds.n_primes} primes, {ds.n_hits} hits, {ms:.3f} ms/run, {ds.n_primes / ms * 1e3:.1f} primes/s, "
          f"residue {st['residue_ms']:.2f} ms, {tps:.3e} terms/s, chk {ds.checksum_int():016x}", flush=True)
