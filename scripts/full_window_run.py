"""Evidence run of a whole BASELINE window on one GPU: hits, near misses (|<r>| < 50), histogram
flatness, checksum, device time and throughput.  Writes gpurun_out/full_<name>.json.
   python scripts/full_window_run.py c4 [mode]"""
import json, os, sys, time, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2101_11157_b200 as wv
from paper_2101_11157_b200.workloads import CONFIGS, SUBWINDOWS

name = sys.argv[1]
w = CONFIGS.get(name) or SUBWINDOWS[name]
mode = int(sys.argv[2]) if len(sys.argv) > 2 else w.mode
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                        "--format=csv,noheader,nounits", "-lms", "2000"], stdout=subprocess.PIPE, text=True)
ds = wv.DeviceSearch(w.lo, w.hi, mode)
wv.stats_reset(); wv.stats_enable(True)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.time()
s.record(); ds.run(); e.record(); torch.cuda.synchronize()
wall = time.time() - t0
ms = s.elapsed_time(e)
st = wv.stats(); wv.stats_enable(False)
near, hw, hv = ds.near_misses(50)
smi.terminate()
clk = [l.split(",") for l in smi.communicate()[0].strip().splitlines()]
sm = sorted(float(c[0]) for c in clk if len(c) >= 2)
hist = hw if mode & 1 else hv
n = ds.n_primes
chi2 = float((((hist.astype(np.float64) - n / 2000) ** 2) / (n / 2000)).sum()) if n else None
out = dict(window=[w.lo, w.hi], name=name, mode=mode, primes=n, hits=ds.hits_np().tolist(),
           near_misses=[(int(x["p"]), int(x["test"]), int(x["symres"])) for x in near],
           checksum=f"{ds.checksum_int():016x}", device_ms=ms, wall_s=wall, primes_per_s=n / (ms / 1e3),
           terms=st["terms"], terms_per_s=st["terms"] / (st["residue_ms"] / 1e3), residue_ms=st["residue_ms"],
           hist_chi2_1999dof=chi2, sm_mhz_median=sm[len(sm) // 2] if sm else None, samples=len(sm),
           reasons=sorted(set(c[3].strip() for c in clk if len(c) >= 4)))
# the oracle goldens of this window (tests/golden/oracle_<name>.npz, written from oracle/ only): every sampled
# prime's residues as produced by this whole-window run, compared element by element
gold = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", f"oracle_{name}.npz")
if os.path.exists(gold):
    z = np.load(gold)
    gp = z["p"]
    pr = ds.primes_np()
    rw, rv = ds.res_np()
    idx = np.searchsorted(pr, gp)
    ok_p = (idx < n) & (pr[np.minimum(idx, n - 1)] == gp)
    bad = []
    for t, got, want in (("W", rw, z["res_w"]), ("V", rv, z["res_v"])):
        if mode & (1 if t == "W" else 2):
            m = ok_p & (got[np.minimum(idx, n - 1)] != want)
            bad += [(int(p), t) for p in gp[m]]
    out["oracle_samples"] = dict(golden=os.path.relpath(gold), samples=int(len(gp)), found=int(ok_p.sum()),
                                 mismatches=bad)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(f"gpurun_out/full_{name}.json", "w"), indent=1)
print(json.dumps(out))
