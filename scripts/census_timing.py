"""Timing of the NEXT-3 census (wv_census) on windows of small primes (CUDA-synchronous host API;
wall clock around the call, which includes the sieve, plan, walk, finalize and D2H).

    python scripts/census_timing.py [LO:HI ...]

Algorithmic work: every index residue of p costs (p-1)/2 walk steps (one Montgomery product each),
so a window costs sum_p nexp(p) (p-1)/2 steps; Gstep/s is compared with the Mont32 ALU peak of
DESIGN.md section 5 (3722 G products/s: 64 IMAD/clk/SM x 148 SMs x 1965 MHz / 5 slots)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2101_11157_b200 as wv

PEAK = 64 * 148 * 1.965e9 / 5 / 1e9
wins = [tuple(int(float(x)) for x in a.split(":")) for a in sys.argv[1:]] or [(5, 10 ** 4), (5, 10 ** 5)]
for lo, hi in wins:
    for mode in (3,):
        wv.census(lo, min(hi, lo + 1000), mode)                        # warm-up (context, module)
        t = time.perf_counter()
        pairs, npr, chk = wv.census(lo, hi, mode)
        dt = time.perf_counter() - t
        ps = wv.sieve_device(lo, hi).astype(np.float64)
        steps = float(np.sum((ps - 3) * ((ps - 1) // 2)))
        nb = int(np.sum(pairs["kind"] == 1)); ne = int(np.sum(pairs["kind"] == 2))
        print(json.dumps(dict(window=[lo, hi], mode=mode, primes=npr, seconds=round(dt, 4),
                              index_residues=int(np.sum(ps - 3)), gsteps_s=round(steps / dt / 1e9, 1),
                              frac_of_mont32_peak=round(steps / dt / 1e9 / PEAK, 3), b_pairs=nb, e_pairs=ne,
                              checksum=f"{chk:016x}")), flush=True)
