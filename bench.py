#!/usr/bin/env python3
"""bench.py -- primes tested per second (W+V) on B200, per the driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl ours|reference]

A "step" is one pass of the whole hot path (sieve -> plan ->
residue -> finalize -> hits/checksum) over one BASELINE window.  The default
workload is configs[1] = C2: every prime p < 3*10^6, both tests (the config the
metric is quoted on that fits one GPU).  With N GPUs
(torchrun) the window is split into interleaved blocks (rank r takes blocks
b == r mod N; strong scaling: total work fixed) and the per-rank hit lists and
checksums are gathered with NCCL (the only collective the path has).

Timing: W untimed warm-up steps; then K steps, each bracketed by CUDA events
on the launching stream, with a 256 MiB L2-flush write between steps (outside
the events); barrier + synchronize around the timed region; the max over ranks
is reported.  nvidia-smi is sampled during the timed region.

`value`  -- device-resident path (wv_search_device into torch buffers).
`e2e`    -- the host-buffer public API (wv_search_shard): results copied D2H
            into host memory every step, wall clock, max over ranks.
`roofline` -- the dominant kernel (residue_kernel) via the library's CUDA-event
            stats hook: algorithmic Montgomery multiplications / its device time,
            against the IMAD-pipe peak from the guide's unit counts.
`cpu_baseline` -- the CPU oracle (oracle/) as it stands, on a bounded sample
            of the same workload, on this box's host cores (rank 0, N=1 only).
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "primes tested/sec (W+V)"
UNIT = "primes/s"

# Modular multiplications per term: c1 <- c1 u + c0, c0 <- c0 u
MULMODS_PER_TERM = 2
# SURVEY.md 8(d) per-unit figure: algorithmic terms per prime (BB30: 227/6480 p, EE33: 27/512 p)
TERMS_PER_P = {1: 227 / 6480, 2: 27 / 512}
# Roofline per prime class: (pipe, lanes/clk/SM, pipe ops per modular product)
#   class 0 (p < 2^30, Mont32): IMAD pipe, 64 IMAD/clk/SM (guide); a Montgomery product is 3 IMAD-class
#            ops (a b wide, m = T p^-1, hi(m p)).  Our microbenchmark measures IMAD.WIDE / IMAD.HI at half
#            rate (5 pipe slots per product); that tighter ceiling is reported alongside (peak_5slot).
#   class 1 (2^30 <= p < 2^44, FP64 EFT): fp64 pipe, 64 DFMA/clk/SM; 6 DP ops per product
#   class 2 (p >= 2^44, Mont64): fmaheavy, ~22 slots per product (11 wide/high 32-bit partial products)
ROOF = {0: ("fmaheavy", 64, 3), 1: ("fp64", 64, 6), 2: ("fmaheavy", 64, 22)}


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi sampling around the timed region (B200_PROFILING.md clocks line).

    Started before the warm-up (nvidia-smi needs ~0.1-0.3 s to emit its first sample), stopped
    after the timed region; samples whose timestamp falls inside the region are kept (if the
    region is shorter than the sampling period, the sample closest to its midpoint)."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = set(gpus)
        self.proc = None
        self.path = f"/tmp/wv_clocks_{os.getpid()}.csv"
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "50"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def stop(self):
        import datetime
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.f.close()
        rows = []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                if int(parts[1]) not in self.gpus:
                    continue
                rows.append((ts, float(parts[2]), float(parts[3]), float(parts[4]),
                             [n for n, v in zip(names, parts[6:10]) if v.lower().startswith("active")]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        inside = [r for r in rows if self.t0 is not None and self.t0 <= r[0] <= self.t1]
        note = "inside timed region"
        if not inside:
            mid = (self.t0 + self.t1) / 2 if self.t0 is not None else rows[-1][0]
            inside = [min(rows, key=lambda r: abs(r[0] - mid))]
            note = "closest sample to the timed region (region shorter than the 50 ms period)"
        sm = sorted(r[1] for r in inside)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(r[2] for r in inside),
                "reasons": sorted({x for r in inside for x in r[4]}), "samples": len(inside),
                "power_w_max": max(r[3] for r in inside), "note": note}


def _window(name):
    from paper_2101_11157_b200.workloads import CONFIGS, SUBWINDOWS
    w = CONFIGS.get(name) or SUBWINDOWS.get(name)
    if w is None:
        raise SystemExit(f"unknown workload {name}")
    return w


def cpu_oracle_rate(w, sample_k, workers):
    """Oracle primes/s on a deterministic sample of the window's primes (all host cores)."""
    import oracle
    from paper_2101_11157_b200.workloads import sample_indices
    ps = oracle.primes(max(w.lo, 5), w.hi)
    sample = [ps[i] for i in sample_indices(len(ps), sample_k)]
    t0 = time.perf_counter()
    oracle.residues(sample, w.mode, workers=workers)
    dt = time.perf_counter() - t0
    return len(sample) / dt, dt, len(sample), len(ps)


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, on the same workload (rank 0 only)."""
    rank = _env_int("RANK", 0)
    if rank != 0:
        return
    w = _window(args.workload)
    cores = os.cpu_count() or 1
    k = max(1, args.ref_sample // 2)
    times = []
    for i in range(args.warmup + args.steps):
        rate, dt, n, n_all = cpu_oracle_rate(w, k, cores)
        if i >= args.warmup:
            times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    value = k / (ms / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": w.name, "window": [w.lo, w.hi], "mode": "W+V" if w.mode == 3 else "WV"[w.mode - 1],
                       "step": f"oracle residues of a {k}-prime deterministic sample (floor(j*N/k)) of the window"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{k} of {n_all} primes of {w.name}, one prime per task"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-sample", type=int, default=2048, help="primes in the oracle's bounded sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2101_11157_b200 as wv

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    w = _window(args.workload)
    ds = wv.DeviceSearch(w.lo, w.hi, w.mode, shard=rank, nshards=world, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def gather(ds):
        """Per-rank hits/checksum -> all ranks (dist.gather_results over NCCL; gloo-tested on CPU)."""
        from paper_2101_11157_b200.dist import gather_results
        return gather_results(ds.hits_np(), None, ds.checksum_int(), device=dev)

    def step():
        ds.run(stream)
        if world > 1:
            return gather(ds)
        return None

    clocks = ClockSampler(range(world) if rank == 0 else [])
    if rank == 0:
        clocks.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    wv.stats_reset()
    wv.stats_enable(True)
    launches0 = wv.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark_start()
    evs = []
    for _ in range(args.steps):
        flush.fill_(1)                                  # L2 flush between steps (outside the events)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        out = step()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    clocks.mark_end()
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if rank == 0 else None
    wv.stats_enable(False)
    st = wv.stats()
    launches = wv.launch_count() - launches0           # our kernels inside the timed region
    ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        n_tot = torch.tensor([ds.n_primes], dtype=torch.int64, device=dev)
        dist.all_reduce(n_tot)
        n_all = int(n_tot.item())
    else:
        n_all = ds.n_primes
    ms_max = float(t.item())
    value = n_all / (ms_max / 1e3)

    # e2e through the host-buffer API (results D2H every step), wall clock, max over ranks
    e2e = None
    if not args.no_e2e:
        keep, hbuf, rbuf = wv.pinned_buffers(w.lo, w.hi, w.mode, rank, world, 0)   # pinned host memory
        for _ in range(2):
            wv.search_shard(w.lo, w.hi, w.mode, rank, world, 0, True, hbuf, rbuf)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            hits_h, res_h, chk = wv.search_shard(w.lo, w.hi, w.mode, rank, world, 0, True, hbuf, rbuf)
        dt = (time.perf_counter() - t0) / args.steps
        te = torch.tensor([dt], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        d2h = int(res_h.nbytes + hits_h.nbytes + 8)
        e2e = {"value": n_all / float(te.item()), "unit": UNIT, "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * float(te.item()),
               "api": "wv_search_shard into pinned host buffers (inputs are the window bounds passed by value)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # roofline of the dominant kernel: the residue kernel of the class with the most device time
    peaks, peak_kind = _peaks()
    steps = args.steps
    cls_terms = {0: st["terms32"] / steps, 1: st["terms_fp"] / steps,
                 2: (st["terms"] - st["terms32"] - st["terms_fp"]) / steps}
    cls_ms = {0: st["residue32_ms"] / steps, 1: st["residue_fp_ms"] / steps,
              2: (st["residue_ms"] - st["residue32_ms"] - st["residue_fp_ms"]) / steps}
    cls = max(cls_ms, key=lambda c: cls_ms[c])
    k_terms, k_ms = cls_terms[cls], cls_ms[cls]
    mhz = float(peaks.get("sm_max_mhz", 1965.0))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    pipe, lanes, slots = ROOF[cls]
    peak_mulmod = lanes * sms * mhz * 1e6 / slots
    # achieved = SURVEY 8(d) per-unit figure x units: 2 mulmods x (227/6480 p [W] + 27/512 p [V]) summed over
    # the primes of the dominant kernel's class, / that kernel's time (executed terms reported alongside)
    pr = ds.primes[: ds.n_primes]
    lim = {0: (0, 1 << 30), 1: (1 << 30, 1 << 44), 2: (1 << 44, 1 << 62)}[cls]
    sel = pr[(pr >= lim[0]) & (pr < lim[1])]
    sum_p = float(sel.double().sum().item()) if sel.numel() else 0.0
    if world > 1:
        t_sp = torch.tensor([sum_p], dtype=torch.float64, device=dev)
        dist.all_reduce(t_sp)
        sum_p = float(t_sp.item())
    alg_terms = sum(TERMS_PER_P[t] * sum_p for t in (1, 2) if w.mode & t)
    achieved = MULMODS_PER_TERM * alg_terms / (k_ms / 1e3) if k_ms > 0 else 0.0
    executed = MULMODS_PER_TERM * k_terms / (k_ms / 1e3) if k_ms > 0 else 0.0
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"r1_{args.workload}_residue_kernel_full.txt")
    if os.path.exists(prof):
        rd = wr = None
        for line in open(prof):
            f = line.split()
            if line.strip().startswith("dram bytes read"):
                rd = float(f[3]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(f[4], 1)
            if line.strip().startswith("dram bytes write"):
                wr = float(f[3]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(f[4], 1)
        if rd is not None and wr is not None:
            traffic = rd + wr
    kname = {0: "residue_lane2_kernel (class 0 lane mode, p < 2^30)", 1: "residue_kernel<Mont64, FP64 engine> (class 1)",
             2: "residue_kernel<Mont64> (class 2, p >= 2^44)"}[cls]
    roof = {"bound": "alu", "kernel": kname, "achieved": achieved / 1e9, "peak": peak_mulmod / 1e9,
            "achieved_basis": "SURVEY.md 8(d): 2 mulmods x (227/6480 p + 27/512 p) per prime (BB30/EE33 work)",
            "executed_gmulmod_s": executed / 1e9,
            "unit": "Gmulmod/s", "frac": achieved / peak_mulmod if peak_mulmod else None, "traffic": traffic,
            "traffic_unit": "bytes/launch (DRAM read+write, ncu --set full, profiles/)",
            "peak_basis": f"{pipe} pipe: {lanes} lanes/clk/SM x {sms} SMs x {mhz:.0f} MHz ({peak_kind} sm_max_mhz) "
                          f"/ {slots} pipe slots per modular product",
            "peak_5slot": lanes * sms * mhz * 1e6 / 5 / 1e9 if cls == 0 else None,
            "kernel_ms_per_step": k_ms, "kernel_share_of_step": k_ms / ms_max if ms_max else None,
            "terms_per_step": sum(cls_terms.values()), "kernel_terms_per_s": k_terms / (k_ms / 1e3) if k_ms else None}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        rate, dt, n, n_all_w = cpu_oracle_rate(w, args.ref_sample, os.cpu_count() or 1)
        cpu = {"value": rate, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "oracle",
               "sample": f"{n} of {n_all_w} primes of {w.name} (floor(j*N/k) sample), both tests, "
                         f"one prime per task, {dt:.1f} s wall"}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": {0: "u32", 1: "f64", 2: "u64"}[cls], "data": "synthetic",
            "config": {"workload": w.name, "window": [w.lo, w.hi], "mode": {1: "W", 2: "V", 3: "W+V"}[w.mode],
                       "primes": n_all, "parallelism": f"interleaved blocks x{world}",
                       "l2_flush": "256 MiB write between timed steps (outside the CUDA events)",
                       "terms_per_step": sum(cls_terms.values()),
                       "mulmods_per_s": MULMODS_PER_TERM * sum(cls_terms.values()) / (ms_max / 1e3)},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
