#!/usr/bin/env python3
"""bench.py -- primes tested per second (W+V) on B200, per the driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl ours|reference]
                    [--frontier-steps F] [--stub]

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

Launch: with --gpus N > 1 and no torchrun environment, bench.py re-executes itself under
`python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1` (one rank per GPU)
and checks that the world it gets has N ranks.  --stub replaces the CUDA step by a host stand-in
over gloo (no method arithmetic; tests the launcher, gather and timing logic on CPU).

`value`  -- device-resident path (wv_search_device into torch buffers).
`e2e`    -- the host-buffer public API (wv_search_shard): results copied D2H
            into host memory every step, wall clock, max over ranks.
`roofline` -- the dominant kernel via the library's CUDA-event stats hook: executed
            modular products per second against the measured product ceiling of the same
            arithmetic (profiles/r2_alu_peaks.json, microbenchmark on B200); the SURVEY 8(d)
            method rate (BB30/EE33-equivalent mulmods/s) and the ncu pipe fractions of the
            committed profile are reported beside it.
`frontier` -- second leg: the FP64 engine (class 1) on a C5 sub-window, one window per rank
            (weak scaling, the paper's own deployment P:L733), fp64-pipe roofline.
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
# Products per executed term of each engine ("Sums of inverses in K-term steps"):
# a K-term step costs 3 modular products (a1 <- a1 D + a0 N, a0 <- a0 D; D, N by finite differences).
#   class 0 (p < 2^30): Mont32, K = 4                 -> 3/4
#   class 1 (2^30 <= p < 2^44): exact FP64 EFT, K = 6 -> 3/6 (6 DP ops per product)
#   class 2 (p >= 2^44): Mont64, one term per step    -> 2
PRODUCTS_PER_TERM = {0: 3 / 4, 1: 3 / 6, 2: 2.0}
# FP64 engine: DP-pipe ops per term (3 products x 6 + 1 + table adds + range reductions per six terms,
# 9 for e = 2, 10 for e = 3)
DP_OPS_PER_TERM = {1: 10.0, 2: 9.0}
ALU_PEAKS = os.path.join(ROOT, "profiles", "r2_alu_peaks.json")


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


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(n):
    """--gpus N > 1 without a torchrun environment: run N ranks (one per GPU) and return their exit code."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")            # communicator / transport lines on stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def _alu_peaks():
    try:
        with open(ALU_PEAKS) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def _ncu_summary(path):
    """Pipe fractions and DRAM bytes of a committed ncu --set full summary (scripts/ncu_summary.py)."""
    if not os.path.exists(path):
        return None
    out = {}
    keys = {"issue slots busy %": "issue", "fmaheavy pipe cycles %": "fmaheavy", "alu pipe cycles %": "alu",
            "fp64 pipe cycles %": "fp64", "fma pipe cycles %": "fma"}
    rd = wr = None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for line in open(path):
        t = line.strip()
        for k, v in keys.items():
            if t.startswith(k):
                out[v] = float(t[len(k):].split()[0]) / 100
        f = t.split()
        if t.startswith("dram bytes read"):
            rd = float(f[3]) * scale.get(f[4], 1)
        if t.startswith("dram bytes write"):
            wr = float(f[3]) * scale.get(f[4], 1)
        if t.startswith("mul opcode share"):
            out["mul_opcode_share"] = float(f[3])
    out["traffic"] = rd + wr if rd is not None and wr is not None else None
    out["source"] = os.path.relpath(path, ROOT)
    return out


def _stub_step(w, rank, world):
    """--stub: a host stand-in for one rank's step (the shard's block list from the same partition the
    library uses, and a stand-in 'checksum' of the block bounds); no method arithmetic, no GPU."""
    from paper_2101_11157_b200.sweep import blocks_of
    blocks = blocks_of(w.lo, w.hi, 1 << 17, rank, world)
    chk = 0
    for a, b in blocks:
        chk = (chk + a * 0x9E3779B97F4A7C15 + b) & ((1 << 64) - 1)
    return sum(b - a for a, b in blocks), chk


def run_stub(args, w, rank, world):
    """CPU/gloo run of the launcher + gather + max-over-ranks logic (tests/test_bench_launcher.py)."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    ts = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        n, chk = _stub_step(w, rank, world)
        if i >= args.warmup:
            ts.append(time.perf_counter() - t0)
    t = torch.tensor([sum(ts) / len(ts), float(n)], dtype=torch.float64)
    if world > 1:
        from paper_2101_11157_b200.dist import gather_results
        import numpy as np
        from paper_2101_11157_b200 import _wv
        _, _, chk_all = gather_results(np.zeros(0, dtype=_wv.HIT_DTYPE), None, chk)
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(t)
        dt, n_all = float(mx[0]), int(t[1])
    else:
        chk_all, dt, n_all = chk, float(t[0]), n
    if rank == 0:
        whole = _stub_step(w, 0, 1)
        print(json.dumps({"metric": METRIC, "value": n_all / dt if dt else None, "unit": "integers/s (stub)",
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "stub": True,
                          "config": {"workload": w.name, "integers": n_all, "checksum": str(chk_all),
                                     "checksum_unsharded": str(whole[1]),
                                     "checksum_matches_unsharded": chk_all == whole[1]}}), flush=True)
    if world > 1:
        dist.destroy_process_group()


FRONTIER = ("c5_frontier", 39 * 10 ** 9, 1 << 15)    # name, window start, integers per rank


def frontier_leg(args, wv, dev, rank, world, stream, flush):
    """The FP64 engine (class 1) at the C5 frontier: rank r takes [lo + r*W, lo + (r+1)*W) (weak scaling),
    W+V, CUDA events per step on the launching stream, its own clocks and an fp64-pipe roofline."""
    import torch
    import torch.distributed as dist
    name, base, width = FRONTIER
    lo = base + rank * width
    ds = wv.DeviceSearch(lo, lo + width, 3, device=dev)
    clocks = ClockSampler([torch.cuda.current_device()] if rank == 0 else [])
    if rank == 0:
        clocks.start()
    for _ in range(args.frontier_warmup):
        ds.run(stream)
    torch.cuda.synchronize()
    wv.stats_reset()
    wv.stats_enable(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark_start()
    evs = []
    for _ in range(args.frontier_steps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ds.run(stream)
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    clocks.mark_end()
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if rank == 0 else None
    wv.stats_enable(False)
    st = wv.stats()
    ms = sum(a.elapsed_time(b) for a, b in evs) / args.frontier_steps
    k = args.frontier_steps
    pr = ds.primes[: ds.n_primes]
    sum_p = float(pr.double().sum().item())
    v = torch.tensor([ms, float(ds.n_primes), sum_p, st["terms_fp"] / k, st["residue_fp_ms"] / k],
                     dtype=torch.float64, device=dev)
    mx = v.clone()
    if world > 1:
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(v)
    ms_max, n_all, sum_p, terms, k_ms_max = float(mx[0]), int(v[1]), float(v[2]), float(v[3]), float(mx[4])
    k_ms_rank0 = st["residue_fp_ms"] / k
    peaks, _ = _peaks()
    alu = _alu_peaks()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    mhz = float(peaks.get("sm_max_mhz", 1965.0))
    dp_peak = (alu["dfma_per_clk_sm"] * sms * mhz * 1e6) if alu and alu.get("dfma_per_clk_sm") else 64 * sms * mhz * 1e6
    terms_rank = st["terms_fp"] / k
    roof = {"bound": "alu", "pipe": "fp64", "unit": "GDPop/s",
            "kernel": "residue_kernel<Mont64,1,1,6,6> (class 1 FP64 engine, six-term steps)",
            "achieved": terms_rank * (DP_OPS_PER_TERM[1] + DP_OPS_PER_TERM[2]) / 2 / (k_ms_rank0 / 1e3) / 1e9
            if k_ms_rank0 else None,
            "peak": dp_peak / 1e9,
            "peak_basis": ("measured DFMA rate (profiles/r2_alu_peaks.json)" if alu and alu.get("dfma_per_clk_sm")
                           else "guide: 64 DFMA/clk/SM") + f" x {sms} SMs x {mhz:.0f} MHz",
            "achieved_basis": "executed terms x DP-pipe ops per term of the six-term FP64 step (10 W / 9 V, "
                              "DESIGN.md section 5) / the kernel's CUDA-event time (rank 0)",
            "products_per_s": terms_rank * PRODUCTS_PER_TERM[1] / (k_ms_rank0 / 1e3) if k_ms_rank0 else None,
            "kernel_ms_per_step": k_ms_rank0, "kernel_share_of_step": k_ms_rank0 / ms if ms else None,
            "terms_per_s": terms_rank / (k_ms_rank0 / 1e3) if k_ms_rank0 else None,
            "ncu": _ncu_summary(os.path.join(ROOT, "profiles", "r2_c5s_residue_kernel_full.txt"))
            or _ncu_summary(os.path.join(ROOT, "profiles", "r1_c5s_residue_kernel_full.txt"))}
    roof["frac"] = roof["achieved"] / roof["peak"] if roof["achieved"] else None
    alg = 2 * sum(TERMS_PER_P[t] * sum_p for t in (1, 2))
    return {"metric": METRIC, "value": n_all / (ms_max / 1e3), "unit": UNIT, "ms_per_step": ms_max,
            "steps": args.frontier_steps, "warmup": args.frontier_warmup, "scaling": "weak", "dtype": "f64",
            "config": {"workload": name, "window_rank0": [base, base + width], "integers_per_rank": width,
                       "mode": "W+V", "primes": n_all, "ranks": world,
                       "partition": "rank r: [3.9e10 + r*2^15, 3.9e10 + (r+1)*2^15) (independent windows, P:L733)",
                       "l2_flush": "256 MiB write between timed steps (outside the CUDA events)"},
            "method_rate_gmulmod_s": alg / (ms_max / 1e3) / 1e9,
            "terms_per_step": terms, "roofline": roof, "clocks": clk}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-sample", type=int, default=2048, help="primes in the oracle's bounded sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--frontier-steps", type=int, default=3, help="timed steps of the frontier leg (0: skip)")
    ap.add_argument("--frontier-warmup", type=int, default=1)
    ap.add_argument("--stub", action="store_true", help="CPU/gloo stand-in step (launcher tests)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    env_world = "WORLD_SIZE" in os.environ
    world = _env_int("WORLD_SIZE", 1)
    if args.gpus is None:
        args.gpus = world
    if args.gpus > 1 and not env_world:
        sys.exit(relaunch_under_torchrun(args.gpus))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} ranks")
    if args.impl == "reference":
        return run_reference(args)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    w = _window(args.workload)
    if args.stub:
        return run_stub(args, w, rank, world)

    import torch
    import torch.distributed as dist
    import paper_2101_11157_b200 as wv

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    ds = wv.DeviceSearch(w.lo, w.hi, w.mode, shard=rank, nshards=world, device=dev)
    ds.run(torch.cuda.current_stream(dev))             # untimed: the prime and hit counts of this window
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def gather(ds):
        """Per-rank hits/checksum -> all ranks (dist.gather_results over NCCL; gloo-tested on CPU)."""
        from paper_2101_11157_b200.dist import gather_results
        return gather_results(ds.hits_np(), None, ds.checksum_int(), device=dev)

    def step():
        if world > 1:
            ds.run(stream)
            return gather(ds)
        ds.run(stream, hit_count=False, prime_count=False)   # N = 1: the host needs no count inside the step
        return None

    clocks = ClockSampler([local] if rank == 0 else [])
    if rank == 0:
        clocks.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = wv.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark_start()
    evs = []
    out = None
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
    launches = wv.launch_count() - launches0           # our kernels inside the timed region
    # kernel-level numbers (CUDA events around every residue launch, executed-term counters) from a second,
    # untimed pass of K steps: the stats hook adds events and a synchronisation, so it stays out of `value`
    wv.stats_reset()
    wv.stats_enable(True)
    for _ in range(args.steps):
        flush.fill_(1)
        step()
    torch.cuda.synchronize()
    wv.stats_enable(False)
    st = wv.stats()
    ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        n_tot = torch.tensor([ds.n_primes], dtype=torch.int64, device=dev)
        dist.all_reduce(n_tot)
        n_all = int(n_tot.item())
        checksum = out[2]
    else:
        n_all = ds.n_primes
        checksum = ds.checksum_int()
        ds.run(stream)                                  # once more with the hit count, outside the timing
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

    # checksum of the gathered shards against one unsharded pass (rank 0, outside every timed region)
    chk_whole = None
    if world > 1 and rank == 0:
        whole = wv.DeviceSearch(w.lo, w.hi, w.mode, device=dev).run(stream)
        chk_whole = whole.checksum_int()
        del whole

    frontier = None
    if args.frontier_steps > 0:
        frontier = frontier_leg(args, wv, dev, rank, world, stream, flush)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # roofline of the dominant kernel: the residue kernel of the class with the most device time
    peaks, peak_kind = _peaks()
    alu = _alu_peaks()
    steps = args.steps
    cls_terms = {0: st["terms32"] / steps, 1: st["terms_fp"] / steps,
                 2: (st["terms"] - st["terms32"] - st["terms_fp"]) / steps}
    cls_ms = {0: st["residue32_ms"] / steps, 1: st["residue_fp_ms"] / steps,
              2: (st["residue_ms"] - st["residue32_ms"] - st["residue_fp_ms"]) / steps}
    cls = max(cls_ms, key=lambda c: cls_ms[c])
    k_terms, k_ms = cls_terms[cls], cls_ms[cls]
    mhz = float(peaks.get("sm_max_mhz", 1965.0))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    # SURVEY 8(d) method rate: 2 mulmods x (227/6480 p [W] + 27/512 p [V]) over the primes of the dominant
    # kernel's class / that kernel's time -- BB30/EE33-equivalent work, which the generated congruences and
    # K-term steps do with fewer products, so it is reported as a rate, never against a peak
    pr = ds.primes[: ds.n_primes]
    lim = {0: (0, 1 << 30), 1: (1 << 30, 1 << 44), 2: (1 << 44, 1 << 62)}[cls]
    sel = pr[(pr >= lim[0]) & (pr < lim[1])]
    sum_p = float(sel.double().sum().item()) if sel.numel() else 0.0
    alg_terms = sum(TERMS_PER_P[t] * sum_p for t in (1, 2) if w.mode & t)
    method_rate = MULMODS_PER_TERM * alg_terms / (k_ms / 1e3) if k_ms > 0 else 0.0
    # achieved: executed modular products / s (3 per K-term step) against the measured product ceiling
    products = PRODUCTS_PER_TERM[cls] * k_terms / (k_ms / 1e3) if k_ms > 0 else 0.0
    key = {0: "mont32_product_per_clk_sm", 1: "dfma_per_clk_sm", 2: "mont64_product_per_clk_sm"}[cls]
    if alu and alu.get(key):
        per_clk = alu[key] / (6 if cls == 1 else 1)
        peak = per_clk * sms * mhz * 1e6
        peak_basis = (f"measured {key} = {alu[key]:.2f}/clk/SM (profiles/r2_alu_peaks.json)"
                      + (" / 6 DP ops per product" if cls == 1 else "") + f" x {sms} SMs x {mhz:.0f} MHz")
    else:
        slots = {0: 5, 1: 6, 2: 22}[cls]
        peak = 64 * sms * mhz * 1e6 / slots
        peak_basis = f"guide: 64 lanes/clk/SM x {sms} SMs x {mhz:.0f} MHz / {slots} pipe slots per product (no measured peak)"
    kname = {0: "residue_lane2_kernel (class 0 lane mode, p < 2^30)", 1: "residue_kernel<Mont64, FP64 engine> (class 1)",
             2: "residue_kernel<Mont64> (class 2, p >= 2^44)"}[cls]
    ncu = _ncu_summary(os.path.join(ROOT, "profiles", f"r2_{args.workload}_residue_kernel_full.txt")) \
        or _ncu_summary(os.path.join(ROOT, "profiles", f"r1_{args.workload}_residue_kernel_full.txt"))
    roof = {"bound": "alu", "kernel": kname, "unit": "Gmulmod/s",
            "achieved": products / 1e9, "peak": peak / 1e9, "frac": products / peak if peak else None,
            "achieved_basis": f"executed modular products: {PRODUCTS_PER_TERM[cls]:.3g} per executed term "
                              f"(K-term steps) x terms counted by the kernel / its CUDA-event time",
            "peak_basis": peak_basis,
            "traffic": ncu.get("traffic") if ncu else None,
            "traffic_unit": "bytes/launch (DRAM read+write, ncu --set full, profiles/)",
            "method_rate_gmulmod_s": method_rate / 1e9,
            "method_rate_basis": "SURVEY.md 8(d): 2 mulmods x (227/6480 p + 27/512 p) per prime (BB30/EE33-"
                                 "equivalent work; the method does less, so this is a rate, not a pipe fraction)",
            "ncu_pipes": ncu,
            "note": ("products are one part of the loop: it also advances the difference tables by modular adds, "
                     "and is bound by the FMA-heavy and ALU pipes together (ncu_pipes); frac is executed products "
                     "against the measured product-only rate" if cls == 0 else None),
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
                       "checksum": str(checksum),
                       "checksum_matches_unsharded": (checksum == chk_whole) if chk_whole is not None else None,
                       "terms_per_step": sum(cls_terms.values()),
                       "products_per_s": sum(PRODUCTS_PER_TERM[c] * cls_terms[c] for c in cls_terms) / (ms_max / 1e3)},
            "roofline": roof, "frontier": frontier, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
