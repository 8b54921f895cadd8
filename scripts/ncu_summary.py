#!/usr/bin/env python3
"""Summarise ncu artefacts for profiles/ (run here, no GPU needed).
   ncu_summary.py rep  <file.ncu-rep>          -> key metrics of each profiled kernel
   ncu_summary.py launches <launches.csv>      -> per-kernel device time and share of the run"""
import csv, io, subprocess, sys, collections

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy pipe cycles %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe cycles %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu pipe cycles %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe cycles %"),
    ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "shared pipe cycles %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 inst %"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps/cycle"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads/warp-instr"),
    ("dram__bytes_read.sum", "dram bytes read"),
    ("dram__bytes_write.sum", "dram bytes write"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math_pipe_throttle"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall not_selected"),
    ("smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio", "stall dispatch"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard"),
]


MUL_OPS = ("IMAD.WIDE", "IMAD.HI", "IMAD", "IMUL")     # integer multiplies (IMAD.IADD / IMAD.MOV / IMAD.X excluded)
STALLS = ("math", "not_selected", "selected", "wait", "dispatch", "no_inst", "short_sb", "long_sb", "mio",
          "branch_resolving")


def opcode_mix(path):
    """Executed SASS instructions per opcode (ncu source page) and stall-sample shares of the first kernel."""
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return None, None
    hdr = rows[1]
    H = {h: i for i, h in enumerate(hdr)}
    ex, st = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        w = r[H["Source"]].split()
        if not w:
            continue
        op = w[1] if w[0].startswith("@") else w[0]
        ex[op] += int(r[H["Instructions Executed"]] or 0)
        for k in STALLS:
            col = "stall_" + k
            if col in H:
                st[k] += int(r[H[col]] or 0)
    return ex, st


def mul_share(ex):
    tot = sum(ex.values())
    mul = sum(c for op, c in ex.items() if op in ("IMAD", "IMUL") or op.startswith(("IMAD.WIDE", "IMAD.HI")))
    return mul, tot


def rep(path):
    ex, st = opcode_mix(path)
    _rep_raw(path)
    if ex:
        mul, tot = mul_share(ex)
        print(f"  {'warp instructions executed':32s} {tot}")
        print(f"  {'mul opcode share':32s} {mul / tot:.4f} (IMAD, IMAD.WIDE, IMAD.HI, IMUL of all executed SASS)")
        print("  opcode mix: " + ", ".join(f"{op} {c / tot:.3f}" for op, c in ex.most_common(12)))
        stot = sum(st.values())
        if stot:
            print("  stall samples: " + ", ".join(f"{k} {v / stot:.2f}" for k, v in st.most_common(8)))


def _rep_raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        print(f"kernel: {d.get('Kernel Name', '?')[:140]}")
        for k, label in KEYS:
            if k in d and d[k] != "":
                print(f"  {label:32s} {d[k]} {u.get(k, '')}")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[1:]:
        if len(r) <= vi or r[ki] == "Kernel Name":
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[ui], 1e-6)
        name = r[ki].split("(")[0][:90]
        tot[name] += v * scale
        cnt[name] += 1
    all_ms = sum(tot.values())
    print(f"{'kernel':92s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
    for name, ms in tot.most_common():
        print(f"{name:92s} {cnt[name]:8d} {ms:10.3f} {100 * ms / all_ms:6.2f}%")
    print(f"{'TOTAL':92s} {sum(cnt.values()):8d} {all_ms:10.3f}")


if __name__ == "__main__":
    {"rep": rep, "launches": launches}[sys.argv[1]](sys.argv[2])
