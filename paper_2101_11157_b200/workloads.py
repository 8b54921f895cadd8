"""Workload definitions and seeded input generators (no arithmetic of the method).

This module is the one place both sides (the CUDA path's tests/bench and the
CPU oracle's golden generator) take their inputs from.  It holds window
bounds, the deterministic sampling rule and seeded random windows -- nothing
that computes a residue, a congruence bound or a prime.

Configs follow BASELINE.json ``configs`` (SURVEY.md section 8 shorthand C1..C5),
with reading R4 of DESIGN.md for C3 (its window holds no Vandiver prime; the
pin window PIN_V holds 1062232319).
"""
from __future__ import annotations

import random
from dataclasses import dataclass

MODE_W = 1
MODE_V = 2
MODE_BOTH = 3


@dataclass(frozen=True)
class Window:
    name: str
    lo: int
    hi: int
    mode: int
    note: str


CONFIGS = {
    "c1": Window("c1", 5, 10 ** 5, MODE_BOTH, "all primes 5 <= p < 10^5, both tests (BASELINE configs[0])"),
    "c2": Window("c2", 5, 3 * 10 ** 6, MODE_BOTH, "all primes p < 3*10^6, both tests (BASELINE configs[1])"),
    "c3": Window("c3", 10 ** 9, 105 * 10 ** 7, MODE_V, "[1.0e9, 1.05e9), Vandiver test (BASELINE configs[2])"),
    "c4": Window("c4", 59 * 10 ** 9, 59 * 10 ** 9 + 10 ** 7, MODE_W, "[5.9e10, 5.9e10+1e7), Wolstenholme (configs[3])"),
    "c5": Window("c5", 39 * 10 ** 9, 40 * 10 ** 9, MODE_BOTH, "[3.9e10, 4.0e10), both tests, 8 GPUs (configs[4])"),
    # reading R4: the window that actually contains the eighth Vandiver prime 1062232319
    "pin_v": Window("pin_v", 106 * 10 ** 7, 1065 * 10 ** 6, MODE_V, "[1.06e9, 1.065e9): recovers 1062232319"),
}

# Sub-windows used where a full config is too long for a test or a bench step.
SUBWINDOWS = {
    "c4_head": Window("c4_head", 59 * 10 ** 9, 59 * 10 ** 9 + 2 * 10 ** 4, MODE_W, "first 2e4 integers of C4"),
    "c5_head": Window("c5_head", 39 * 10 ** 9, 39 * 10 ** 9 + 10 ** 4, MODE_BOTH, "first 1e4 integers of C5"),
    "c5_scale": Window("c5_scale", 39 * 10 ** 9, 39 * 10 ** 9 + 4 * 10 ** 6, MODE_BOTH,
                       "first 4e6 integers of C5 (SURVEY.md 8(d) scaling sub-window)"),
    "c5_frontier": Window("c5_frontier", 39 * 10 ** 9, 39 * 10 ** 9 + (1 << 15), MODE_BOTH,
                          "bench.py frontier leg, rank 0's window (rank r: +r*2^15)"),
    "c2_probe": Window("c2_probe", 1 << 44, (1 << 44) + 60, MODE_W, "primes just above 2^44 (64-bit Montgomery class)"),
    "c3_slice": Window("c3_slice", 10 ** 9, 10 ** 9 + 5 * 10 ** 5, MODE_V, "first 5e5 integers of C3"),
    "c3_slice_both": Window("c3_slice_both", 10 ** 9, 10 ** 9 + 5 * 10 ** 5, MODE_BOTH, "first 5e5 integers of C3, W+V"),
}


def sample_indices(n: int, k: int) -> list[int]:
    """Deterministic sample of k indices out of n: floor(j*n/k)."""
    if n <= 0:
        return []
    k = min(k, n)
    return [(j * n) // k for j in range(k)]


def random_windows(seed: int, count: int, lo: int, hi: int, width_lo: int, width_hi: int):
    """Seeded random half-open windows [a, b) inside [lo, hi) (ragged sizes)."""
    rng = random.Random(seed)
    out = []
    for _ in range(count):
        w = rng.randrange(width_lo, width_hi + 1)
        a = rng.randrange(lo, max(lo + 1, hi - w))
        out.append((a, a + w))
    return out
