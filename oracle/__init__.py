"""CPU oracle for the Wolstenholme / Vandiver residues -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  The
product (``paper_2101_11157_b200``) never imports it and shares no code with
it.  The arithmetic lives in ``wv_oracle.c`` (plain C, exact integers); this
module only compiles/loads it and marshals arguments.

Tiers (see wv_oracle.c for the cited passages):

* tier A  -- definitions: Bernoulli recurrence / secant recurrence mod p,
  O(p^2), used for p <= 2000 (and in pins up to a few 10^4); it yields every
  index 2k <= p-3 at once, so it is also the oracle of the general-index census
  (``index_residues``);
* tier B  -- W: sum_{k<p} k^-2 mod p^2 (eqnWolst + Glaisher): one 64-bit word
  for p < 2^32, base-p digit pairs for 2^32 <= p < 2^62;
  V: Glaisher's quarter sum, -4 E_{p-3} == sum_{s<p/4} s^-2 (R1);
* tier C  -- cross-check pin only: Stafford-Vandiver eqnSV == eqnBB1
  (21 B_{p-3} == sum_{p/6<s<p/4} s^-3), the paper's own reduced congruence;
  never the oracle of a prime.

All functions return canonical residues in [0, p).
"""
from __future__ import annotations

import ctypes
import os
import multiprocessing
import subprocess
from concurrent.futures import ProcessPoolExecutor

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "wv_oracle.c")
_LIB = os.path.join(_HERE, "_liboracle.so")
_BAD = (1 << 64) - 1

_lib = None
# Worker processes are spawned, never forked: the callers (pytest -m gpu, smoke, bench) hold an
# initialised CUDA context, which a forked child must not inherit.
_SPAWN = multiprocessing.get_context("spawn")


def build(force: bool = False) -> str:
    """Compile wv_oracle.c into _liboracle.so with gcc (plain -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        u64 = ctypes.c_uint64
        p64 = ctypes.POINTER(ctypes.c_uint64)
        for name in ("oracle_residue_B", "oracle_residue_E", "oracle_B_harmonic", "oracle_B_glaisher",
                     "oracle_E_quarter", "oracle_quarter_sum", "oracle_B_stafford_vandiver",
                     "oracle_wolstenholme_h2", "oracle_B_harmonic_wide"):
            f = getattr(lib, name)
            f.argtypes = [u64]
            f.restype = u64
        lib.oracle_bernoulli_mod_p.argtypes = [u64, u64, p64]
        lib.oracle_bernoulli_mod_p.restype = u64
        lib.oracle_euler_mod_p.argtypes = [u64, u64, p64]
        lib.oracle_euler_mod_p.restype = u64
        lib.oracle_primes.argtypes = [u64, u64, p64, u64]
        lib.oracle_primes.restype = u64
        lib.oracle_binom_2p_1_mod_p4.argtypes = [u64, p64, p64]
        lib.oracle_binom_2p_1_mod_p4.restype = ctypes.c_int
        lib.oracle_wolstenholme_h2_wide.argtypes = [u64, p64, p64]
        lib.oracle_wolstenholme_h2_wide.restype = ctypes.c_int
        lib.oracle_p2_mul.argtypes = [u64, u64, u64, u64, u64, p64, p64]
        lib.oracle_p2_mul.restype = ctypes.c_int
        lib.oracle_invmod.argtypes = [u64, u64]
        lib.oracle_invmod.restype = u64
        lib.oracle_mulmod.argtypes = [u64, u64, u64]
        lib.oracle_mulmod.restype = u64
        _lib = lib
    return _lib


def _chk(v: int) -> int:
    if v == _BAD:
        raise ValueError("oracle: argument outside the function's domain")
    return int(v)


# ---------------------------------------------------------------- primes
def primes(lo: int, hi: int) -> list[int]:
    """All primes q with lo <= q < hi (plain segmented Eratosthenes)."""
    lib = _load()
    n = lib.oracle_primes(lo, hi, None, 0)
    buf = (ctypes.c_uint64 * max(n, 1))()
    lib.oracle_primes(lo, hi, buf, n)
    return list(buf[:n])


def prime_count(lo: int, hi: int) -> int:
    return int(_load().oracle_primes(lo, hi, None, 0))


# ---------------------------------------------------------------- tier A
def bernoulli_mod_p(p: int, n: int | None = None) -> list[int]:
    """[B_0, ..., B_n] mod p by the recurrence (n defaults to p-3)."""
    n = p - 3 if n is None else n
    buf = (ctypes.c_uint64 * (n + 1))()
    _chk(_load().oracle_bernoulli_mod_p(p, n, buf))
    return list(buf)


def euler_mod_p(p: int, twon: int | None = None) -> list[int]:
    """[E_0, E_2, ..., E_{2n}] mod p (secant convention)."""
    twon = p - 3 if twon is None else twon
    buf = (ctypes.c_uint64 * (twon // 2 + 1))()
    _chk(_load().oracle_euler_mod_p(p, twon, buf))
    return list(buf)


def B_recurrence(p: int) -> int:
    return _chk(_load().oracle_bernoulli_mod_p(p, p - 3, None))


def E_recurrence(p: int) -> int:
    return _chk(_load().oracle_euler_mod_p(p, p - 3, None))


# ---------------------------------------------------------------- tier B / C
def wolstenholme_h2(p: int) -> int:
    return _chk(_load().oracle_wolstenholme_h2(p))


def B_harmonic(p: int) -> int:
    return _chk(_load().oracle_B_harmonic(p))


def wolstenholme_h2_wide(p: int) -> int:
    """sum_{0<k<p} k^-2 mod p^2 in base-p digit arithmetic (5 <= p < 2^62)."""
    d0, d1 = ctypes.c_uint64(), ctypes.c_uint64()
    if _load().oracle_wolstenholme_h2_wide(p, ctypes.byref(d0), ctypes.byref(d1)) != 0:
        raise ValueError("oracle: p outside [5, 2^62)")
    return d0.value + d1.value * p


def B_harmonic_wide(p: int) -> int:
    return _chk(_load().oracle_B_harmonic_wide(p))


def p2_mul(a: int, b: int, p: int) -> int:
    """a*b mod p^2 through the oracle's base-p long multiplication (a, b < p^2)."""
    r0, r1 = ctypes.c_uint64(), ctypes.c_uint64()
    if _load().oracle_p2_mul(a % p, a // p, b % p, b // p, p, ctypes.byref(r0), ctypes.byref(r1)) != 0:
        raise ValueError("oracle: operands outside the digit domain")
    return r0.value + r1.value * p


def B_glaisher(p: int) -> int:
    return _chk(_load().oracle_B_glaisher(p))


def binom_2p_1_mod_p4(p: int) -> int:
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    if _load().oracle_binom_2p_1_mod_p4(p, ctypes.byref(lo), ctypes.byref(hi)) != 0:
        raise ValueError("oracle: p outside [5, 2^31)")
    return (hi.value << 64) | lo.value


def quarter_sum(p: int) -> int:
    return _chk(_load().oracle_quarter_sum(p))


def E_quarter(p: int) -> int:
    return _chk(_load().oracle_E_quarter(p))


def B_stafford_vandiver(p: int) -> int:
    return _chk(_load().oracle_B_stafford_vandiver(p))


def residue_B(p: int) -> int:
    """B_{p-3} mod p, canonical [0, p), tier by size of p."""
    return _chk(_load().oracle_residue_B(p))


def residue_E(p: int) -> int:
    """E_{p-3} mod p (secant convention), canonical [0, p)."""
    return _chk(_load().oracle_residue_E(p))


def symres(r: int, p: int) -> int:
    """Symmetric representative in (-p/2, p/2]."""
    return r - p if r > (p - 1) // 2 else r


# ---------------------------------------------------------------- batch driver
def _one(args):
    p, mode = args
    w = residue_B(p) if mode & 1 else None
    v = residue_E(p) if mode & 2 else None
    return p, w, v


def residues(plist, mode: int = 3, workers: int | None = None):
    """[(p, B_{p-3} mod p or None, E_{p-3} mod p or None)] for each p, one prime per task."""
    plist = list(plist)
    workers = workers or os.cpu_count() or 1
    if workers == 1 or len(plist) < 2:
        return [_one((p, mode)) for p in plist]
    _load()
    with ProcessPoolExecutor(max_workers=workers, mp_context=_SPAWN) as ex:
        return list(ex.map(_one, [(p, mode) for p in plist], chunksize=max(1, len(plist) // (workers * 16))))


# ---------------------------------------------------------------- general indices (NEXT-3)
def index_residues(p: int):
    """Tier A for every even index (the irregular-pair census): lists
    (index, B_index mod p, E_index mod p) for index = 2, 4, ..., p-3, straight from the
    recurrences of the generating functions (bernoulli_mod_p / euler_mod_p)."""
    B = bernoulli_mod_p(p, p - 3)
    E = euler_mod_p(p, p - 3)
    return [(i, B[i], E[i // 2]) for i in range(2, p - 2, 2)]


def _index_one(p):
    return p, index_residues(p)


def index_residues_many(plist, workers: int | None = None):
    """{p: index_residues(p)} over a list of primes (process pool)."""
    plist = list(plist)
    workers = workers or os.cpu_count() or 1
    if workers == 1 or len(plist) < 2:
        return dict(_index_one(p) for p in plist)
    _load()
    with ProcessPoolExecutor(max_workers=workers, mp_context=_SPAWN) as ex:
        return dict(ex.map(_index_one, plist, chunksize=1))


def irregular_pairs(p: int):
    """([2k: p | B_2k], [2k: p | E_2k]) for 2 <= 2k <= p-3 ((E-)irregular pairs)."""
    r = index_residues(p)
    return [i for i, b, _ in r if b == 0], [i for i, _, e in r if e == 0]
