"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and the paper.

Bit-exact comparison of canonical residues (integer work: the bar is equality).
Inputs are the BASELINE configs (paper_2101_11157_b200.workloads) and seeded
random windows; expected values come from oracle/ (on the fly for small
windows, or tests/golden/oracle_*.npz written by scripts/gen_oracle_goldens.py)
and from the paper's printed tables (tests/golden/paper_*).
"""
import csv
import json
import os

import numpy as np
import pytest

import oracle
from paper_2101_11157_b200.workloads import CONFIGS, SUBWINDOWS, random_windows, sample_indices

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
NONE = (1 << 64) - 1


def _golden(name):
    path = os.path.join(GOLD, f"oracle_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (scripts/gen_oracle_goldens.py {name})")
    z = np.load(path)
    return z["p"], z["res_w"], z["res_v"], json.loads(str(z["meta"]))


def _table(name):
    with open(os.path.join(GOLD, name)) as f:
        return list(csv.DictReader(r for r in f if not r.startswith("#")))


def _oracle_arrays(ps, mode):
    out = oracle.residues(ps, mode)
    rw = np.array([NONE if r[1] is None else r[1] for r in out], dtype=np.uint64)
    rv = np.array([NONE if r[2] is None else r[2] for r in out], dtype=np.uint64)
    return rw, rv


def _assert_equal(p, got, want, what):
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{what}: {bad.size} mismatches, first p={p[bad[:5]].tolist()} " \
                          f"got={got[bad[:5]].tolist()} want={want[bad[:5]].tolist()}"


# ---------------------------------------------------------------- whole windows
def test_c1_full_bit_exact(wv):
    """configs[0]: every prime 5 <= p < 10^5, both tests, vs oracle goldens; hits recovered."""
    w = CONFIGS["c1"]
    hits, res = wv.search(w.lo, w.hi, w.mode)
    gp, gw, gv, meta = _golden("c1")
    assert res["p"].tolist() == gp.tolist()
    _assert_equal(gp, res["res_w"], gw, "W")
    _assert_equal(gp, res["res_v"], gv, "V")
    assert {(int(h["p"]), int(h["flags"])) for h in hits} == {(149, 2), (241, 2), (16843, 1)}


def test_c2_full_bit_exact(wv):
    """configs[1]: every prime p < 3*10^6, both tests, through the device API bench.py times."""
    w = CONFIGS["c2"]
    gp, gw, gv, meta = _golden("c2")
    ds = wv.DeviceSearch(w.lo, w.hi, w.mode).run()
    p = ds.primes_np()
    assert p.tolist() == gp.tolist()
    rw, rv = ds.res_np()
    _assert_equal(gp, rw, gw, "W")
    _assert_equal(gp, rv, gv, "V")
    hits = {(int(h["p"]), int(h["flags"])) for h in ds.hits_np()}
    assert hits == {(149, 2), (241, 2), (16843, 1), (2124679, 1), (2946901, 2)}
    want_chk = sum(wv.checksum_term(int(a), int(b), int(c)) for a, b, c in zip(gp, gw, gv)) % (1 << 64)
    assert ds.checksum_int() == want_chk


def test_random_windows_vs_oracle(wv):
    """Seeded ragged windows (several sieve segments and residue chunks, odd tails)."""
    for i, (a, b) in enumerate(random_windows(2101, 6, 5, 4 * 10 ** 6, 1, 300000)):
        mode = 1 + i % 3
        hits, res = wv.search(a, b, mode)
        ps = oracle.primes(max(a, 5), b)
        assert res["p"].tolist() == ps, (a, b)
        rw, rv = _oracle_arrays(ps, mode)
        p = np.array(ps, dtype=np.uint64)
        _assert_equal(p, res["res_w"], rw, f"W [{a},{b})")
        _assert_equal(p, res["res_v"], rv, f"V [{a},{b})")


def test_c3_full_window_sampled(wv):
    """configs[2] at full size ([1.0e9, 1.05e9), V): 64 sampled primes vs oracle goldens,
    no Vandiver prime (reading R4) and no |<E>| < 50 (Table 3 is complete)."""
    w = CONFIGS["c3"]
    gp, gw, gv, meta = _golden("c3")
    ds = wv.DeviceSearch(w.lo, w.hi, w.mode).run()
    p = ds.primes_np()
    assert len(p) == meta["primes_in_window"] == 2409816
    idx = sample_indices(len(p), 64)
    assert p[idx].tolist() == gp.tolist()
    rw, rv = ds.res_np()
    _assert_equal(gp, rv[idx], gv, "V sample")
    assert (rw == NONE).all()
    assert ds.n_hits == 0
    sym = np.where(rv > (p - 1) // 2, rv.astype(np.int64) - p.astype(np.int64), rv.astype(np.int64))
    assert int((np.abs(sym) < 50).sum()) == 0


def test_pin_window_recovers_1062232319(wv):
    w = CONFIGS["pin_v"]
    gp, gw, gv, meta = _golden("pin_v")
    hits, res = wv.search(w.lo, w.hi, w.mode)
    assert [(int(h["p"]), int(h["flags"])) for h in hits] == [(1062232319, 2)]
    d = dict(zip(res["p"].tolist(), res["res_v"].tolist()))
    assert [d[int(x)] for x in gp] == gv.tolist()


# ---------------------------------------------------------------- paper-printed values
def _sym(r, p):
    return r - p if r > (p - 1) // 2 else r


def test_table2_all_rows(wv):
    """Table 2: all 19 near misses of B_{p-3} in (1e9, 6e10), sign-exact (64-bit path)."""
    rows = _table("paper_table2_bernoulli.csv")
    ps = [int(r["p"]) for r in rows]
    rw, rv = wv.residues_of(ps, wv.MODE_W)
    for r, x in zip(rows, rw.tolist()):
        assert _sym(int(x), int(r["p"])) == int(r["symres_B"]), r


def test_table3_all_rows(wv):
    """Table 3: 11 rows exact, 7 rows |value| with the secant sign (reading R2)."""
    rows = _table("paper_table3_euler.csv")
    ps = [int(r["p"]) for r in rows]
    rw, rv = wv.residues_of(ps, wv.MODE_V)
    for r, x in zip(rows, rv.tolist()):
        v, want = _sym(int(x), int(r["p"])), int(r["symres_E"])
        if int(r["sign_exact"]):
            assert v == want, r
        else:
            assert v == -want and want != 0, r


def test_known_primes(wv):
    k = json.load(open(os.path.join(GOLD, "paper_known_primes.json")))
    ps = k["wolstenholme_below_6e10"] + k["vandiver_below_4e10"]
    rw, rv = wv.residues_of(ps, wv.MODE_BOTH)
    for p, a, b in zip(ps, rw.tolist(), rv.tolist()):
        assert (a == 0) == (p in k["wolstenholme_below_6e10"]), p
        assert (b == 0) == (p in k["vandiver_below_4e10"]), p
    rw, rv = wv.residues_of([2124679], wv.MODE_V)
    assert _sym(int(rv[0]), 2124679) == -85724         # reading R3


def test_sieve_counts_match_paper(wv):
    """The device sieve reproduces the paper's prime counts and textbook pi(x)."""
    counts = json.load(open(os.path.join(GOLD, "paper_prime_counts.json")))["counts"]
    for c in counts:
        assert wv.prime_count(max(c["lo"], 5), c["hi"]) == c["n"] - (2 if c["lo"] < 5 and c["hi"] > 3 else 0), c


# ---------------------------------------------------------------- cross-congruence / schedule
def test_every_congruence_on_gpu(wv):
    """Force each congruence (VOR12 at p >= 7) on a mixed-width unsorted list vs the oracle/paper."""
    rng = np.random.default_rng(5)
    small = oracle.primes(11, 30000)
    ps = sorted(set(rng.choice(small, 40, replace=False).tolist()) | {11, 13, 29989})
    big_w = [1025793739, 2139716869, 56604583391]       # Table 2
    big_v = [1062232319, 1836806681, 36652898767]       # Table 3 (sign-exact rows)
    conf = {c["name"]: (c["id"], c["e"]) for c in wv.congruences()}
    try:
        for name, (cid, e) in conf.items():
            e3 = e == 3
            wv.set_schedule_override(cid if e3 else -1, -1 if e3 else cid)
            lst = ps + (big_w if e3 else big_v)
            rng.shuffle(lst)
            rw, rv = wv.residues_of(lst, wv.MODE_W if e3 else wv.MODE_V)
            got = rw if e3 else rv
            for p, x in zip(lst, got.tolist()):
                want = (oracle.residue_B(p) if p < 10 ** 8 else None) if e3 else \
                       (oracle.residue_E(p) if p < 10 ** 8 else None)
                if want is None:
                    tab = {1025793739: -9, 2139716869: 2, 56604583391: -25, 1062232319: 0,
                           1836806681: -15, 36652898767: -9}
                    assert _sym(int(x), p) == tab[p], (name, p)
                else:
                    assert int(x) == want, (name, p)
    finally:
        wv.set_schedule_override(-1, -1)


# ---------------------------------------------------------------- sharding / edge cases
def test_shards_union_equals_whole(wv):
    """Interleaved blocks: union of shards == unsharded; checksums add up."""
    lo, hi = 1000, 1000 + 40 * 131072 + 777
    _, whole, chk = wv.search_shard(lo, hi, 3, 0, 1, 0)
    for nsh in (2, 3, 8):
        parts, tot = [], 0
        for s in range(nsh):
            _, r, c = wv.search_shard(lo, hi, 3, s, nsh, 131072)
            parts.append(r)
            tot = (tot + c) % (1 << 64)
        merged = np.sort(np.concatenate(parts), order="p")
        assert merged.tobytes() == whole.tobytes()
        assert tot == chk


@pytest.mark.parametrize("nsh", [8])
def test_c2_shards_bit_exact(wv, nsh):
    """The bench's N-GPU split of C2 (interleaved blocks, default block size): each shard is a small
    window, so the lane kernel cuts its groups into several slices (Q > 1); the merged residues equal
    the oracle's on every prime and the shard checksums add up to the whole window's."""
    w = CONFIGS["c2"]
    gp, gw, gv, _ = _golden("c2")
    parts, tot = [], 0
    for s in range(nsh):
        ds = wv.DeviceSearch(w.lo, w.hi, w.mode, s, nsh).run()
        rw, rv = ds.res_np()
        parts.append((ds.primes_np(), rw, rv))
        tot = (tot + ds.checksum_int()) % (1 << 64)
    p = np.concatenate([a for a, _, _ in parts])
    order = np.argsort(p, kind="stable")
    assert p[order].tolist() == gp.tolist()
    _assert_equal(gp, np.concatenate([b for _, b, _ in parts])[order], gw, "W")
    _assert_equal(gp, np.concatenate([c for _, _, c in parts])[order], gv, "V")
    want_chk = sum(wv.checksum_term(int(a), int(b), int(c)) for a, b, c in zip(gp, gw, gv)) % (1 << 64)
    assert tot == want_chk


def test_edge_windows(wv):
    h, r = wv.search(100, 101, 3)
    assert len(r) == 0 and len(h) == 0
    h, r = wv.search(0, 5, 3)
    assert len(r) == 0
    h, r = wv.search(5, 6, 3)
    assert r.tolist() == [(5, 1, 1)]
    h, r = wv.search(7, 8, 3)
    assert r.tolist() == [(7, 3, 5)]                      # B_4 = -1/30 == 3, E_4 = 5 (mod 7)
    h, r = wv.search(5, 12, 1)
    assert r["res_v"].tolist() == [NONE] * 3 and r["res_w"].tolist() == [1, 3, 4]
    for bad in [(10, 10, 3), (10, 5, 3), (5, 100, 0), (5, 100, 4), (5, (1 << 62) + 1, 3)]:
        with pytest.raises(wv.WVError):
            wv.search(*bad)
    with pytest.raises(wv.WVError):
        wv.search_shard(5, 100, 3, 2, 2, 0)


def test_ragged_tail_64bit_window(wv):
    """A small window just above 2^30 (first 64-bit primes) and one at 5.9e10 (C4 head), vs oracle."""
    a, b = (1 << 30) - 3000, (1 << 30) + 3000
    hits, res = wv.search(a, b, 3)
    ps = oracle.primes(a, b)
    assert res["p"].tolist() == ps
    sub = res[sample_indices(len(res), 4)]
    rw, rv = _oracle_arrays([int(p) for p in sub["p"]], 3)         # tier B (definition-level), p < 2^32
    _assert_equal(sub["p"], sub["res_w"], rw, "W above 2^30")
    _assert_equal(sub["p"], sub["res_v"], rv, "V above 2^30")
    w = SUBWINDOWS["c4_head"]
    hits, res = wv.search(w.lo, w.hi, w.mode)
    assert res["p"].tolist() == oracle.primes(w.lo, w.hi)
    # the C4 head's residues: every C4 oracle golden sample inside it (tier B, base-p digits)
    gp, gw, gv, _ = _golden("c4")
    inside = (gp >= w.lo) & (gp < w.hi)
    assert inside.sum() >= 1
    idx = np.searchsorted(res["p"], gp[inside])
    _assert_equal(gp[inside], res["res_w"][idx], gw[inside], "C4 head W")


def test_kernel_variants_bit_identical(wv):
    """Every residue-kernel variant (engine x streams per lane) gives the same residues:
    a window spanning the 2^30 class boundary plus Table 2/3 primes (class 1)."""
    lo, hi = (1 << 30) - 20000, (1 << 30) + 20000
    ref_h, ref_r = wv.search(lo, hi, 3)
    tab = [1025793739, 1348936931, 10158743171, 56604583391]
    ref_w, ref_v = wv.residues_of(tab, 3)
    try:
        for vid, name, cls in wv.kernel_variants():
            if cls == 2:
                continue
            wv.set_kernel_variant(cls, vid)
            h, r = wv.search(lo, hi, 3)
            assert r.tobytes() == ref_r.tobytes(), name
            rw, rv = wv.residues_of(tab, 3)
            assert rw.tolist() == ref_w.tolist() and rv.tolist() == ref_v.tolist(), name
            wv.set_kernel_variant(cls, -1)
    finally:
        for c in range(3):
            wv.set_kernel_variant(c, -1)


@pytest.mark.parametrize("items", ["0.001", "3", "1000000"])
def test_lane2_slicing_bit_exact(wv, items, monkeypatch):
    """Class-0 lane mode v2 cuts each group's sums into Q slices (one slice size per launch, from
    WV_LANE_ITEMS items per resident warp): whole sums (Q = 1) and the finest cut (Q up to 128) give the
    residues of the chunk kernel and of the oracle, on a C2-size window (both tests, p < 2^28) and a
    window above 2^28 (the lazy-subtract variant of the pair step)."""
    ids = {name: vid for vid, name, cls in wv.kernel_variants()}
    windows = [(5, 300000, 3), ((1 << 28) - 3000, (1 << 28) + 3000, 3), (10 ** 9, 10 ** 9 + 6000, 2)]
    try:
        for lo, hi, mode in windows:
            wv.set_kernel_variant(0, ids["c0 int s2/2 pairs"])
            _, ref = wv.search(lo, hi, mode)
            wv.set_kernel_variant(0, ids["c0 lane2"])
            monkeypatch.setenv("WV_LANE_ITEMS", items)
            _, got = wv.search(lo, hi, mode)
            monkeypatch.delenv("WV_LANE_ITEMS")
            assert got.tobytes() == ref.tobytes(), (lo, hi, items)
            ps = got["p"].tolist()
            idx = sample_indices(len(ps), 48)
            rw, rv = _oracle_arrays([ps[i] for i in idx], mode)
            _assert_equal(got["p"][idx], got["res_w"][idx], rw, f"W [{lo},{hi})")
            _assert_equal(got["p"][idx], got["res_v"][idx], rv, f"V [{lo},{hi})")
    finally:
        wv.set_kernel_variant(0, -1)


@pytest.mark.parametrize("chain", ["0", "1", "4"])
def test_lane2_chain_modes_bit_exact(wv, chain, monkeypatch):
    """Chain mode (one table and one accumulator through adjacent sums, summation by parts) is on by default
    (e = 2 and e = 3 four-term steps: WV_LANE_CHAIN = 5); no chains with W pair steps (0), e = 2 only (1) and
    e = 3 only (4) must give the same residues on windows where sums are a few terms long (BB30 / EE33 just
    above 4096: empty, one- and two-term sums), on a C2-size window and on windows straddling 2^23 and the
    tier bound 2^24, and agree with the oracle."""
    windows = [(4000, 9000, 3), (5, 300000, 3), ((1 << 23) - 6000, (1 << 23) + 6000, 3),
               ((1 << 24) - 4000, (1 << 24) + 4000, 3)]
    for lo, hi, mode in windows:
        _, ref = wv.search(lo, hi, mode)
        monkeypatch.setenv("WV_LANE_CHAIN", chain)
        _, got = wv.search(lo, hi, mode)
        monkeypatch.delenv("WV_LANE_CHAIN")
        assert got.tobytes() == ref.tobytes(), (lo, hi, chain)
    ps = got["p"].tolist()
    idx = sample_indices(len(ps), 32)
    rw, rv = _oracle_arrays([ps[i] for i in idx], 3)
    _assert_equal(got["p"][idx], got["res_w"][idx], rw, "W")
    _assert_equal(got["p"][idx], got["res_v"][idx], rv, "V")


def test_class2_64bit_montgomery_cross_congruence(wv):
    """p >= 2^44 runs the 64-bit Montgomery engine: two different congruences agree
    (BB1 vs BB30 for W, EE3 vs EE33 for V) on a prime just above 2^44 (property check)."""
    p = 17592186044423          # smallest prime > 2^44
    names = {c["name"]: c["id"] for c in wv.congruences()}
    out = {}
    try:
        for w, v in [("BB1", "EE3"), ("BB30", "EE33")]:
            wv.set_schedule_override(names[w], names[v])
            rw, rv = wv.residues_of([p], 3)
            out[w] = (int(rw[0]), int(rv[0]))
    finally:
        wv.set_schedule_override(-1, -1)
    assert out["BB1"] == out["BB30"]
    assert 0 <= out["BB1"][0] < p and 0 <= out["BB1"][1] < p
    # the default class-2 engine (Mont64 eight-term steps with lazy tables, BG_BIG / EG_BIG) against the
    # term-by-term Mont64 engine, on the default schedule, for two primes above 2^44
    ids = {name: vid for vid, name, cls in wv.kernel_variants()}
    ps = [p, 17592186044437]                  # the two smallest primes above 2^44
    dw, dv = wv.residues_of(ps, 3)
    try:
        wv.set_kernel_variant(2, ids["c2 int s1/1"])
        sw, sv = wv.residues_of(ps, 3)
    finally:
        wv.set_kernel_variant(2, -1)
    assert dw.tolist() == sw.tolist() and dv.tolist() == sv.tolist()
    assert (int(dw[0]), int(dv[0])) == out["BB1"]


def test_fp64_tuple_steps_near_class_top(wv):
    """The FP64 engine's six-term steps range-reduce their difference tables every rb steps, rb the
    largest with p sum_{i<=Ke} C(rb, i) <= 2^49: smallest just below 2^44.  Primes there (and a few
    ragged ones at C4 size) must give the term-by-term FP64 variant's residues, and BIG-tier residues
    must equal those of the paper's printed congruences BB30 / EE33 (non-sum-aligned, term by term)."""
    ids = {name: vid for vid, name, cls in wv.kernel_variants()}
    names = {c["name"]: c["id"] for c in wv.congruences()}
    ps = [17592186044399, 17592186044297, 59000000023, 59000000149]   # < 2^44 (largest class-1 p); C4 size
    try:
        wv.set_kernel_variant(1, ids["c1 fp tuples 6/6"])
        tw, tv = wv.residues_of(ps, 3)
        wv.set_kernel_variant(1, ids["c1 fp s2/2"])
        sw, sv = wv.residues_of(ps, 3)
        assert tw.tolist() == sw.tolist() and tv.tolist() == sv.tolist()
        # the 64-bit Montgomery engine (the class-2 arithmetic) on the same primes: IMAD pipe, not FP64
        wv.set_kernel_variant(1, ids["c1 int s1/1"])
        mw, mv = wv.residues_of(ps, 3)
        assert mw.tolist() == tw.tolist() and mv.tolist() == tv.tolist()
        wv.set_kernel_variant(1, -1)
        wv.set_schedule_override(names["BB30"], names["EE33"])
        pw, pv = wv.residues_of(ps[2:], 3)
        assert pw.tolist() == tw[2:].tolist() and pv.tolist() == tv[2:].tolist()
    finally:
        wv.set_schedule_override(-1, -1)
        wv.set_kernel_variant(1, -1)


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_c4_c5_sampled_primes(wv, name):
    """configs[3], configs[4]: the oracle's deterministic 8-prime samples of the full windows
    (p ~ 5.9e10 and 3.9e10: the FP64-engine class), bit-exact; also through the sieve path
    on the first sample's neighbourhood."""
    gp, gw, gv, meta = _golden(name)
    w = CONFIGS[name]
    rw, rv = wv.residues_of(gp.tolist(), w.mode)
    if w.mode & 1:
        _assert_equal(gp, rw, gw, f"{name} W")
    if w.mode & 2:
        _assert_equal(gp, rv, gv, f"{name} V")
    p0 = int(gp[0])
    hits, res = wv.search(p0, p0 + 1, w.mode)
    assert res["p"].tolist() == [p0]
    assert (int(res["res_w"][0]) if w.mode & 1 else NONE) == int(gw[0])


@pytest.mark.gpu
def test_coarse_seg_index_fallback(wv):
    """Sum-aligned (> 96-sum) congruences locate a chunk's sum through a coarse per-record index
    sized by the workspace.  The C4/C5 samples (BG_BIG / EG_BIG, ~3500 sums) with a workspace for
    primes <= 2^30 (no room for their index: every record scans its sums) and with the full
    index give the same, oracle-exact residues."""
    import torch
    for name in ("c4", "c5"):
        gp, gw, gv, meta = _golden(name)
        w = CONFIGS[name]
        t = torch.tensor(gp.astype(np.int64), device="cuda")
        small = [x.cpu().numpy().view(np.uint64) for x in wv.residues_device(t, w.mode, max_p=1 << 30)]
        full = [x.cpu().numpy().view(np.uint64) for x in wv.residues_device(t, w.mode)]
        for got in (small, full):
            if w.mode & 1:
                _assert_equal(gp, got[0], gw, f"{name} W")
            if w.mode & 2:
                _assert_equal(gp, got[1], gv, f"{name} V")


# ---------------------------------------------------------------- NEXT-1: near misses and histograms
def _near_window(wv, lo, hi, mode, bound=50):
    ds = wv.DeviceSearch(lo, hi, mode).run()
    near, hw, hv = ds.near_misses(bound)
    return ds, {(int(x["p"]), int(x["test"])): int(x["symres"]) for x in near}, hw, hv


TABLE_WINDOWS = [
    # (center, half-width, mode): Tables 2 and 3 are complete on (1e9, 6e10) / (1e9, 4e10),
    # so a window around a listed prime must contain exactly the listed near misses
    (2139716869, 100000, 1), (56604583391, 30000, 1), (1836806681, 100000, 2), (36830964851, 20000, 2),
]


@pytest.mark.parametrize("center,half,mode", TABLE_WINDOWS)
def test_near_misses_match_complete_tables(wv, center, half, mode):
    t2 = {int(r["p"]): int(r["symres_B"]) for r in _table("paper_table2_bernoulli.csv")}
    t3 = {int(r["p"]): (int(r["symres_E"]), int(r["sign_exact"])) for r in _table("paper_table3_euler.csv")}
    lo, hi = center - half, center + half
    ds, near, hw, hv = _near_window(wv, lo, hi, mode)
    if mode == 1:
        want = {(p, 1): v for p, v in t2.items() if lo <= p < hi}
    else:
        want = {(p, 2): (v if ex else -v) for p, (v, ex) in t3.items() if lo <= p < hi}   # reading R2
    assert near == want
    hist = hw if mode == 1 else hv
    assert int(hist.sum()) == ds.n_primes


def test_near_misses_pin_window_and_c2_histograms(wv):
    w = CONFIGS["pin_v"]
    ds, near, hw, hv = _near_window(wv, w.lo, w.hi, w.mode)
    assert near == {(1062232319, 2): 0}
    w = CONFIGS["c2"]
    ds, near, hw, hv = _near_window(wv, w.lo, w.hi, w.mode)
    p = ds.primes_np().astype(object)
    rw, rv = ds.res_np()
    for res, hist, test in ((rw, hw, 1), (rv, hv, 2)):
        r = res.astype(object)
        sym = [int(a) - int(q) if int(a) > (int(q) - 1) // 2 else int(a) for a, q in zip(r, p)]
        bins = np.bincount([(2 * s + int(q)) * 1000 // int(q) for s, q in zip(sym, p)], minlength=2000)
        assert bins.tolist() == hist.tolist()
        small = {(int(q), test): s for s, q in zip(sym, p) if abs(s) < 50}
        assert {k: v for k, v in near.items() if k[1] == test} == small


def test_c3_wolstenholme_near_misses_table2(wv):
    """configs[2] window in W mode: Table 2 lists exactly 1025793739 (-9) and 1029113299 (-7) there
    (table complete on (1e9, 6e10)); the histogram is flat (Fig. 1)."""
    w = CONFIGS["c3"]
    ds, near, hw, hv = _near_window(wv, w.lo, w.hi, 1)
    assert near == {(1025793739, 1): -9, (1029113299, 1): -7}
    n = ds.n_primes
    exp = n / 2000
    chi2 = float((((hw.astype(np.float64) - exp) ** 2) / exp).sum())
    assert 1700 < chi2 < 2300            # 1999 degrees of freedom


def test_bench_contract_line():
    """bench.py (the driver's contract) runs on the GPU and prints one well-formed JSON line."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--steps", "3", "--warmup", "3",
                          "--ref-sample", "64"], capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in line, k
    assert line["value"] > 1e5 and line["config"]["primes"] == 216814
    assert 0 < line["roofline"]["frac"] <= 1.5 and line["gpu_launches"] > 0
    assert line["e2e"]["d2h_bytes_per_step"] > 0 and line["cpu_baseline"]["kind"] == "oracle"


def test_frontier_window_primes_and_samples(wv):
    """bench.py's frontier leg (C5 sub-window [3.9e10, 3.9e10 + 2^15), the FP64 engine): its prime list
    equals the oracle's sieve, and every C5 oracle golden sample inside it is reproduced bit-exactly
    through the same DeviceSearch path the bench times."""
    w = SUBWINDOWS["c5_frontier"]
    ds = wv.DeviceSearch(w.lo, w.hi, w.mode).run()
    got = ds.primes_np()
    assert got.tolist() == oracle.primes(w.lo, w.hi)
    rw, rv = ds.res_np()
    gp, gw, gv, _ = _golden("c5")
    inside = (gp >= w.lo) & (gp < w.hi)
    assert inside.sum() >= 1
    idx = np.searchsorted(got, gp[inside])
    _assert_equal(gp[inside], rw[idx], gw[inside], "frontier W")
    _assert_equal(gp[inside], rv[idx], gv[inside], "frontier V")



def test_wv_search_symbol_and_enospc_two_call(wv):
    """wv_search itself (not wv_search_shard): the two-call contract of include/wv.h -- too-small capacities
    give WV_ENOSPC with *n_hits / *n_primes set to the sizes needed and nothing written; a second call with
    those sizes succeeds and equals wv_search_shard; residues may be skipped (NULL, cap 0)."""
    from paper_2101_11157_b200 import _wv
    w = CONFIGS["c1"]
    sh, sr, _ = wv.search_shard(w.lo, w.hi, w.mode, 0, 1, 0)
    hits = np.zeros(1, dtype=_wv.HIT_DTYPE)
    res = np.zeros(10, dtype=_wv.RES_DTYPE)
    hits["p"] = 12345
    rc, nh, npr = _wv.search_raw(w.lo, w.hi, w.mode, hits, res)
    assert rc == _wv.WV_ENOSPC and (nh, npr) == (3, 9590)
    assert int(hits["p"][0]) == 12345 and not res["p"].any()          # nothing written
    hits = np.zeros(nh, dtype=_wv.HIT_DTYPE)
    res = np.zeros(npr, dtype=_wv.RES_DTYPE)
    rc, nh2, npr2 = _wv.search_raw(w.lo, w.hi, w.mode, hits, res)
    assert rc == _wv.WV_OK and (nh2, npr2) == (nh, npr)
    assert hits.tobytes() == sh.tobytes() and res.tobytes() == sr.tobytes()
    rc, nh3, npr3 = _wv.search_raw(w.lo, w.hi, w.mode, hits, None)     # hits only
    assert rc == _wv.WV_OK and nh3 == nh
    gh, gr = wv.search(w.lo, w.hi, w.mode)                             # the binding's wv_search path
    assert gh.tobytes() == sh.tobytes() and gr.tobytes() == sr.tobytes()
    rc, _, _ = _wv.search_raw(10, 5, 3, hits, res)
    assert rc == _wv.WV_EINVAL


def test_lane_mode_batches_bit_exact(wv, monkeypatch):
    """Lane mode cut into batches of the partial-pair buffer (group-aligned record ranges; the default
    budget of 2^24 slots is only exceeded by windows of ~10^8 primes, so WV_PART_BUDGET = 2^18 forces
    many batches here): C2 and a window straddling 2^30 (lane batches next to class-1 chunk items) give the
    default bytes and checksums, and the lane kernels' term count is the unbatched one."""
    for lo, hi, mode in [(5, 3 * 10 ** 6, 3), ((1 << 30) - 300000, (1 << 30) + 20000, 3)]:
        ref = wv.DeviceSearch(lo, hi, mode).run()
        r_res, r_chk = ref.res_np(), ref.checksum_int()
        wv.stats_reset()
        wv.stats_enable(True)
        wv.DeviceSearch(lo, hi, mode).run()
        t_ref = wv.stats()["terms32"]
        monkeypatch.setenv("WV_PART_BUDGET", str(1 << 18))
        wv.stats_reset()
        got = wv.DeviceSearch(lo, hi, mode).run()
        t_got = wv.stats()["terms32"]
        wv.stats_enable(False)
        monkeypatch.delenv("WV_PART_BUDGET")
        g_res = got.res_np()
        assert got.n_primes == ref.n_primes
        assert g_res[0].tobytes() == r_res[0].tobytes() and g_res[1].tobytes() == r_res[1].tobytes(), (lo, hi)
        assert got.checksum_int() == r_chk and t_got == t_ref


@pytest.mark.parametrize("allsl", ["0", "1"])
def test_lane2_sliced_code_for_whole_groups(wv, allsl, monkeypatch):
    """Whole lane groups (Q = 1) give the same bytes through the sliced chain code (a whole group is slice 0
    of 1) as through the unsliced one: WV_LANE_ALLSL forces either choice; the default picks by launch
    (most groups sliced -> sliced code for all).  C2 whole and one shard of an 8-way split."""
    for shard, n in [(0, 1), (5, 8)]:
        w = CONFIGS["c2"]
        ref = wv.DeviceSearch(w.lo, w.hi, w.mode, shard, n).run()
        monkeypatch.setenv("WV_LANE_ALLSL", allsl)
        got = wv.DeviceSearch(w.lo, w.hi, w.mode, shard, n).run()
        monkeypatch.delenv("WV_LANE_ALLSL")
        a, b = ref.res_np(), got.res_np()
        assert a[0].tobytes() == b[0].tobytes() and a[1].tobytes() == b[1].tobytes()
        assert ref.checksum_int() == got.checksum_int()


def test_async_device_search_equals_synchronous(wv):
    """wv_search_device with neither count wanted (n_primes = n_hits = NULL) runs a class-0 window without any
    host synchronisation (item counts and the sliced-code choice read on the device); its residues, hits and
    checksum equal the synchronous call's, on C2 and an 8-way shard of it (the bench's timed step), and a
    window reaching past 2^30 (which falls back to the synchronous plan) is unaffected."""
    import torch
    for args in [(5, 3 * 10 ** 6, 3, 0, 1), (5, 3 * 10 ** 6, 3, 5, 8), ((1 << 30) - 20000, (1 << 30) + 20000, 3, 0, 1)]:
        ref = wv.DeviceSearch(*args).run()
        r_res, r_chk, r_hits = ref.res_np(), ref.checksum_int(), ref.hits_np().tobytes()
        got = wv.DeviceSearch(*args)
        got.res_w.fill_(-1)
        got.res_v.fill_(-1)
        got.run(hit_count=False, prime_count=False)
        torch.cuda.synchronize()
        got.n_primes, got.n_hits = ref.n_primes, ref.n_hits        # counts were not reported by the async call
        g_res = got.res_np()
        assert g_res[0].tobytes() == r_res[0].tobytes() and g_res[1].tobytes() == r_res[1].tobytes(), args
        assert got.checksum_int() == r_chk and got.hits_np().tobytes() == r_hits, args
