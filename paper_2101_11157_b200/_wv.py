"""Thin ctypes binding over libwv.so (include/wv.h) -- argument marshalling only.

Every step of the path runs in the library's CUDA kernels; this module only
converts Python ints / numpy arrays / torch tensors to pointers and back.
There is no CPU fallback: if libwv.so is missing or the device is not an
sm_100 GPU, calls raise WVError.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WV_LIB") or os.path.join(_HERE, "libwv.so")   # WV_LIB: A/B builds only

MODE_W, MODE_V, MODE_BOTH = 1, 2, 3
RES_NONE = (1 << 64) - 1
WV_OK, WV_EINVAL, WV_ENOSPC, WV_ECUDA, WV_ENOMEM = 0, -1, -2, -3, -4
HIT_W, HIT_V = 1, 2

HIT_DTYPE = np.dtype([("p", "<u8"), ("flags", "<u4"), ("reserved", "<u4")])
RES_DTYPE = np.dtype([("p", "<u8"), ("res_w", "<u8"), ("res_v", "<u8")])
NEAR_DTYPE = np.dtype([("p", "<u8"), ("symres", "<i8"), ("test", "<u4"), ("reserved", "<u4")])
PAIR_DTYPE = np.dtype([("p", "<u8"), ("index", "<u4"), ("kind", "<u4")])        # kind 1: p | B_index, 2: E
IDXRES_DTYPE = np.dtype([("p", "<u8"), ("index", "<u4"), ("reserved", "<u4"), ("res_b", "<u8"), ("res_e", "<u8")])
KIND_B, KIND_E = 1, 2


class WVError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libwv error {code}: {msg}")
        self.code = code


class _Term(ctypes.Structure):
    _fields_ = [("a", ctypes.c_int64), ("xn", ctypes.c_uint32), ("xd", ctypes.c_uint32),
                ("yn", ctypes.c_uint32), ("yd", ctypes.c_uint32)]


class _CongHdr(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 8), ("L_lo", ctypes.c_uint64), ("L_hi", ctypes.c_uint64),
                ("L_neg", ctypes.c_uint32), ("e", ctypes.c_uint32), ("m", ctypes.c_uint32),
                ("min_p", ctypes.c_uint32), ("excluded_p", ctypes.c_uint32), ("seg", ctypes.c_uint32)]


class _Term128(ctypes.Structure):
    _fields_ = [("a_lo", ctypes.c_uint64), ("a_hi", ctypes.c_uint64), ("neg", ctypes.c_uint32),
                ("xn", ctypes.c_uint32), ("xd", ctypes.c_uint32), ("yn", ctypes.c_uint32), ("yd", ctypes.c_uint32)]


class _Cong(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 8), ("L", ctypes.c_int64), ("e", ctypes.c_uint32),
                ("m", ctypes.c_uint32), ("min_p", ctypes.c_uint32), ("excluded_p", ctypes.c_uint32),
                ("t", _Term * 33)]


class Stats(ctypes.Structure):
    _fields_ = [("terms", ctypes.c_uint64), ("terms32", ctypes.c_uint64), ("terms_fp", ctypes.c_uint64),
                ("residue_launches", ctypes.c_uint64), ("records", ctypes.c_uint64), ("chunks", ctypes.c_uint64),
                ("residue_ms", ctypes.c_double), ("residue32_ms", ctypes.c_double), ("residue_fp_ms", ctypes.c_double)]


# (name, restype, argtypes) for every symbol include/wv.h declares
_u64, _u32, _sz, _vp, _i = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_int
_P = ctypes.POINTER
SIGNATURES = {
    "wv_search": (_i, [_u64, _u64, _u32, _vp, _sz, _P(_sz), _vp, _sz, _P(_sz)]),
    "wv_search_shard": (_i, [_u64, _u64, _u32, _u32, _u32, _u64, _vp, _sz, _P(_sz), _vp, _sz, _P(_sz), _P(_u64)]),
    "wv_device_workspace_bytes": (_i, [_u64, _u64, _u32, _u32, _u32, _u64, _P(_sz), _P(_sz)]),
    "wv_search_device": (_i, [_u64, _u64, _u32, _u32, _u32, _u64, _vp, _vp, _vp, _vp, _vp, _sz, _vp, _sz, _vp,
                              _P(_sz), _P(_sz)]),
    "wv_residues_workspace_bytes": (_i, [_sz, _u64, _u32, _P(_sz)]),
    "wv_residues_device": (_i, [_vp, _sz, _u32, _vp, _vp, _vp, _sz, _vp]),
    "wv_sieve_device": (_i, [_u64, _u64, _vp, _sz, _P(_sz), _vp, _sz, _vp]),
    "wv_prime_count": (_i, [_u64, _u64, _P(_u64)]),
    "wv_near_misses_device": (_i, [_vp, _vp, _vp, _sz, _u64, _vp, _sz, _P(_sz), _vp, _vp, _vp, _vp]),
    "wv_shard_blocks": (_i, [_u64, _u64, _u32, _u32, _u64, _vp, _sz, _P(_sz), _P(_u64)]),
    "wv_checksum_term": (_u64, [_u64, _u64, _u64]),
    "wv_congruence_count": (_i, []),
    "wv_congruence_get": (_i, [_i, _P(_Cong)]),
    "wv_congruence_header": (_i, [_i, _P(_CongHdr)]),
    "wv_congruence_term": (_i, [_i, _u32, _P(_Term128)]),
    "wv_set_schedule_override": (_i, [_i, _i]),
    "wv_schedule": (_i, [_u64, _u32]),
    "wv_stats_enable": (_i, [_i]),
    "wv_stats_get": (_i, [_P(Stats)]),
    "wv_stats_reset": (_i, []),
    "wv_kernel_variant_info": (_i, [_i, ctypes.c_char_p, _sz, _P(_i)]),
    "wv_set_kernel_variant": (_i, [_i, _i]),
    "wv_census": (_i, [_u64, _u64, _u32, _vp, _sz, _P(_sz), _P(_sz), _P(_u64)]),
    "wv_census_residues": (_i, [_u64, _u64, _u32, _vp, _sz, _P(_sz)]),
    "wv_census_checksum_term": (_u64, [_u64, _u32, _u32, _u64]),
    "wv_launch_count": (_u64, []),
    "wv_version": (ctypes.c_char_p, []),
    "wv_last_error": (ctypes.c_char_p, []),
}

_lib = None


def lib():
    """Load libwv.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc):
    if rc != WV_OK:
        raise WVError(rc, lib().wv_last_error().decode(errors="replace"))


def _ptr(t):
    """Device/host pointer of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return ctypes.c_void_p(t.data_ptr())
    return t.ctypes.data_as(ctypes.c_void_p)


# ------------------------------------------------------------------ host-buffer API
def search(lo: int, hi: int, mode: int = MODE_BOTH, residues: bool = True):
    """wv_search: returns (hits: np.ndarray[HIT_DTYPE], residues: np.ndarray[RES_DTYPE] or None).

    Buffers are sized from the library's prime bound (wv_device_workspace_bytes); on WV_ENOSPC (the
    two-call contract of include/wv.h) they are resized to the reported counts and the call repeated."""
    L = lib()
    ws, cap = ctypes.c_size_t(), ctypes.c_size_t()
    _check(L.wv_device_workspace_bytes(lo, hi, mode, 0, 1, 0, ctypes.byref(ws), ctypes.byref(cap)))
    nh_cap = npr_cap = max(int(cap.value), 1)
    for _ in range(2):
        hits = np.zeros(nh_cap, dtype=HIT_DTYPE)
        res = np.zeros(npr_cap, dtype=RES_DTYPE) if residues else None
        nh, npr = ctypes.c_size_t(), ctypes.c_size_t()
        rc = L.wv_search(lo, hi, mode, _ptr(hits), len(hits), ctypes.byref(nh), _ptr(res),
                         len(res) if residues else 0, ctypes.byref(npr))
        if rc == WV_ENOSPC:
            nh_cap, npr_cap = max(int(nh.value), 1), max(int(npr.value), 1)
            continue
        _check(rc)
        return hits[: nh.value].copy(), (res[: npr.value].copy() if residues else None)
    _check(rc)


def search_raw(lo: int, hi: int, mode: int, hits: np.ndarray | None, res: np.ndarray | None):
    """One wv_search call into the given buffers (tests of the WV_ENOSPC contract):
    returns (rc, n_hits, n_primes) without raising."""
    nh, npr = ctypes.c_size_t(), ctypes.c_size_t()
    rc = lib().wv_search(lo, hi, mode, _ptr(hits), 0 if hits is None else len(hits), ctypes.byref(nh), _ptr(res),
                         0 if res is None else len(res), ctypes.byref(npr))
    return int(rc), int(nh.value), int(npr.value)


def search_shard(lo: int, hi: int, mode: int, shard: int, nshards: int, block: int = 0, residues: bool = True,
                 hits_out: np.ndarray | None = None, res_out: np.ndarray | None = None):
    """wv_search_shard: returns (hits, residues or None, checksum).

    hits_out / res_out: optional caller buffers (HIT_DTYPE / RES_DTYPE arrays, e.g. views of pinned
    memory from pinned_buffers()) with room for prime_cap entries; the results are views into them."""
    L = lib()
    ws, cap = ctypes.c_size_t(), ctypes.c_size_t()
    _check(L.wv_device_workspace_bytes(lo, hi, mode, shard, nshards, block, ctypes.byref(ws), ctypes.byref(cap)))
    n = max(int(cap.value), 1)
    hits = hits_out if hits_out is not None and len(hits_out) >= n else np.zeros(n, dtype=HIT_DTYPE)
    res = None
    if residues:
        res = res_out if res_out is not None and len(res_out) >= n else np.zeros(n, dtype=RES_DTYPE)
    nh, npr, chk = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_uint64()
    _check(L.wv_search_shard(lo, hi, mode, shard, nshards, block, _ptr(hits), len(hits), ctypes.byref(nh), _ptr(res),
                             len(res) if residues else 0, ctypes.byref(npr), ctypes.byref(chk)))
    hv = hits[: nh.value] if hits is hits_out else hits[: nh.value].copy()
    rv = None
    if residues:
        rv = res[: npr.value] if res is res_out else res[: npr.value].copy()
    return hv, rv, int(chk.value)


def pinned_buffers(lo: int, hi: int, mode: int = MODE_BOTH, shard: int = 0, nshards: int = 1, block: int = 0):
    """Page-locked (torch pin_memory) host buffers sized for wv_search_shard over this window."""
    import torch
    ws, cap = ctypes.c_size_t(), ctypes.c_size_t()
    _check(lib().wv_device_workspace_bytes(lo, hi, mode, shard, nshards, block, ctypes.byref(ws), ctypes.byref(cap)))
    n = max(int(cap.value), 1)
    th = torch.empty(n * HIT_DTYPE.itemsize, dtype=torch.uint8).pin_memory()
    tr = torch.empty(n * RES_DTYPE.itemsize, dtype=torch.uint8).pin_memory()
    hits = th.numpy().view(HIT_DTYPE)
    res = tr.numpy().view(RES_DTYPE)
    return (th, tr), hits, res


# ------------------------------------------------------------------ device API (torch tensors)
class DeviceSearch:
    """Preallocated device buffers (torch) for repeated wv_search_device calls on one window."""

    def __init__(self, lo, hi, mode=MODE_BOTH, shard=0, nshards=1, block=0, device=None):
        import torch
        L = lib()
        ws, cap = ctypes.c_size_t(), ctypes.c_size_t()
        _check(L.wv_device_workspace_bytes(lo, hi, mode, shard, nshards, block, ctypes.byref(ws), ctypes.byref(cap)))
        self.args = (lo, hi, mode, shard, nshards, block)
        self.device = torch.device(device or "cuda")
        self.cap = max(int(cap.value), 1)
        self.ws_bytes = int(ws.value)
        u = dict(dtype=torch.int64, device=self.device)      # uint64 bit patterns
        self.primes = torch.empty(self.cap, **u)
        self.res_w = torch.empty(self.cap, **u)
        self.res_v = torch.empty(self.cap, **u)
        self.hits = torch.empty(self.cap * 2, **u)          # wv_hit = 16 bytes
        self.checksum = torch.zeros(1, **u)
        self.workspace = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        self.n_primes = 0
        self.n_hits = 0

    def run(self, stream=None, hit_count=True, prime_count=True):
        """One wv_search_device call.  hit_count=False: do not wait for the hit count; with prime_count=False
        as well, the call may return as soon as the work is enqueued (include/wv.h); the counts not asked for
        keep the values of the last run that reported them (the same window gives the same counts)."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        npr, nh = ctypes.c_size_t(), ctypes.c_size_t()
        lo, hi, mode, shard, nshards, block = self.args
        _check(lib().wv_search_device(lo, hi, mode, shard, nshards, block, _ptr(self.primes), _ptr(self.res_w),
                                      _ptr(self.res_v), _ptr(self.hits), _ptr(self.checksum), self.cap,
                                      _ptr(self.workspace), self.ws_bytes, ctypes.c_void_p(st.cuda_stream),
                                      ctypes.byref(npr) if (prime_count or hit_count) else None,
                                      ctypes.byref(nh) if hit_count else None))
        if prime_count or hit_count:
            self.n_primes = int(npr.value)
        if hit_count:
            self.n_hits = int(nh.value)
        return self

    # host views (copies) of the outputs
    def primes_np(self):
        return self.primes[: self.n_primes].cpu().numpy().view(np.uint64)

    def res_np(self):
        return (self.res_w[: self.n_primes].cpu().numpy().view(np.uint64),
                self.res_v[: self.n_primes].cpu().numpy().view(np.uint64))

    def hits_np(self):
        raw = self.hits[: 2 * self.n_hits].cpu().numpy().view(np.uint8)
        return np.frombuffer(raw.tobytes(), dtype=HIT_DTYPE)

    def checksum_int(self):
        return int(self.checksum.cpu().numpy().view(np.uint64)[0])

    def near_misses(self, bound=50, histograms=True, cap=1 << 16):
        """NEXT-1: near misses |<r>_p| < bound (sorted by p, test) and the
        2000-bin histograms of <r>_p / p for W and V (numpy uint64[2000] each, zeros if not requested)."""
        return near_misses_device(self.primes, self.res_w, self.res_v, self.n_primes, bound, histograms, cap)


def near_misses_device(primes, res_w, res_v, n, bound=50, histograms=True, cap=1 << 16, stream=None):
    """wv_near_misses_device on torch cuda tensors -> (near: NEAR_DTYPE sorted, hist_w, hist_v)."""
    import torch
    dev = primes.device
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    out = torch.empty(max(cap, 1) * 3, dtype=torch.int64, device=dev)        # NEAR_DTYPE = 24 bytes
    hw = torch.zeros(2000, dtype=torch.int64, device=dev) if histograms else None
    hv = torch.zeros(2000, dtype=torch.int64, device=dev) if histograms else None
    cnt = ctypes.c_size_t()
    _check(lib().wv_near_misses_device(_ptr(primes), _ptr(res_w), _ptr(res_v), n, bound, _ptr(out), cap,
                                       ctypes.byref(cnt), _ptr(hw), _ptr(hv), None, ctypes.c_void_p(st.cuda_stream)))
    raw = out[: 3 * cnt.value].cpu().numpy().view(np.uint8)
    near = np.sort(np.frombuffer(raw.tobytes(), dtype=NEAR_DTYPE), order=["p", "test"])
    z = np.zeros(2000, dtype=np.uint64)
    return near, (hw.cpu().numpy().view(np.uint64) if hw is not None else z), \
        (hv.cpu().numpy().view(np.uint64) if hv is not None else z)


def residues_device(primes, mode=MODE_BOTH, stream=None, max_p=None):
    """wv_residues_device on a torch uint64/int64 cuda tensor of primes -> (res_w, res_v) tensors.
    The workspace is sized for primes <= max_p (default: the list's maximum; a smaller bound only
    drops the coarse seg index for the larger primes, which then scan their sums)."""
    import torch
    n = primes.numel()
    if max_p is None:
        max_p = int(primes.max().item()) if n else 0
    ws = ctypes.c_size_t()
    _check(lib().wv_residues_workspace_bytes(n, max_p, mode, ctypes.byref(ws)))
    work = torch.empty(max(int(ws.value), 1), dtype=torch.uint8, device=primes.device)
    rw = torch.empty_like(primes)
    rv = torch.empty_like(primes)
    st = stream if stream is not None else torch.cuda.current_stream(primes.device)
    _check(lib().wv_residues_device(_ptr(primes), n, mode, _ptr(rw), _ptr(rv), _ptr(work), int(ws.value),
                                    ctypes.c_void_p(st.cuda_stream)))
    return rw, rv


def residues_of(plist, mode=MODE_BOTH, device="cuda"):
    """Convenience: residues for a Python list of primes -> (np res_w, np res_v)."""
    import torch
    arr = np.asarray(plist, dtype=np.uint64)
    t = torch.from_numpy(arr.view(np.int64)).to(device)
    rw, rv = residues_device(t, mode)
    torch.cuda.synchronize()
    return rw.cpu().numpy().view(np.uint64), rv.cpu().numpy().view(np.uint64)


def sieve_device(lo, hi, device="cuda"):
    """wv_sieve_device -> np.ndarray of primes in [max(lo,5), hi)."""
    import torch
    L = lib()
    ws, cap = ctypes.c_size_t(), ctypes.c_size_t()
    _check(L.wv_device_workspace_bytes(lo, hi, 1, 0, 1, 0, ctypes.byref(ws), ctypes.byref(cap)))
    out = torch.empty(max(int(cap.value), 1), dtype=torch.int64, device=device)
    work = torch.empty(int(ws.value), dtype=torch.uint8, device=device)
    n = ctypes.c_size_t()
    st = torch.cuda.current_stream(out.device)
    _check(L.wv_sieve_device(lo, hi, _ptr(out), int(cap.value), ctypes.byref(n), _ptr(work), int(ws.value),
                             ctypes.c_void_p(st.cuda_stream)))
    return out[: n.value].cpu().numpy().view(np.uint64)


def prime_count(lo, hi):
    """wv_prime_count: primes in [max(lo,5), hi) counted on the device."""
    c = ctypes.c_uint64()
    _check(lib().wv_prime_count(lo, hi, ctypes.byref(c)))
    return int(c.value)


def shard_blocks(lo, hi, shard, nshards, block=0):
    """Host-only: ([(a, b), ...] integer ranges of this shard's blocks, block size used)."""
    L = lib()
    n, bu = ctypes.c_size_t(), ctypes.c_uint64()
    _check(L.wv_shard_blocks(lo, hi, shard, nshards, block, None, 0, ctypes.byref(n), ctypes.byref(bu)))
    buf = np.zeros(2 * max(n.value, 1), dtype=np.uint64)
    _check(L.wv_shard_blocks(lo, hi, shard, nshards, block, _ptr(buf), n.value, ctypes.byref(n), ctypes.byref(bu)))
    return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(n.value)], int(bu.value)


# ------------------------------------------------------------------ small utilities
def checksum_term(p, rw, rv):
    return int(lib().wv_checksum_term(p, rw, rv))


def census(lo: int, hi: int, mode: int = MODE_BOTH, cap: int = 1 << 16):
    """Irregular (kind 1) and E-irregular (kind 2) pairs of the primes in [lo, hi) (NEXT-3):
    (pairs[PAIR_DTYPE] sorted by (p, kind, index), n_primes, checksum)."""
    n, npr, chk = _sz(), _sz(), _u64()
    out = np.zeros(cap, dtype=PAIR_DTYPE)
    rc = lib().wv_census(lo, hi, mode, out.ctypes.data, cap, ctypes.byref(n), ctypes.byref(npr), ctypes.byref(chk))
    if rc == WV_ENOSPC:
        out = np.zeros(n.value, dtype=PAIR_DTYPE)
        rc = lib().wv_census(lo, hi, mode, out.ctypes.data, n.value, ctypes.byref(n), ctypes.byref(npr),
                             ctypes.byref(chk))
    _check(rc)
    return out[: n.value], npr.value, chk.value


def census_residues(lo: int, hi: int, mode: int = MODE_BOTH):
    """B_{2k} / E_{2k} mod p for every prime in [lo, hi) and 2 <= 2k <= p-3 (IDXRES_DTYPE records)."""
    n = _sz()
    rc = lib().wv_census_residues(lo, hi, mode, None, 0, ctypes.byref(n))
    if rc not in (WV_OK, WV_ENOSPC):
        _check(rc)
    out = np.zeros(n.value, dtype=IDXRES_DTYPE)
    _check(lib().wv_census_residues(lo, hi, mode, out.ctypes.data if n.value else None, n.value, ctypes.byref(n)))
    return out


def census_checksum_term(p, index, kind, res):
    return int(lib().wv_census_checksum_term(p, index, kind, res))


def congruences():
    """The library's congruence table as a list of dicts (Python-int coefficients)."""
    L = lib()
    out = []
    for i in range(L.wv_congruence_count()):
        h = _CongHdr()
        _check(L.wv_congruence_header(i, ctypes.byref(h)))
        lft = (h.L_hi << 64) | h.L_lo
        terms = []
        for j in range(h.m):
            t = _Term128()
            _check(L.wv_congruence_term(i, j, ctypes.byref(t)))
            a = (t.a_hi << 64) | t.a_lo
            terms.append((-a if t.neg else a, t.xn, t.xd, t.yn, t.yd))
        out.append(dict(id=i, name=h.name.decode(), L=-lft if h.L_neg else lft, e=h.e, min_p=h.min_p,
                        excluded_p=h.excluded_p, seg=h.seg, terms=terms))
    return out


def set_schedule_override(w_id=-1, v_id=-1):
    _check(lib().wv_set_schedule_override(w_id, v_id))


def schedule(p, test):
    return int(lib().wv_schedule(p, test))


def stats_enable(on=True):
    _check(lib().wv_stats_enable(1 if on else 0))


def stats_reset():
    _check(lib().wv_stats_reset())


def stats():
    s = Stats()
    _check(lib().wv_stats_get(ctypes.byref(s)))
    return {k: getattr(s, k) for k, _ in Stats._fields_}


def kernel_variants():
    """[(id, name, class)] of the residue-kernel variants."""
    out, i = [], 0
    while True:
        buf = ctypes.create_string_buffer(64)
        c = ctypes.c_int()
        if lib().wv_kernel_variant_info(i, buf, 64, ctypes.byref(c)) != WV_OK:
            return out
        out.append((i, buf.value.decode(), c.value))
        i += 1


def set_kernel_variant(cls, vid=-1):
    _check(lib().wv_set_kernel_variant(cls, vid))


def launch_count():
    return int(lib().wv_launch_count())


def version():
    return lib().wv_version().decode()
