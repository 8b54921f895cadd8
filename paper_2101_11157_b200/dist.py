"""Multi-GPU search: one process per GPU, interleaved prime blocks, NCCL gather of results.

SURVEY.md 8(e): [lo, hi) is cut into fixed blocks dealt to the N ranks in
rounds of N, snake order (round j gives block jN + r to rank r for even j and
block jN + N-1-r for odd j), with the rounds aligned to the top of the window
(pad = (-nblocks) mod N virtual empty blocks below block 0, so the one partial
round holds the lightest blocks) -- wv_shard_blocks / wv_search_shard in
include/wv.h.  Interleaving balances prime density and per-prime work, which
both drift with p.  Each rank sieves and computes its own blocks with no
communication (wv_search_shard on its device).  The only exchange is after
compute: an all_gather of (n_primes, n_hits, checksum) per rank, then of the
hit lists padded to the largest count (and, only if asked, of the residues).
Rank 0 (every rank, in fact) merges: hits and residues sorted by p, checksum
= sum of the rank checksums mod 2^64 -- identical to the 1-GPU result.

Works with NCCL (tensors on the rank's cuda device) and with gloo (CPU
tensors), so the host-side logic is tested on CPU with world_size 2.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _wv

M64 = (1 << 64) - 1


def _to_i64(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64).copy())


def gather_results(hits: np.ndarray, res: np.ndarray | None, checksum: int, device=None, group=None):
    """all_gather per-rank results; returns (hits, residues or None, checksum) merged and sorted by p."""
    world = dist.get_world_size(group)
    dev = torch.device(device) if device is not None else torch.device("cpu")
    nres = 0 if res is None else len(res)
    meta = torch.tensor([len(hits), nres, checksum - (1 << 64) if checksum >= (1 << 63) else checksum],
                        dtype=torch.int64, device=dev)
    metas = [torch.empty_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta, group=group)
    metas = [m.cpu().tolist() for m in metas]
    chk = sum(m[2] & M64 for m in metas) & M64

    def gather_rows(arr, dtype, count_idx):
        width = dtype.itemsize // 8
        mx = max(m[count_idx] for m in metas)
        buf = torch.zeros(max(mx, 1) * width, dtype=torch.int64, device=dev)
        if arr is not None and len(arr):
            buf[: len(arr) * width] = _to_i64(arr.view(np.uint8).view(np.uint64)).to(dev)
        bufs = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(bufs, buf, group=group)
        parts = []
        for m, b in zip(metas, bufs):
            raw = b.cpu().numpy()[: m[count_idx] * width].view(np.uint8)
            parts.append(np.frombuffer(raw.tobytes(), dtype=dtype))
        out = np.concatenate(parts) if parts else np.zeros(0, dtype=dtype)
        return np.sort(out, order="p")

    all_hits = gather_rows(hits, _wv.HIT_DTYPE, 0)
    all_res = gather_rows(res, _wv.RES_DTYPE, 1) if res is not None else None
    return all_hits, all_res, chk


def search_distributed(lo: int, hi: int, mode: int = _wv.MODE_BOTH, block: int = 0, residues: bool = False,
                       group=None):
    """Every rank: wv_search_shard on its current cuda device, then gather (NCCL if initialised so)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    hits, res, chk = _wv.search_shard(lo, hi, mode, rank, world, block, residues)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    return gather_results(hits, res, chk, device=dev, group=group)
