"""B200-native Wolstenholme / Vandiver residue search (arXiv:2101.11157 hot path).

Public API (thin binding over the C ABI in include/wv.h, implemented by the
CUDA library libwv.so built from csrc/):

    search(lo, hi, mode)                   -> (hits, residues)      host buffers
    search_shard(lo, hi, mode, s, n, blk)  -> (hits, residues, checksum)
    DeviceSearch(lo, hi, mode).run()       device-resident buffers (torch)
    residues_device(primes_tensor, mode)   residue step only
    sieve_device(lo, hi)                   sieve step only
    congruences(), schedule(p, test), set_schedule_override(w, v)

Residues are canonical in [0, p): B_{p-3} mod p (mode W) and E_{p-3} mod p in
the secant convention (mode V).  ``workloads`` holds the BASELINE configs.
"""
from ._wv import (NEAR_DTYPE, near_misses_device, HIT_DTYPE, HIT_V, HIT_W, MODE_BOTH, MODE_V, MODE_W, RES_DTYPE, RES_NONE, DeviceSearch,  # noqa: F401
                  WVError, checksum_term, congruences, launch_count, lib, prime_count, residues_device, residues_of, schedule,
                  search, search_shard, shard_blocks, pinned_buffers, set_schedule_override, sieve_device, kernel_variants, set_kernel_variant, stats, stats_enable, stats_reset,
                  version, census, census_residues, census_checksum_term, PAIR_DTYPE, IDXRES_DTYPE, KIND_B, KIND_E)
