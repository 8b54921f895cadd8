// wv_scan.cuh -- exclusive prefix sums of uint64 counts (sieve segment counts,
// per-(prime,test) chunk counts, hit flags).  Three passes: per-tile totals,
// one-block scan of the tile totals, per-tile scan + tile offset.  Tiles of
// 2048 elements (256 threads x 8).  Out-of-range inputs read as 0.
#pragma once
#include <stdint.h>

namespace wv {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_PER_THREAD = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_PER_THREAD;

__device__ __forceinline__ uint64_t warp_incl_scan(uint64_t v) {
    const int lane = threadIdx.x & 31;
    #pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// block-wide exclusive scan of one value per thread; returns the block total via *total
__device__ __forceinline__ uint64_t block_excl_scan(uint64_t v, uint64_t *total) {
    __shared__ uint64_t warp_tot[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    uint64_t inc = warp_incl_scan(v);
    if (lane == 31) warp_tot[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        uint64_t t = lane < nw ? warp_tot[lane] : 0;
        uint64_t ti = warp_incl_scan(t);
        if (lane < nw) warp_tot[lane] = ti - t;      // exclusive warp offsets
        if (lane == nw - 1) warp_tot[31] = ti;       // (nw <= 31 here: blocks <= 992 threads)
    }
    __syncthreads();
    uint64_t res = warp_tot[wid] + inc - v;
    if (total) *total = warp_tot[31];
    __syncthreads();
    return res;
}

template <typename T>
__global__ void scan_tile_totals(const T *in, uint64_t n, uint64_t *tile_tot) {
    uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE;
    uint64_t s = 0;
    for (int j = 0; j < SCAN_PER_THREAD; j++) {
        uint64_t i = base + (uint64_t)threadIdx.x * SCAN_PER_THREAD + j;
        if (i < n) s += (uint64_t)in[i];
    }
    uint64_t tot;
    block_excl_scan(s, &tot);
    if (threadIdx.x == 0) tile_tot[blockIdx.x] = tot;
}

// single block: exclusive scan of ntiles totals in place; grand total to *total
__global__ void scan_tiles_single(uint64_t *tile_tot, uint64_t ntiles, uint64_t *total) {
    uint64_t carry = 0;
    for (uint64_t base = 0; base < ntiles; base += blockDim.x) {
        uint64_t i = base + threadIdx.x;
        uint64_t v = i < ntiles ? tile_tot[i] : 0;
        uint64_t tot;
        uint64_t ex = block_excl_scan(v, &tot);
        if (i < ntiles) tile_tot[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

template <typename T>
__global__ void scan_tile_apply(const T *in, uint64_t n, const uint64_t *tile_off, uint64_t *out) {
    uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_PER_THREAD;
    uint64_t v[SCAN_PER_THREAD];
    uint64_t s = 0;
    for (int j = 0; j < SCAN_PER_THREAD; j++) {
        uint64_t i = base + j;
        v[j] = i < n ? (uint64_t)in[i] : 0;
        s += v[j];
    }
    uint64_t ex = block_excl_scan(s, nullptr) + tile_off[blockIdx.x];
    for (int j = 0; j < SCAN_PER_THREAD; j++) {
        uint64_t i = base + j;
        if (i < n) out[i] = ex;
        ex += v[j];
    }
}

}  // namespace wv
