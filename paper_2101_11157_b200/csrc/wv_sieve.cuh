// wv_sieve.cuh -- segmented sieve of Eratosthenes on sm_100a.
//
// The paper enumerates primes on the host ("for each prime p within its
// assigned interval"); here the prime list is produced on the
// device.  A window is a list of "segments" of 2^15 integers, each holding
// 2^14 odd numbers as a 2 KB bitmap in shared memory (one CTA per segment).
// Segments are laid out block-by-block for the interleaved shard partition
// (block b of [lo,hi) belongs to shard b mod nshards).
//
// Marking, per segment:
//   phase 1  q in {3..31}: each thread builds whole 32-bit words from the
//            residue n mod q (no atomics);
//   phase 2  37 <= q < 2048: one warp per q, its lanes stride over the multiples
//            (shared-memory atomicOr), the warps on different q;
//   phase 3  q >= 2048: one thread per prime.
// Marks start at max(q^2, first odd multiple >= segment start), so base primes
// inside the window survive.  Then count (per-segment totals -> scan) and a
// second kernel writes the primes in ascending order.
#pragma once
#include <stdint.h>
#include "wv_scan.cuh"

namespace wv {

constexpr int SIEVE_ODDS = 16384;                 // odd numbers per segment
constexpr int SIEVE_SPAN = 2 * SIEVE_ODDS;        // integers per segment (also the shard block granule)
constexpr int SIEVE_WORDS = SIEVE_ODDS / 32;      // 512
constexpr int SIEVE_THREADS = 256;
constexpr uint32_t SIEVE_MED = 2048;              // phase-2 / phase-3 split

// Block b of the window belongs to shard snake(b): blocks are dealt out in rounds of
// nshards, alternating direction (0,1,..,N-1, N-1,..,1,0, ...), so that the linear
// growth of per-prime work with p is balanced across shards.  The j-th block of
// shard s is  j*N + (j even ? s : N-1-s)  - pad.  The rounds are aligned to the top of the window:
// pad = (-nblocks) mod N virtual (empty) blocks sit below block 0, so the one partial round holds
// the lightest blocks (smallest p) rather than the heaviest.
__host__ __device__ __forceinline__ uint64_t shard_block(uint64_t j, uint32_t s, uint32_t n) {
    return j * n + ((j & 1) ? (uint64_t)(n - 1 - s) : (uint64_t)s);
}
__host__ __device__ __forceinline__ uint64_t shard_pad(uint64_t nblocks, uint32_t n) {
    return (n - nblocks % n) % n;
}

struct SegMap {             // segment index -> integer range, for a shard of blocks
    uint64_t lo, hi;        // window [lo, hi)
    uint64_t block;         // block size (multiple of SIEVE_SPAN)
    uint32_t shard, nshards;
    uint64_t segs_per_block;
    uint64_t minp;          // smallest prime to report (5 for the search, 3 for base lists)
    uint64_t pad;           // virtual empty blocks below block 0 (shard_pad)

    __host__ __device__ void range(uint64_t seg, uint64_t *a, uint64_t *b) const {
        uint64_t j = seg / segs_per_block, r = seg % segs_per_block;
        uint64_t blk = shard_block(j, shard, nshards);
        if (blk < pad) {                          // virtual block: empty
            *a = *b = lo;
            return;
        }
        blk -= pad;
        uint64_t bs = lo + blk * block;           // may exceed hi for trailing segments
        uint64_t s = bs + r * (uint64_t)SIEVE_SPAN;
        uint64_t e = s + SIEVE_SPAN;
        uint64_t be = bs + block;
        if (e > be) e = be;
        if (e > hi) e = hi;
        if (s > hi) s = hi;
        if (s < minp) s = minp < e ? minp : e;
        *a = s; *b = e > s ? e : s;
    }
};

__device__ __forceinline__ uint64_t first_odd_ge(uint64_t x) { return x | 1ull; }

// One CTA per segment.  bitmap[seg][w]: bit b set <=> n = n0 + 2(32w + b) is prime.
__global__ void __launch_bounds__(SIEVE_THREADS)
sieve_segments_kernel(SegMap map, const uint32_t *__restrict__ base, uint32_t nbase_host,
                      const uint64_t *__restrict__ nbase_dev,
                      uint32_t *__restrict__ bitmap, uint64_t *__restrict__ seg_count) {
    __shared__ uint32_t comp[SIEVE_WORDS];        // 1 = composite
    const uint32_t nbase = nbase_dev ? (uint32_t)*nbase_dev : nbase_host;
    const uint64_t seg = blockIdx.x;
    uint64_t a, b;
    map.range(seg, &a, &b);
    const uint64_t n0 = first_odd_ge(a);          // odd number of bit 0 (segment-local origin)
    const uint64_t ne = b;                        // numbers < ne are in the segment

    // phase 1: q = 3..31 by word patterns
    for (int w = threadIdx.x; w < SIEVE_WORDS; w += blockDim.x) {
        const uint64_t nw = n0 + 64ull * w;
        uint32_t mask = 0;
        #pragma unroll
        for (int qi = 0; qi < 10; qi++) {
            const uint32_t Q[10] = {3, 5, 7, 11, 13, 17, 19, 23, 29, 31};
            const uint32_t q = Q[qi];
            if ((uint64_t)q * q >= ne) continue;
            uint32_t r = (uint32_t)(nw % q);
            uint32_t b0 = (uint32_t)(((uint64_t)((q - r) % q) * ((q + 1) / 2)) % q);  // (nw + 2 b0) == 0 mod q
            for (uint32_t bb = b0; bb < 32; bb += q) mask |= 1u << bb;
            if (q >= nw && q < nw + 64) mask &= ~(1u << ((q - nw) >> 1));              // q itself is prime
        }
        comp[w] = mask;
    }
    __syncthreads();

    // phase 2: medium primes, one warp per q (warps take q_j, q_{j+8}, ...), lanes stride over its multiples;
    // the per-q start offset (a 64-bit division) is computed by one warp instead of serially by all threads
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    uint32_t j3 = 10, hi3 = nbase;                // j3 = first index with base[j3] >= SIEVE_MED (ascending)
    while (j3 < hi3) {
        const uint32_t mid = (j3 + hi3) >> 1;
        if (base[mid] < SIEVE_MED) j3 = mid + 1; else hi3 = mid;
    }
    const uint64_t lim = (ne - n0 + 1) >> 1;      // bit indices < lim are in range
    for (uint32_t jj = 10 + warp; jj < j3; jj += nwarps) {   // base[] = 3,5,7,...: entries 0..9 are <= 31
        const uint32_t q = base[jj];
        const uint64_t qq = (uint64_t)q * q;
        if (qq >= ne) break;                      // ascending: later q of this warp are larger
        uint64_t st = n0 > qq ? n0 : qq;
        uint64_t m = (st + q - 1) / q * q;
        if (!(m & 1)) m += q;
        if (m >= ne) continue;
        const uint64_t i0 = (m - n0) >> 1;
        for (uint64_t i = i0 + (uint64_t)lane * q; i < lim; i += 32ull * q)
            atomicOr(&comp[i >> 5], 1u << (i & 31));
    }
    const uint32_t j = j3;
    // phase 3: large primes, one thread each
    for (uint32_t k = j + threadIdx.x; k < nbase; k += blockDim.x) {
        const uint32_t q = base[k];
        const uint64_t qq = (uint64_t)q * q;
        if (qq >= ne) break;                        // base[] ascending
        uint64_t st = n0 > qq ? n0 : qq;
        uint64_t m = (st + q - 1) / q * q;
        if (!(m & 1)) m += q;
        for (uint64_t i = (m - n0) >> 1; i < lim; i += q) atomicOr(&comp[i >> 5], 1u << (i & 31));
    }
    __syncthreads();

    // count primes: odd n in [max(a, minp), ne), n != 1
    uint64_t cnt = 0;
    for (int w = threadIdx.x; w < SIEVE_WORDS; w += blockDim.x) {
        const uint64_t nw = n0 + 64ull * w;
        uint32_t valid = 0;
        if (nw < ne) {
            uint64_t nbits = (ne - nw + 1) >> 1;
            valid = nbits >= 32 ? 0xffffffffu : ((1u << nbits) - 1u);
        }
        if (nw <= 1 && valid) valid &= ~1u;                           // 1 is not prime
        uint32_t primes = ~comp[w] & valid;
        if (bitmap) bitmap[seg * SIEVE_WORDS + w] = primes;
        cnt += __popc(primes);
    }
    uint64_t tot;
    block_excl_scan(cnt, &tot);
    if (threadIdx.x == 0) seg_count[seg] = tot;
}

// One CTA per segment: write the primes of the segment in ascending order.
template <typename T>
__global__ void __launch_bounds__(SIEVE_THREADS)
sieve_write_kernel(SegMap map, const uint32_t *__restrict__ bitmap, const uint64_t *__restrict__ seg_off,
                   T *__restrict__ out, uint64_t cap) {
    constexpr int WPT = SIEVE_WORDS / SIEVE_THREADS;   // 2 words per thread
    const uint64_t seg = blockIdx.x;
    uint64_t a, b;
    map.range(seg, &a, &b);
    const uint64_t n0 = first_odd_ge(a);
    uint32_t w[WPT];
    uint64_t c = 0;
    #pragma unroll
    for (int k = 0; k < WPT; k++) {
        w[k] = bitmap[seg * SIEVE_WORDS + threadIdx.x * WPT + k];
        c += __popc(w[k]);
    }
    uint64_t pos = seg_off[seg] + block_excl_scan(c, nullptr);
    #pragma unroll
    for (int k = 0; k < WPT; k++) {
        uint32_t x = w[k];
        const uint64_t nw = n0 + 64ull * (threadIdx.x * WPT + k);
        while (x) {
            int bb = __ffs(x) - 1;
            x &= x - 1;
            if (pos < cap) out[pos] = (T)(nw + 2ull * bb);
            pos++;
        }
    }
}

}  // namespace wv
