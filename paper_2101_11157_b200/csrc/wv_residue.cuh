// wv_residue.cuh -- plan, residue (hot loop) and finalize kernels.
//
// Per (prime, test) "record" k, the congruence L X == sum_j a_j S(x_j, y_j)
// has T = sum_j #{s : x_j p < s < y_j p} terms.  The
// T terms, concatenated sum after sum, are cut into chunks of 32*L terms;
// a chunk is one warp's work item, each lane a contiguous run of <= L terms.
//
// Lane hot loop: eqnComputeS
//     c1 <- c1 u + c0 ;  c0 <- c0 u          (u = s^e, e = 3 for W, 2 for V)
// with both products Montgomery products, the "+ c0" folded into the first
// REDC, and u = s^e advanced by exact finite differences (e = 3:
// u += d1, d1 += d2, d2 += 6; e = 2: u += d1, d1 += 2) -- modular adds only,
// so 2 Montgomery multiplies per term.  c1/c0 is then sum 1/u = S(x, y): the
// recurrence is Montgomery's batched-inversion trick specialised to a sum of
// inverses (one inversion per record, in finalize).
//
// At the end of a sum's run the lane folds the coefficient (c1 <- a_j c1) and
// merges the run into its accumulator with eqnCombinePairs:
//     (c0, c1) (+) (c0', c1') = (c0 c0', c0 c1' + c1 c0').
// Lanes merge by 5 xor-shuffle rounds; lane 0 stores the chunk's pair.
// Finalize merges a record's chunk pairs and returns
//     X = C1 * (C0 * L)^{-1}  mod p.
#pragma once
#include <stdint.h>
#include <type_traits>
#include "wv_mont.cuh"
#include "wv_scan.cuh"

namespace wv {

// A congruence  L X == sum_j a_j S(x_j, y_j)  (mod p).  Coefficients are stored as
// sign + 128-bit magnitude (generated congruences have ~80-bit integers); headers
// live in constant memory, terms in a global array (lanes read different terms).
struct Term { uint64_t a_lo, a_hi; uint32_t neg, xn, xd, yn, yd, pad; };       // 40 bytes
struct Cong {
    char name[8];
    uint64_t L_lo, L_hi;
    uint32_t L_neg, e, m, min_p, excluded_p;
    uint32_t seg;           // 1: sum-aligned chunking (many-sum congruences)
    uint32_t off;           // index of term 0 in c_terms
    uint32_t pad;
};

constexpr int NCONG_MAX = 32;
__constant__ Cong c_cong[NCONG_MAX];
__constant__ int c_ncong;
__constant__ const Term *c_terms;

// (a_hi 2^64 + a_lo) * (-1)^neg  mod p, in [0, p)
__device__ __forceinline__ uint64_t big_mod(uint64_t lo, uint64_t hi, uint32_t neg, uint64_t p) {
    uint64_t r;
    if (hi == 0) r = lo < p ? lo : lo % p;
    else r = (uint64_t)((((unsigned __int128)hi << 64) | lo) % p);
    return neg ? (r ? p - r : 0) : r;
}
__device__ __forceinline__ uint64_t coef_mod(const Term &t, uint64_t p) { return big_mod(t.a_lo, t.a_hi, t.neg, p); }
__device__ __forceinline__ uint64_t left_mod(const Cong &c, uint64_t p) { return big_mod(c.L_lo, c.L_hi, c.L_neg, p); }

struct Rec {                // one (prime, test) pair; 32 bytes
    uint64_t p;
    uint64_t T;             // number of terms
    uint32_t cid;           // congruence id
    uint32_t L;             // terms per lane in a full chunk
    uint32_t idx;           // output index of the prime
    uint32_t test;          // 0 = W (B_{p-3}), 1 = V (E_{p-3})
};

constexpr int SCHED_TIERS = 10;
struct Sched {              // tiered schedule + overrides
    // test t (0 = W, 1 = V): use id[t][i] for the largest i with p >= th[t][i]; th[t] ascends, th[t][0] = 0
    uint64_t th[2][SCHED_TIERS];
    int id[2][SCHED_TIERS];
    int n[2];
    int w_force, v_force;   // -1 = none
};

constexpr uint32_t CAP_CHUNKS = 1024;   // target max chunks per record
constexpr uint32_t MAX_CONTIG_M = 96;   // contiguous (non-seg) chunking handles congruences up to 96 sums
constexpr uint32_t LMIN = 4096;         // min terms per lane in a full chunk
constexpr uint64_t LANE_SLICE = 8192;   // lane mode: target terms per lane per slice
constexpr uint64_t LANE_QMAX = 128;     // lane mode: max slices per record
constexpr uint64_t WIDTH32_MAX = 1ull << 30;  // Mont32 (lazy, fused) needs p < 2^30
constexpr uint64_t FP64_MAX = 1ull << 44;     // ModD (FP64 engine) needs p < 2^44
__host__ __device__ __forceinline__ int prime_class(uint64_t p) { return p < WIDTH32_MAX ? 0 : (p < FP64_MAX ? 1 : 2); }

// ids in congruences.inc order
enum { C_VOR12 = 0, C_BB1 = 1, C_BB2, C_BB6, C_BB9, C_BB16, C_BB22, C_BB30,
       C_EE3, C_EE5, C_EE9, C_EE16, C_EE24, C_EE33 };

__host__ __device__ __forceinline__ int schedule(const Sched &s, uint64_t p, int test) {
    if (test == 0) {
        if (s.w_force >= 0) return s.w_force;
        if (p == 7) return C_VOR12;
    } else if (s.v_force >= 0) {
        return s.v_force;
    }
    int i = s.n[test] - 1;                       // the largest threshold <= p (th ascending)
    while (i > 0 && p < s.th[test][i]) i--;
    return s.id[test][i];
}

__constant__ const double2 *c_termr;     // {fl(1/xd), fl(1/yd)} per term (same index as c_terms)

// floor(n / d) for n < 2^62, 0 < d < 2^32, quotient < 2^40, rd = fl(1/d): double estimate (off by at
// most one), then an exact integer correction.
__device__ __forceinline__ uint64_t fdiv(uint64_t n, uint32_t d, double rd) {
    uint64_t q = (uint64_t)__dmul_rz(__ull2double_rz(n), rd);
    const int64_t r = (int64_t)(n - q * d);
    if (r < 0) q--;
    else if (r >= (int64_t)d) q++;
    return q;
}

// first and count of integers s with x p < s < y p  (x = xn/xd, y = yn/yd), exact; p < 2^32
// (xn p < 2^59), divisions by reciprocal estimate + correction
__device__ __forceinline__ void sum_bounds_r(uint64_t p, const Term &t, double2 rr, uint64_t *first, uint64_t *count) {
    const uint64_t f = fdiv((uint64_t)t.xn * p, t.xd, rr.x) + 1;                  // floor(x p) + 1
    const uint64_t l = fdiv((uint64_t)t.yn * p + t.yd - 1, t.yd, rr.y) - 1;       // ceil(y p) - 1
    *first = f;
    *count = l >= f ? l - f + 1 : 0;
}

// first and count of integers s with x p < s < y p  (x = xn/xd, y = yn/yd), exact.
__device__ __forceinline__ void sum_bounds(uint64_t p, const Term &t, uint64_t *first, uint64_t *count) {
    if (p < (1ull << 32)) {                 // 32-bit divisions; num * rem may exceed 32 bits
        const uint32_t p32 = (uint32_t)p;
        const uint32_t qx = p32 / t.xd, rx = p32 % t.xd, qy = p32 / t.yd, ry = p32 % t.yd;
        const uint64_t fl = (uint64_t)t.xn * qx + ((uint64_t)t.xn * rx) / t.xd;
        const uint64_t ce = (uint64_t)t.yn * qy + ((uint64_t)t.yn * ry + t.yd - 1) / t.yd;
        const uint64_t f = fl + 1, l = ce - 1;
        *first = f;
        *count = l >= f ? l - f + 1 : 0;
        return;
    }
    uint64_t qx = p / t.xd, rx = p % t.xd;
    uint64_t fl = (uint64_t)t.xn * qx + ((uint64_t)t.xn * rx) / t.xd;      // floor(x p)
    uint64_t qy = p / t.yd, ry = p % t.yd;
    uint64_t ce = (uint64_t)t.yn * qy + ((uint64_t)t.yn * ry + t.yd - 1) / t.yd;  // ceil(y p)
    uint64_t f = fl + 1, l = ce - 1;
    *first = f;
    *count = l >= f ? l - f + 1 : 0;
}

// ---------------------------------------------------------------- plan
// One thread per record k = i * ntests + t (i < n_primes read from device).
__global__ void plan_kernel(const uint64_t *__restrict__ primes, const uint64_t *__restrict__ n_primes_dev,
                            uint64_t n_primes_host, uint64_t kmax, uint32_t mode, Sched sched,
                            Rec *__restrict__ recs, uint64_t *__restrict__ nchunks,
                            unsigned long long *__restrict__ first64, int *__restrict__ err,
                            unsigned long long *__restrict__ terms, uint64_t *__restrict__ gq,
                            uint32_t *__restrict__ segidx, uint32_t segstride, uint64_t lane_slice,
                            uint64_t lane_qmax, unsigned long long *__restrict__ lane_total) {
    const uint32_t ntests = (mode == 3) ? 2 : 1;
    const uint64_t n = n_primes_dev ? *n_primes_dev : n_primes_host;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < kmax;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = k / ntests;
        if (i >= n) { nchunks[k] = 0; recs[k].T = 0; recs[k].p = 0; continue; }   // (warp-uniform tail)
        const uint32_t test = (mode == 3) ? (uint32_t)(k % ntests) : (mode == 1 ? 0u : 1u);
        const uint64_t p = primes[i];
        const int cid = schedule(sched, p, (int)test);
        if (cid < 0 || cid >= c_ncong || p < c_cong[cid].min_p || p == c_cong[cid].excluded_p ||
            (test == 0) != (c_cong[cid].e == 3) || p < 5 || p >= (1ull << 62)) {
            atomicExch(err, 1);
            nchunks[k] = 0; recs[k].T = 0; recs[k].p = 0; continue;
        }
        const Cong &c = c_cong[cid];
        // lane mode v2 (class 0): the lane kernel counts its own terms and needs no chunking; only a
        // group's first record computes the group's term count (below)
        const bool lane2rec = lane_total && gq && p < WIDTH32_MAX;
        uint64_t T = 0;
        if (lane2rec) {
        } else if (p < (1ull << 32)) {
            for (uint32_t j = 0; j < c.m; j++) {
                uint64_t f, cnt;
                sum_bounds_r(p, c_terms[c.off + j], c_termr[c.off + j], &f, &cnt);
                T += cnt;
            }
        } else {
            for (uint32_t j = 0; j < c.m; j++) {
                uint64_t f, cnt;
                sum_bounds(p, c_terms[c.off + j], &f, &cnt);
                T += cnt;
            }
        }
        uint64_t L = (T + 32ull * CAP_CHUNKS - 1) / (32ull * CAP_CHUNKS);
        if (L < LMIN) L = LMIN;
        if (L > 0x40000000ull) L = 0x40000000ull;
        uint64_t nc = (T + 32 * L - 1) / (32 * L);
        if (c.seg && !lane2rec) {                      // sum-aligned chunks: ceil(n_j / CT) per sum
            // coarse index (when the stride holds it): segidx[k * segstride + r] = chunks of sums < 32 r
            const uint64_t CT = 32 * L;
            const bool idx = segidx && (c.m + 31) / 32 <= segstride;
            nc = 0;
            for (uint32_t j = 0; j < c.m; j++) {
                if (idx && (j & 31) == 0) segidx[k * segstride + (j >> 5)] = (uint32_t)nc;
                uint64_t f, cnt;
                sum_bounds(p, c_terms[c.off + j], &f, &cnt);
                nc += (cnt + CT - 1) / CT;
            }
        }
        if (gq && p < WIDTH32_MAX) {
            // lane mode: group g = 32 consecutive primes of this test, one per lane; Q slices,
            // Q fixed by the group's last prime so all 32 records agree (T grows with p)
            const uint64_t g = i / 32;
            const uint64_t il = (32 * g + 31 < n) ? 32 * g + 31 : n - 1;
            const uint64_t pl = primes[il];
            const int cl = schedule(sched, pl, (int)test);
            uint64_t Tl = 0;
            if (lane_total) {
                // lane mode v2: the group's term count comes from lane_group_terms_kernel (one warp per group)
            } else if (il == i && cl == cid && !lane2rec) {
                Tl = T;                                          // this record is the group's last prime
            } else if (cl >= 0 && cl < c_ncong) {
                for (uint32_t jj = 0; jj < c_cong[cl].m; jj++) {
                    uint64_t f, cnt;
                    sum_bounds_r(pl, c_terms[c_cong[cl].off + jj], c_termr[c_cong[cl].off + jj], &f, &cnt);
                    Tl += cnt;
                }
            }
            if (lane_total) {
                // deferred: gq = the group's term count (lane_group_terms_kernel), converted to slices by
                // lane_slices_kernel
                nc = 1;
            } else {
                uint64_t Q = (Tl + lane_slice - 1) / lane_slice;
                if (Q < 1) Q = 1;
                if (Q > lane_qmax) Q = lane_qmax;
                nc = Q;
                if (i == 32 * g) gq[g * ntests + (mode == 3 ? test : 0)] = Q;
            }
        }
        Rec r;
        r.p = p; r.T = T; r.cid = (uint32_t)cid; r.L = (uint32_t)L; r.idx = (uint32_t)i; r.test = test;
        recs[k] = r;
        nchunks[k] = nc;
        if (p >= WIDTH32_MAX && nc > 0) atomicMin(first64, (unsigned long long)k);
        if (p >= FP64_MAX && nc > 0) atomicMin(first64 + 1, (unsigned long long)k);
        if (!lane2rec) atomicAdd(&terms[prime_class(p)], (unsigned long long)T);
    }
    // lane-mode groups whose first prime is not class 0 (or beyond n) get Q = 0
    if (gq) {
        const uint64_t ngt = ((kmax / ntests + 31) / 32) * ntests;
        for (uint64_t gt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; gt < ngt;
             gt += (uint64_t)gridDim.x * blockDim.x) {
            const uint64_t i0 = (gt / ntests) * 32;
            if (i0 >= n || primes[i0] >= WIDTH32_MAX) gq[gt] = 0;
        }
    }
}

// Lane mode v2, after plan_kernel: the term count of each class-0 group-test (the group's last prime, whose
// congruence and counts bound the group's), one warp per group-test with the lanes striding over the
// sums -> gq[gt], and their total -> lane_total.  Groups plan_kernel marked non-class-0 (gq = 0) are skipped.
__global__ void lane_group_terms_kernel(const uint64_t *__restrict__ primes, const uint64_t *__restrict__ n_primes_dev,
                                        uint64_t n_primes_host, uint32_t mode, Sched sched, uint64_t ngt,
                                        uint64_t *__restrict__ gq, unsigned long long *__restrict__ lane_total) {
    const uint32_t ntests = (mode == 3) ? 2 : 1;
    const uint64_t n = n_primes_dev ? *n_primes_dev : n_primes_host;
    const int lane = threadIdx.x & 31;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t gt = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; gt < ngt; gt += nw) {
        const uint64_t i0 = 32 * (gt / ntests);
        if (i0 >= n || primes[i0] >= WIDTH32_MAX) continue;          // warp-uniform
        const uint32_t test = (mode == 3) ? (uint32_t)(gt % ntests) : (mode == 1 ? 0u : 1u);
        const uint64_t pl = primes[i0 + 31 < n ? i0 + 31 : n - 1];
        const int cl = schedule(sched, pl, (int)test);
        uint64_t Tl = 0;
        if (cl >= 0 && cl < c_ncong) {
            const Cong &c = c_cong[cl];
            for (uint32_t jj = lane; jj < c.m; jj += 32) {
                uint64_t f, cnt;
                sum_bounds_r(pl, c_terms[c.off + jj], c_termr[c.off + jj], &f, &cnt);
                Tl += cnt;
            }
        }
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) Tl += __shfl_xor_sync(0xffffffffu, Tl, o);
        if (lane == 0) {
            gq[gt] = Tl;
            atomicAdd(lane_total, (unsigned long long)Tl);
        }
    }
}

// Lane mode v2: slices per group-test from its term count Tl (gq on entry): one slice size for the
// whole launch, total / (items wanted), so large groups are cut finer and small ones stay whole.
// Sets gq[gt] = Q and the slot count of each class-0 record of the group.
__global__ void lane_slices_kernel(uint64_t *__restrict__ gq, uint64_t ngt, uint32_t ntests, const Rec *__restrict__ recs,
                                   uint64_t K, uint64_t *__restrict__ nchunks,
                                   const unsigned long long *__restrict__ lane_total, double items_wanted,
                                   uint64_t min_slice, uint64_t qmax, unsigned long long *__restrict__ counts) {
    // one warp per group-test: lane l owns record (32 g + l) ntests + t.
    // counts[0] += group-tests cut into Q > 1 slices, counts[1] += lane-mode group-tests
    const double tot = (double)*lane_total;
    uint64_t slice = (uint64_t)ceil(tot / (items_wanted > 1.0 ? items_wanted : 1.0));
    if (slice < min_slice) slice = min_slice;
    const int lane = threadIdx.x & 31;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t gt = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; gt < ngt; gt += nw) {
        const uint64_t Tl = gq[gt];
        __syncwarp();
        if (Tl == 0) continue;                       // not a lane-mode group (warp-uniform)
        uint64_t Q = (Tl + slice - 1) / slice;
        if (Q < 1) Q = 1;
        if (Q > qmax) Q = qmax;
        if (lane == 0) {
            gq[gt] = Q;
            if (counts) {
                atomicAdd(&counts[1], 1ull);
                if (Q > 1) atomicAdd(&counts[0], 1ull);
            }
        }
        const uint64_t g = gt / ntests, t = gt % ntests;
        const uint64_t k = (32 * g + lane) * ntests + t;
        if (k < K) {
            const uint64_t p = recs[k].p;
            if (p != 0 && p < WIDTH32_MAX) nchunks[k] = Q;
        }
    }
}

// item g -> record k: the largest k in [klo, khi) with start[k] <= g
__device__ __forceinline__ uint64_t find_rec(const uint64_t *__restrict__ start, uint64_t klo, uint64_t khi, uint64_t g) {
    uint64_t lo = klo, hi = khi;          // invariant: start[lo] <= g, answer in [lo, hi)
    while (hi - lo > 1) {
        uint64_t mid = (lo + hi) >> 1;
        if (start[mid] <= g) lo = mid; else hi = mid;
    }
    return lo;
}

// Same result, warp-cooperative (all 32 lanes, g warp-uniform): a 32-ary search, each round
// probing 31 cut points at once -- log32 rounds of loads instead of log2 dependent ones.
__device__ __forceinline__ uint64_t find_rec_warp(const uint64_t *__restrict__ start, uint64_t klo, uint64_t khi,
                                                  uint64_t g) {
    const int lane = threadIdx.x & 31;
    uint64_t lo = klo, hi = khi;          // invariant: start[lo] <= g < start[hi] (start[khi] = end)
    while (hi - lo > 32) {
        const uint64_t step = (hi - lo + 31) / 32;
        const uint64_t idx = lo + (uint64_t)lane * step;             // lane 0 probes lo itself
        const bool ok = idx < hi && start[idx] <= g;
        const uint32_t m = __ballot_sync(0xffffffffu, ok);           // prefix of lanes (start ascending)
        const int last = 31 - __clz(m);
        const uint64_t nlo = lo + (uint64_t)last * step;
        const uint64_t nhi = nlo + step < hi ? nlo + step : hi;
        lo = nlo;
        hi = nhi;
    }
    const uint64_t idx = lo + lane;
    const bool ok = idx < hi && start[idx] <= g;
    const uint32_t m = __ballot_sync(0xffffffffu, ok);
    return lo + (31 - __clz(m));
}

// ---------------------------------------------------------------- term runs
// A "run" is the state of consecutive terms s, s+1, ... of one sum: u = s^E,
// its forward differences, and the pair (a0, a1) of prod (z + u).  Two
// engines implement the same interface (setup / step / reduce / result):
//   Run<M,E>  -- Montgomery products on the IMAD pipe (lazy values in [0,2p));
//   RunD<E>   -- exact FP64 error-free-transform products (ModD, p < 2^44) on
//                the DFMA pipe, balanced values, periodic range reduction.
template <class M, int E>
struct Run {
    // u = s^E is kept as a plain residue (lazy [0, 2p)), not in Montgomery form.  The products
    // a1 <- REDC(a1 u + a0 R), a0 <- REDC(a0 u) then scale the ratio a1/a0 by R at every term
    // (a1/a0 -> a1/a0 + R/u), so result() returns c1 = a1 R^{-1}.  For E = 2 this makes
    // d1 = 2s + 1 (< 2p) and d2 = 2 plain integers that never need a reduction.
    using W = typename M::W;
    static constexpr bool kFP = false;
    W u, d1, d2, d3, a0, a1;
    __device__ __forceinline__ void setup(const M &mo, const ModD &, uint64_t s0) {   // s0 < p
        const W sm = mo.mul((W)s0, mo.r2);                         // s R
        const W s2m = mo.mul(sm, sm);                              // s^2 R
        const W s = (W)s0;
        if (E == 3) {
            u = mo.mul(mo.mul(s2m, sm), (W)1);                     // s^3
            const W s2 = mo.mul(s2m, (W)1);                        // s^2
            const W s2x3 = mo.add(mo.add(s2, s2), s2);
            const W sx3 = mo.add(mo.add(s, s), s);
            d1 = mo.add(mo.add(s2x3, sx3), (W)1);                  // 3s^2 + 3s + 1
            const W sx6 = mo.add(sx3, sx3);
            d2 = mo.add(sx6, (W)6);                                // 6s + 6
            d3 = 6;
        } else {
            u = mo.mul(s2m, (W)1);                                 // s^2
            d1 = 2 * s + 1;                                        // 2s + 1 < 2p, plain
            d2 = 2;
            d3 = 0;
        }
        a0 = mo.r1;
        a1 = 0;
    }
    // one term of eqnComputeS: a1 <- a1 u + a0; a0 <- a0 u; then s <- s + 1
    __device__ __forceinline__ void step(const M &mo, const ModD &) {
        a1 = mo.muladd(a1, u, a0);
        a0 = mo.mul(a0, u);
        u = mo.add(u, d1);
        if (E == 3) {
            d1 = mo.add(d1, d2);
            d2 = mo.add(d2, d3);
        } else {
            d1 += d2;
        }
    }
    // two terms at once: 1/u1 + 1/u2 = (u1 + u2) / (u1 u2), so with D = u1 u2, N = u1 + u2:
    //   a1 <- a1 D + a0 N  (one REDC for both products),  a0 <- a0 D
    // 5 Montgomery-product halves instead of 6 for the pair (PAIRS engines only).  For Mont32
    // N < 4p is left unreduced (mul2add: 2p 2p + 2p 4p + m p < 2^64 for p < 2^30).
    __device__ __forceinline__ void step2(const M &mo, const ModD &) {
        const W u2 = mo.add(u, d1);
        if (E == 3) {
            d1 = mo.add(d1, d2);
            d2 = mo.add(d2, d3);
        } else {
            d1 += d2;
        }
        const W N = sizeof(W) == 4 ? u + u2 : mo.add(u, u2);     // Mont64 (p up to 2^62): reduce
        const W D = mo.mul(u, u2);
        u = mo.add(u2, d1);
        if (E == 3) {
            d1 = mo.add(d1, d2);
            d2 = mo.add(d2, d3);
        } else {
            d1 += d2;
        }
        a1 = mo.mul2add(a1, D, a0, N);
        a0 = mo.mul(a0, D);
    }
    // a step whose (a0, a1) update only lands on lanes with act (the differences always advance)
    __device__ __forceinline__ void step_masked(const M &mo, const ModD &, bool act) {
        const W n1 = mo.muladd(a1, u, a0);
        const W n0 = mo.mul(a0, u);
        a1 = act ? n1 : a1;
        a0 = act ? n0 : a0;
        u = mo.add(u, d1);
        if (E == 3) {
            d1 = mo.add(d1, d2);
            d2 = mo.add(d2, d3);
        } else {
            d1 += d2;
        }
    }
    __device__ __forceinline__ void reduce(const ModD &) {}
    __device__ __forceinline__ void result(const M &mo, const ModD &, W &c0, W &c1) const {
        c0 = a0;
        c1 = mo.mul(a1, (W)1);                   // undo the factor R the plain u puts on a1/a0
    }
    // sum-start state (u, d1, d2) to / from shared memory; coefficient rescaling at a sum switch
    __device__ __forceinline__ void save_start(uint64_t *st) const { st[0] = u; st[1] = d1; st[2] = d2; }
    __device__ __forceinline__ void load_start(const uint64_t *st) { u = (W)st[0]; d1 = (W)st[1]; d2 = (W)st[2]; }
    // cross from sum j to j+1: keep V = a_{j+1} a1 / a0 by a1 <- a_j a1, a0 <- a_{j+1} a0
    __device__ __forceinline__ void scale2(const M &mo, const ModD &, uint64_t cj_m, uint64_t cn_m, uint64_t,
                                           uint64_t) {
        a1 = mo.mul(a1, (W)cj_m);
        a0 = mo.mul(a0, (W)cn_m);
    }
};

template <class M, int E>
struct RunD {
    using W = typename M::W;
    static constexpr bool kFP = true;
    double u, d1, d2, a0, a1;
    __device__ __forceinline__ void setup(const M &, const ModD &md, uint64_t s0) {   // s0 < p/2
        const double s = (double)s0;
        if (E == 3) {
            const double s2 = md.mul(s, s);                                    // |s2| <= p
            u = md.mul(s2, s);
            d1 = md.reduce(__fma_rn(3.0, __dadd_rn(s2, s), 1.0));              // 3s^2 + 3s + 1 (< 2^47: exact)
            d2 = __fma_rn(6.0, s, 6.0);                                        // 6s + 6, exact
        } else {
            u = md.mul(s, s);
            d1 = __fma_rn(2.0, s, 1.0);                                        // 2s + 1 < p, exact
            d2 = 2.0;
        }
        a0 = 1.0;
        a1 = 0.0;
    }
    __device__ __forceinline__ void step(const M &, const ModD &md) {
        a1 = __dadd_rn(md.mul(a1, u), a0);       // |a1| <= 2p
        a0 = md.mul(a0, u);                      // |a0| <= p
        u = __dadd_rn(u, d1);
        d1 = __dadd_rn(d1, d2);
        if (E == 3) d2 = __dadd_rn(d2, 6.0);
    }
    __device__ __forceinline__ void step2(const M &mo, const ModD &md) { step(mo, md); step(mo, md); }
    __device__ __forceinline__ void step_masked(const M &, const ModD &md, bool act) {
        const double n1 = __dadd_rn(md.mul(a1, u), a0);
        const double n0 = md.mul(a0, u);
        a1 = act ? n1 : a1;
        a0 = act ? n0 : a0;
        u = __dadd_rn(u, d1);
        d1 = __dadd_rn(d1, d2);
        if (E == 3) d2 = __dadd_rn(d2, 6.0);
    }
    __device__ __forceinline__ void reduce(const ModD &md) {
        u = md.reduce(u);
        if (E == 3) d1 = md.reduce(d1);
    }
    __device__ __forceinline__ void result(const M &mo, const ModD &md, W &c0, W &c1) const {
        c0 = mo.mul((W)md.canon(a0), mo.r2);     // into the combine domain (Montgomery form)
        c1 = mo.mul((W)md.canon(a1), mo.r2);
    }
    __device__ __forceinline__ void save_start(uint64_t *st) const {
        st[0] = (uint64_t)__double_as_longlong(u);
        st[1] = (uint64_t)__double_as_longlong(d1);
        st[2] = (uint64_t)__double_as_longlong(d2);
    }
    __device__ __forceinline__ void load_start(const uint64_t *st) {
        u = __longlong_as_double((long long)st[0]);
        d1 = __longlong_as_double((long long)st[1]);
        d2 = __longlong_as_double((long long)st[2]);
    }
    __device__ __forceinline__ void scale2(const M &, const ModD &md, uint64_t, uint64_t, uint64_t cj_c,
                                           uint64_t cn_c) {
        a1 = md.mul(a1, (double)cj_c);          // |a1| <= 2p, coefficient < p: |result| <= p
        a0 = md.mul(a0, (double)cn_c);
    }
};

// FP64 engine, K terms per step (sum-aligned chunks, 2^30 <= p < 2^44):
//     1/u_0 + ... + 1/u_{K-1} = N / D,  u_i = (s+i)^E,
//     D(s) = (s (s+1) ... (s+K-1))^E  (degree KE),   N(s) = sum_i prod_{j != i} u_j  (degree (K-1)E),
// advanced by step-K forward differences held as exact integers in doubles.  Per step:
// a1 <- a1 D + a0 N, a0 <- a0 D (3 exact EFT products, ModD) and (2K-1)E additions, against
// K x (2 products + E additions) term by term.  Balanced values grow under the additions; every `rb`
// steps all non-constant table entries are range-reduced, rb the largest with
// p sum_{i <= KE} C(rb, i) <= 2^49 (then |D_0|, |N_0| <= 2^49 as ModD::mul needs, and every entry
// stays an exact integer).
template <int E, int K>
struct RunDK {
    static constexpr int DD = K * E, DN = (K - 1) * E;
    double D[DD + 1], N[DN + 1], a0, a1;
    __device__ __forceinline__ void setup(const ModD &md, uint64_t x) {     // x < p/2
        const double s = (double)x;
        double u, d1, d2;
        if (E == 3) {
            const double s2 = md.mul(s, s);
            u = md.mul(s2, s);
            d1 = md.reduce(__fma_rn(3.0, __dadd_rn(s2, s), 1.0));           // 3s^2 + 3s + 1
            d2 = __fma_rn(6.0, s, 6.0);                                        // 6s + 6
        } else {
            u = md.mul(s, s);
            d1 = __fma_rn(2.0, s, 1.0);
            d2 = 2.0;
        }
        #pragma unroll
        for (int i = 0; i <= DD; i++) {
            double q[K], pre[K + 1], suf[K];
            #pragma unroll
            for (int k = 0; k < K; k++) {
                q[k] = u;
                u = md.reduce(__dadd_rn(u, d1));
                d1 = __dadd_rn(d1, d2);
                if (E == 3) { d1 = md.reduce(d1); d2 = __dadd_rn(d2, 6.0); }
            }
            pre[1] = q[0];
            #pragma unroll
            for (int k = 1; k < K; k++) pre[k + 1] = md.mul(pre[k], q[k]);
            D[i] = pre[K];
            if (i <= DN) {
                suf[K - 1] = q[K - 1];
                #pragma unroll
                for (int k = K - 2; k >= 1; k--) suf[k] = md.mul(suf[k + 1], q[k]);
                double n = suf[1];                                             // prod_{j != 0}
                #pragma unroll
                for (int k = 1; k < K - 1; k++) n = md.reduce(__dadd_rn(n, md.mul(pre[k], suf[k + 1])));
                N[i] = md.reduce(__dadd_rn(n, pre[K - 1]));                    // prod_{j != K-1}
            }
        }
        #pragma unroll
        for (int k = 1; k <= DD; k++) {
            #pragma unroll
            for (int i = DD; i >= k; i--) D[i] = md.reduce(__dadd_rn(D[i], -D[i - 1]));
        }
        #pragma unroll
        for (int k = 1; k <= DN; k++) {
            #pragma unroll
            for (int i = DN; i >= k; i--) N[i] = md.reduce(__dadd_rn(N[i], -N[i - 1]));
        }
        a0 = 1.0;
        a1 = 0.0;
    }
    template <bool MASK>
    __device__ __forceinline__ void step(const ModD &md, bool act) {
        const double n1 = __dadd_rn(md.mul(a1, D[0]), md.mul(a0, N[0]));   // |a1| <= 2p
        const double n0 = md.mul(a0, D[0]);
        a1 = (!MASK || act) ? n1 : a1;
        a0 = (!MASK || act) ? n0 : a0;
        #pragma unroll
        for (int i = 0; i < DD; i++) D[i] = __dadd_rn(D[i], D[i + 1]);
        #pragma unroll
        for (int i = 0; i < DN; i++) N[i] = __dadd_rn(N[i], N[i + 1]);
    }
    __device__ __forceinline__ void reduce(const ModD &md) {
        #pragma unroll
        for (int i = 0; i < DD; i++) D[i] = md.reduce(D[i]);
        #pragma unroll
        for (int i = 0; i < DN; i++) N[i] = md.reduce(N[i]);
    }
    // one term s = x, masked (u recomputed: masked steps advanced the tables of every lane)
    __device__ __forceinline__ void single(const ModD &md, uint64_t x, bool act) {
        const double s = (double)x;
        const double w = E == 3 ? md.mul(md.mul(s, s), s) : md.mul(s, s);
        const double n1 = __dadd_rn(md.mul(a1, w), a0);
        const double n0 = md.mul(a0, w);
        a1 = act ? n1 : a1;
        a0 = act ? n0 : a0;
    }
};

// steps between range reductions of a RunDK table (see above), for the warp's largest p
template <int DD>
__device__ __forceinline__ uint32_t rundk_interval(uint64_t p) {
    const double budget = 562949953421312.0 / (double)p;    // 2^49 / p
    double c = 1.0, g = 1.0;                                 // C(r, i) running terms; g = sum_{i <= DD} C(r, i)
    uint32_t r = 0;
    for (;;) {                                               // g(r + 1) = sum_{i <= DD} C(r + 1, i)
        const uint32_t rn = r + 1;
        double gn = 0.0;
        c = 1.0;
        for (int i = 0; i <= DD && i <= (int)rn; i++) {
            gn += c;
            c = c * (double)(rn - i) / (double)(i + 1);
        }
        if (gn > budget || rn > 64) break;
        r = rn;
        g = gn;
    }
    (void)g;
    return r ? r : 1;
}

template <class M, int E, int K>
__device__ __forceinline__ void fp_tuple_work(const M &mo, const ModD &md, uint64_t p, uint64_t x0, uint64_t n,
                                              typename M::W coef_m, typename M::W &C0, typename M::W &C1) {
    using W = typename M::W;
    const uint64_t ns = n / K, rem = n - K * ns;
    const bool act = n != 0;
    const uint64_t kmin = __reduce_min_sync(0xffffffffu, act ? (uint32_t)ns : 0xffffffffu);
    if (kmin == 0xffffffffu) return;
    const uint64_t kmax = __reduce_max_sync(0xffffffffu, act ? (uint32_t)ns : 0u);
    const uint32_t rmax = __reduce_max_sync(0xffffffffu, (uint32_t)rem);
    const uint32_t rb = __reduce_min_sync(0xffffffffu, rundk_interval<K * E>(p));
    RunDK<E, K> run;
    run.setup(md, act ? x0 : 1);
    uint32_t since = 0;
    uint64_t i = 0;
    #pragma unroll 1
    for (; i < kmin; i++) {
        run.template step<false>(md, true);
        if (++since == rb) { run.reduce(md); since = 0; }
    }
    #pragma unroll 1
    for (; i < kmax; i++) {
        run.template step<true>(md, i < ns);
        if (++since == rb) { run.reduce(md); since = 0; }
    }
    for (uint32_t r = 0; r < rmax; r++) run.single(md, x0 + K * ns + r, r < rem);
    if (act) {
        W c0 = mo.mul((W)md.canon(run.a0), mo.r2);     // into the combine domain (Montgomery form)
        W c1 = mo.mul((W)md.canon(run.a1), mo.r2);
        c1 = mo.mul(c1, coef_m);                        // fold a_j
        typename M::W n1 = mo.add(mo.mul(C0, c1), mo.mul(C1, c0));
        C0 = mo.mul(C0, c0);
        C1 = n1;
    }
}

// ---------------------------------------------------------------- class 2: Mont64 K-term steps
// The same K-term step as RunDK (a1 <- a1 D + a0 N, a0 <- a0 D; D, N polynomials of degree Ke, (K-1)e in s
// advanced by step-K forward differences) in 64-bit Montgomery arithmetic (R = 2^64, p < 2^62), for the
// primes no narrower engine covers (p >= 2^44).  A 64-bit product costs ~20 IMAD-class instructions
// (32-bit limbs), so the tables are *lazy*: plain 64-bit additions (two instructions, no compare /
// select) and a Barrett reduction of every entry to [0, 2p) at most rb steps apart, rb = 63 - bitlen(p)
// (capped at 16): after n unreduced steps an entry is a binomial-weighted sum of entries < 2p, so it is
// < 2p 2^n <= 2^64.  Only D_0 and N_0 enter products, through mulr (b may be any 64-bit value).
template <int E, int K>
struct RunMK {
    static constexpr int DD = K * E, DN = (K - 1) * E;
    uint64_t D[DD + 1], N[DN + 1], a0, a1;
    static __device__ __forceinline__ uint64_t red2(const Mont64 &mo, uint64_t t) {   // [0, 3p) -> [0, 2p)
        return t >= mo.p2 ? t - mo.p2 : t;
    }
    // a b R^{-1} for a < 2p and any 64-bit b: (a b + m p) / R < 2p + p, one conditional subtract
    static __device__ __forceinline__ uint64_t mulr(const Mont64 &mo, uint64_t a, uint64_t b) {
        return red2(mo, mo.mul(a, b));
    }
    static __device__ __forceinline__ uint64_t sub(const Mont64 &mo, uint64_t a, uint64_t b) {  // [0, 2p)
        const uint64_t s = a + mo.p2 - b;                                                       // (0, 4p)
        return s >= mo.p2 ? s - mo.p2 : s;
    }
    // x < 2^64 -> [0, 2p), same residue: q = hi(x mu), mu = floor(2^64 / p), is floor(x / p) or one less
    static __device__ __forceinline__ uint64_t bred(const Mont64 &mo, uint64_t mu, uint64_t x) {
        return x - __umul64hi(x, mu) * mo.p;
    }
    __device__ __forceinline__ void setup(const Mont64 &mo, uint64_t x) {   // x < p
        const uint64_t xt = mo.to(x), xx = mo.mul(xt, xt);
        uint64_t u, d1, d2, d3 = 0;
        if (E == 3) {
            const uint64_t r3 = mo.add(mo.add(mo.r1, mo.r1), mo.r1), x3 = mo.add(mo.add(xt, xt), xt);
            u = mo.mul(xx, xt);                                                // x^3
            d1 = mo.add(mo.add(mo.add(xx, xx), xx), mo.add(x3, mo.r1));        // 3x^2 + 3x + 1
            d3 = mo.add(r3, r3);                                               // 6
            d2 = mo.add(mo.add(x3, x3), d3);                                   // 6x + 6
        } else {
            u = xx;                                                            // x^2
            d1 = mo.add(mo.add(xt, xt), mo.r1);                                // 2x + 1
            d2 = mo.add(mo.r1, mo.r1);                                         // 2
        }
        #pragma unroll
        for (int i = 0; i <= DD; i++) {
            uint64_t q[K], pre[K + 1], suf[K + 1];
            #pragma unroll
            for (int k = 0; k < K; k++) {
                q[k] = u;
                u = mo.add(u, d1);
                d1 = mo.add(d1, d2);
                if (E == 3) d2 = mo.add(d2, d3);
            }
            pre[1] = q[0];
            #pragma unroll
            for (int k = 1; k < K; k++) pre[k + 1] = mo.mul(pre[k], q[k]);
            D[i] = pre[K];
            if (i <= DN) {
                suf[K - 1] = q[K - 1];
                #pragma unroll
                for (int k = K - 2; k >= 1; k--) suf[k] = mo.mul(suf[k + 1], q[k]);
                uint64_t n = mo.add(suf[1], pre[K - 1]);                       // prod_{j != 0} + prod_{j != K-1}
                #pragma unroll
                for (int k = 1; k < K - 1; k++) n = mo.add(n, mo.mul(pre[k], suf[k + 1]));
                N[i] = n;
            }
        }
        #pragma unroll
        for (int k = 1; k <= DD; k++) {
            #pragma unroll
            for (int i = DD; i >= k; i--) D[i] = sub(mo, D[i], D[i - 1]);
        }
        #pragma unroll
        for (int k = 1; k <= DN; k++) {
            #pragma unroll
            for (int i = DN; i >= k; i--) N[i] = sub(mo, N[i], N[i - 1]);
        }
        a0 = mo.r1;
        a1 = 0;
    }
    template <bool MASK>
    __device__ __forceinline__ void step(const Mont64 &mo, bool act) {
        const uint64_t n1 = mo.add(mulr(mo, a1, D[0]), mulr(mo, a0, N[0]));
        const uint64_t n0 = mulr(mo, a0, D[0]);
        a1 = (!MASK || act) ? n1 : a1;
        a0 = (!MASK || act) ? n0 : a0;
        #pragma unroll
        for (int i = 0; i < DD; i++) D[i] += D[i + 1];
        #pragma unroll
        for (int i = 0; i < DN; i++) N[i] += N[i + 1];
    }
    __device__ __forceinline__ void reduce(const Mont64 &mo, uint64_t mu) {
        #pragma unroll
        for (int i = 0; i < DD; i++) D[i] = bred(mo, mu, D[i]);
        #pragma unroll
        for (int i = 0; i < DN; i++) N[i] = bred(mo, mu, N[i]);
    }
    __device__ __forceinline__ void single(const Mont64 &mo, uint64_t x, bool act) {   // one term s = x
        const uint64_t xt = mo.to(x), x2 = mo.mul(xt, xt);
        const uint64_t w = E == 3 ? mo.mul(x2, xt) : x2;
        const uint64_t n1 = mo.add(mo.mul(a1, w), a0);
        const uint64_t n0 = mo.mul(a0, w);
        a1 = act ? n1 : a1;
        a0 = act ? n0 : a0;
    }
};

// lane's run [x0, x0 + n) of one sum with Mont64 K-term steps, folded with a_j and merged into (C0, C1)
template <int E, int K>
__device__ __forceinline__ void int_tuple_work(const Mont64 &mo, uint64_t p, uint64_t x0, uint64_t n, uint64_t coef_m,
                                               uint64_t &C0, uint64_t &C1) {
    const uint64_t ns = n / K, rem = n - K * ns;
    const bool act = n != 0;
    const uint64_t kmin = __reduce_min_sync(0xffffffffu, act ? (uint32_t)ns : 0xffffffffu);
    if (kmin == 0xffffffffu) return;
    const uint64_t kmax = __reduce_max_sync(0xffffffffu, act ? (uint32_t)ns : 0u);
    const uint32_t rmax = __reduce_max_sync(0xffffffffu, (uint32_t)rem);
    const int bl = 64 - __clzll(p);
    const uint32_t rb = __reduce_min_sync(0xffffffffu, bl >= 62 ? 1u : (63 - bl > 16 ? 16u : (uint32_t)(63 - bl)));
    const uint64_t mu = ~0ull / p;                                            // floor((2^64 - 1) / p) = floor(2^64 / p)
    RunMK<E, K> run;
    run.setup(mo, act ? x0 : 1);
    uint32_t since = 0;
    uint64_t i = 0;
    #pragma unroll 1
    for (; i < kmin; i++) {
        run.template step<false>(mo, true);
        if (++since == rb) { run.reduce(mo, mu); since = 0; }
    }
    #pragma unroll 1
    for (; i < kmax; i++) {
        run.template step<true>(mo, i < ns);
        if (++since == rb) { run.reduce(mo, mu); since = 0; }
    }
    for (uint32_t r = 0; r < rmax; r++) run.single(mo, x0 + K * ns + r, r < rem);
    if (act) {
        const uint64_t c1 = mo.mul(run.a1, coef_m);                          // fold a_j
        const uint64_t n1 = mo.add(mo.mul(C0, c1), mo.mul(C1, run.a0));      // eqnCombinePairs
        C0 = mo.mul(C0, run.a0);
        C1 = n1;
    }
}

template <class M>
__device__ __forceinline__ void combine(const M &mo, typename M::W &C0, typename M::W &C1,
                                        typename M::W c0, typename M::W c1) {
    typename M::W n1 = mo.add(mo.mul(C0, c1), mo.mul(C1, c0));
    C0 = mo.mul(C0, c0);
    C1 = n1;
}

constexpr int RES_THREADS = 256;
constexpr int RES_WARPS = RES_THREADS / 32;

// One lane's terms [t0, t1) of the record's flattened term space, split into S
// contiguous "streams" (independent runs interleaved in one instruction stream
// for ILP: a single Montgomery stream is dependency-latency bound on sm_100a).
// All lanes and streams advance by the same count k = the minimum, over the
// warp, of the terms left in any active run (__reduce_min_sync), so the hot
// loop never diverges; only the switch to the next sum (fold a_j, merge,
// re-seed u and its differences) runs where a run ended.  Finished streams keep
// stepping on dead state (ignored).  The FP64 engine range-reduces its u (and
// d1) every rb terms, counted warp-uniformly.
// Per-warp item tables in shared memory (contiguous chunking, up to MAX_CONTIG_M sums).
struct WarpTab {
    uint64_t first[MAX_CONTIG_M];       // first s of each sum
    uint64_t cum[MAX_CONTIG_M + 1];     // prefix counts (flattened term space)
    uint64_t coef[MAX_CONTIG_M];        // a_j mod p, Montgomery form
    uint64_t st[MAX_CONTIG_M][3];       // run state (u, d1, d2) at s = first_j
    uint64_t coefc[MAX_CONTIG_M];       // a_j mod p, canonical (FP64 engine)
    uint32_t cont;                      // 1: every a_j is a unit mod p -> continuous runs across sums
};

// Fill st[] (and coefc[]) warp-cooperatively for the continuous switch: a stream that leaves
// sum j at its end enters sum j+1 at its start, so it loads that sum's start state and keeps
// V = a_{j+1} a1 / a0 invariant by a1 <- a_j a1, a0 <- a_{j+1} a0 -- no merge, no re-seed and
// no modular inverse.  Requires every a_j to be a unit mod p (else tab.cont = 0: merge path).
template <class M, class R>
__device__ __forceinline__ void prepare_switch(const M &mo, const ModD &md, WarpTab &tb, uint32_t m) {
    using W = typename M::W;
    const int lane = threadIdx.x & 31;
    bool unit = true;
    for (uint32_t j = lane; j < m; j += 32) {
        R tmp;
        tmp.setup(mo, md, tb.first[j]);
        tmp.save_start(tb.st[j]);
        const uint64_t cc = mo.canon((W)tb.coef[j]);
        tb.coefc[j] = cc;
        unit = unit && cc != 0;
    }
    const bool all = __all_sync(0xffffffffu, unit);
    if (lane == 0) tb.cont = all ? 1u : 0u;
    __syncwarp();
}

template <class M, class R, int E, int S, bool PAIRS>
__device__ __forceinline__ void lane_work(const M &mo, const ModD &md, const WarpTab &tab, uint64_t p,
                                          uint64_t t0, uint64_t t1, typename M::W &C0, typename M::W &C1) {
    using W = typename M::W;
    const uint64_t *coefm = tab.coef, *first = tab.first, *cum = tab.cum;
    const bool cont = tab.cont != 0;
    R run[S];
    uint32_t j[S], nrun[S];
    uint64_t t[S], te[S];
    const uint32_t rb = R::kFP ? (E == 3 ? md.rb3 : md.rb2) : 0xffffffffu;
    uint32_t since = 0;
    const uint64_t len = t1 > t0 ? t1 - t0 : 0;
    const uint64_t q = (len + S - 1) / S;
    #pragma unroll
    for (int i = 0; i < S; i++) {
        t[i] = t0 + i * q;
        te[i] = t[i] + q < t1 ? t[i] + q : t1;
        j[i] = 0;
        nrun[i] = 0;
        if (t[i] < te[i]) {
            while (cum[j[i] + 1] <= t[i]) j[i]++;
            nrun[i] = (uint32_t)((te[i] < cum[j[i] + 1] ? te[i] : cum[j[i] + 1]) - t[i]);
            run[i].setup(mo, md, first[j[i]] + (t[i] - cum[j[i]]));
        } else {
            run[i].setup(mo, md, 1);          // dead stream: defined state
        }
    }
    for (;;) {
        uint32_t mn = 0xffffffffu;
        #pragma unroll
        for (int i = 0; i < S; i++)
            if (nrun[i] && nrun[i] < mn) mn = nrun[i];
        const uint32_t k = __reduce_min_sync(0xffffffffu, mn);
        if (k == 0xffffffffu) break;
        // (batching run switches behind a window of masked steps was measured slower on C2:
        //  23.4 ms unbatched vs 24.7 / 25.7 / 27.2 ms with 16 / 32 / 64-step windows)
        uint32_t left = k;
        while (left) {
            const uint32_t kk = left < rb - since ? left : rb - since;
            uint32_t i = 0;
            if (PAIRS) {
                #pragma unroll 1
                for (; i + 4 <= kk; i += 4) {
                    #pragma unroll
                    for (int u = 0; u < 2; u++) {
                        #pragma unroll
                        for (int s_ = 0; s_ < S; s_++) run[s_].step2(mo, md);
                    }
                }
            } else {
                #pragma unroll 1
                for (; i + 4 <= kk; i += 4) {
                    #pragma unroll
                    for (int u = 0; u < 4; u++) {
                        #pragma unroll
                        for (int s_ = 0; s_ < S; s_++) run[s_].step(mo, md);
                    }
                }
            }
            if (PAIRS && i + 2 <= kk) {                // remainder: at most one pair + one single step
                #pragma unroll
                for (int s_ = 0; s_ < S; s_++) run[s_].step2(mo, md);
                i += 2;
            }
            for (; i < kk; i++) {
                #pragma unroll
                for (int s_ = 0; s_ < S; s_++) run[s_].step(mo, md);
            }
            left -= kk;
            if (R::kFP) {
                since += kk;
                if (since == rb) {
                    #pragma unroll
                    for (int s_ = 0; s_ < S; s_++) run[s_].reduce(md);
                    since = 0;
                }
            }
        }
        #pragma unroll
        for (int i = 0; i < S; i++) {
            if (!nrun[i]) continue;
            nrun[i] -= k;
            t[i] += k;
            if (nrun[i] == 0) {
                if (cont && t[i] < te[i]) {
                    // continuous switch: enter the next non-empty sum at its start
                    do {
                        run[i].scale2(mo, md, tab.coef[j[i]], tab.coef[j[i] + 1], tab.coefc[j[i]], tab.coefc[j[i] + 1]);
                        j[i]++;
                    } while (cum[j[i] + 1] <= t[i]);
                    run[i].load_start(tab.st[j[i]]);
                    nrun[i] = (uint32_t)((te[i] < cum[j[i] + 1] ? te[i] : cum[j[i] + 1]) - t[i]);
                } else {
                    W c0, c1;
                    run[i].result(mo, md, c0, c1);
                    c1 = mo.mul(c1, (W)coefm[j[i]]);                               // fold a_j (Montgomery form)
                    combine(mo, C0, C1, c0, c1);
                    if (t[i] < te[i]) {
                        j[i]++;
                        while (cum[j[i] + 1] <= t[i]) j[i]++;
                        nrun[i] = (uint32_t)((te[i] < cum[j[i] + 1] ? te[i] : cum[j[i] + 1]) - t[i]);
                        run[i].setup(mo, md, first[j[i]] + (t[i] - cum[j[i]]));
                    }
                }
            }
        }
    }
}

// Prime classes: 0: p < 2^30 (Mont32 combine; IMAD or FP64 runs)
//                1: 2^30 <= p < 2^44 (Mont64 combine; FP64 or IMAD runs)
//                2: p >= 2^44 (Mont64, IMAD runs only)

// ENGINE: 0 = IMAD runs, 1 = FP64 runs;  S = streams per lane (E = 2 / E = 3 sums)
// Persistent: each warp pulls items g in [g_lo, g_hi) from *counter (reset to 0 before launch).
// minimum resident blocks per SM (caps registers): FP64 / 64-bit engines 3 (<= 80 regs: +2-3 % on
// C4/C5 over 98 regs); the 32-bit IMAD engine is left unconstrained (a 64-register cap cost 8 % on C2)
template <class M, int CLASS, int ENGINE, int S2, int S3, bool PAIRS = false>
#ifndef WV_FPT_MINB
#define WV_FPT_MINB 2       // FP64 K-term kernels: resident blocks per SM targeted by register allocation
#endif
#ifndef WV_IT_MINB
#define WV_IT_MINB 2        // Mont64 K-term kernels: resident blocks per SM targeted by register allocation
#endif
__global__ void __launch_bounds__(RES_THREADS, (ENGINE == 0 && CLASS == 0) ? 1
                                              : ((ENGINE == 1 && PAIRS) ? WV_FPT_MINB
                                              : ((ENGINE == 0 && PAIRS && (S2 > 1 || S3 > 1)) ? WV_IT_MINB : 3)))
residue_kernel(const Rec *__restrict__ recs, const uint64_t *__restrict__ start, uint64_t klo, uint64_t khi,
               uint64_t g_lo, uint64_t g_hi, uint64_t part_base, ulonglong2 *__restrict__ partials,
               unsigned long long *__restrict__ counter, uint32_t class_mask,
               const uint32_t *__restrict__ segidx, uint32_t segstride) {
    using W = typename M::W;
    __shared__ WarpTab s_tab[RES_WARPS];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (;;) {
        unsigned long long gi = 0;
        if (lane == 0) gi = atomicAdd(counter, 1ull);
        gi = __shfl_sync(0xffffffffu, gi, 0);
        const uint64_t g = g_lo + gi;
        if (g >= g_hi) break;
        const uint64_t k = find_rec_warp(start, klo, khi, g);
        const Rec r = recs[k];
        if (!((class_mask >> prime_class(r.p)) & 1)) continue;   // another class's launch does it
        const uint64_t c = g - start[k];
        const Cong &cg = c_cong[r.cid];
        const uint32_t m = cg.m;
        M mo;
        mo.init(r.p);
        const uint64_t CT = 32ull * r.L;
        const Term *tb = c_terms + cg.off;       // this record's terms
        uint64_t t0, t1;
        if (cg.seg) {
            // sum-aligned chunk: locate (sum js, chunk cc) of local chunk c by a warp scan of
            // ceil(n_j / CT) over the sums, 32 sums per round, starting at the block of 32 sums
            // the plan kernel's coarse index places c in (entries nondecreasing: count them <= c)
            uint64_t carry = 0, sf = 0, sn = 0, cc = 0;
            uint32_t js = 0, base0 = 0;
            const uint32_t R = (m + 31) / 32;
            if (segidx && R <= segstride) {
                const uint32_t *ix = segidx + k * segstride;
                uint32_t cntle = 0;
                for (uint32_t rr = 0; rr < R; rr += 32) {
                    const bool le = rr + lane < R && (uint64_t)ix[rr + lane] <= c;
                    cntle += __popc(__ballot_sync(0xffffffffu, le));
                }
                base0 = (cntle - 1) * 32;                 // entry 0 is 0 <= c
                carry = ix[cntle - 1];
            }
            for (uint32_t base = base0; base < m; base += 32) {
                const uint32_t jj = base + lane;
                uint64_t f = 0, n = 0;
                if (jj < m) sum_bounds(r.p, tb[jj], &f, &n);
                const uint64_t ch = (n + CT - 1) / CT;
                const uint64_t inc = warp_incl_scan(ch);
                const uint32_t hit = __ballot_sync(0xffffffffu, carry + inc > c);
                if (hit) {
                    const int l0 = __ffs(hit) - 1;
                    const uint64_t inc0 = __shfl_sync(0xffffffffu, inc, l0), ch0 = __shfl_sync(0xffffffffu, ch, l0);
                    sf = __shfl_sync(0xffffffffu, f, l0);
                    sn = __shfl_sync(0xffffffffu, n, l0);
                    cc = c - (carry + inc0 - ch0);
                    js = base + l0;
                    break;
                }
                carry += __shfl_sync(0xffffffffu, inc, 31);
            }
            const uint64_t a0 = cc * CT, len = (sn - a0) < CT ? (sn - a0) : CT;
            const uint64_t per = (len + 31) >> 5;
            t0 = lane * per;
            t1 = t0 + per < len ? t0 + per : len;
            if (lane == 0) {                           // a one-sum table for lane_work
                s_tab[wid].first[0] = sf + a0;
                s_tab[wid].cum[0] = 0;
                s_tab[wid].cum[1] = len;
                s_tab[wid].coef[0] = (uint64_t)mo.mul((W)coef_mod(tb[js], r.p), mo.r2);
                s_tab[wid].cont = 0;                   // one run per stream: nothing to switch
            }
            __syncwarp();
        } else {
            for (uint32_t j = lane; j < m; j += 32) {
                uint64_t f, cnt;
                sum_bounds(r.p, tb[j], &f, &cnt);
                s_tab[wid].first[j] = f;
                s_tab[wid].cum[j + 1] = cnt;
                s_tab[wid].coef[j] = (uint64_t)mo.mul((W)coef_mod(tb[j], r.p), mo.r2);
            }
            __syncwarp();
            {                                          // warp-parallel prefix sums of the counts
                uint64_t carry = 0;
                for (uint32_t base = 0; base < m; base += 32) {
                    const uint32_t j = base + lane;
                    const uint64_t v = j < m ? s_tab[wid].cum[j + 1] : 0;
                    const uint64_t inc = warp_incl_scan(v) + carry;
                    if (j < m) s_tab[wid].cum[j + 1] = inc;
                    carry = __shfl_sync(0xffffffffu, inc, 31);
                }
                if (lane == 0) s_tab[wid].cum[0] = 0;
            }
            __syncwarp();
            const uint64_t base = c * CT;
            const uint64_t nck = (r.T - base) < CT ? (r.T - base) : CT;
            const uint64_t per = (nck + 31) >> 5;
            t0 = base + lane * per;
            t1 = t0 + per;
            const uint64_t tend = base + nck;
            if (t1 > tend) t1 = tend;
        }
        W C0 = mo.r1, C1 = 0;
        ModD md;
        WarpTab &tab = s_tab[wid];
        const bool prep = !cg.seg && m > 1;
        if (!prep && !cg.seg) {
            if (lane == 0) tab.cont = 0;
            __syncwarp();
        }
        bool tuples = false;
        if constexpr (ENGINE == 0 && PAIRS && (S2 > 1 || S3 > 1) && std::is_same<M, Mont64>::value) {
            if (cg.seg) {                                    // Mont64 K-term steps over the lane's run (class 2)
                const uint64_t x0 = tab.first[0] + t0, nl = t1 > t0 ? t1 - t0 : 0;
                if (cg.e == 3) int_tuple_work<3, (S3 > 1 ? S3 : 2)>(mo, r.p, x0, nl, tab.coef[0], C0, C1);
                else int_tuple_work<2, (S2 > 1 ? S2 : 2)>(mo, r.p, x0, nl, tab.coef[0], C0, C1);
                tuples = true;
            }
        }
        if (tuples) {
        } else if (ENGINE == 1 && PAIRS && cg.seg) {                // four-term FP64 steps over the lane's run
            md.init(r.p);
            const uint64_t x0 = tab.first[0] + t0, nl = t1 > t0 ? t1 - t0 : 0;
            // tuple widths: S2 / S3 reinterpreted as K for e = 2 / e = 3 (at least 2)
            if (cg.e == 3) fp_tuple_work<M, 3, (S3 > 1 ? S3 : 2)>(mo, md, r.p, x0, nl, (W)tab.coef[0], C0, C1);
            else fp_tuple_work<M, 2, (S2 > 1 ? S2 : 2)>(mo, md, r.p, x0, nl, (W)tab.coef[0], C0, C1);
        } else if (ENGINE == 1) {
            md.init(r.p);
            if (cg.e == 3) {
                if (prep) prepare_switch<M, RunD<M, 3>>(mo, md, tab, m);
                lane_work<M, RunD<M, 3>, 3, S3, false>(mo, md, tab, r.p, t0, t1, C0, C1);
            } else {
                if (prep) prepare_switch<M, RunD<M, 2>>(mo, md, tab, m);
                lane_work<M, RunD<M, 2>, 2, S2, false>(mo, md, tab, r.p, t0, t1, C0, C1);
            }
        } else {
            if (cg.e == 3) {
                if (prep) prepare_switch<M, Run<M, 3>>(mo, md, tab, m);
                lane_work<M, Run<M, 3>, 3, S3, PAIRS>(mo, md, tab, r.p, t0, t1, C0, C1);
            } else {
                if (prep) prepare_switch<M, Run<M, 2>>(mo, md, tab, m);
                lane_work<M, Run<M, 2>, 2, S2, PAIRS>(mo, md, tab, r.p, t0, t1, C0, C1);
            }
        }
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            W o0 = __shfl_xor_sync(0xffffffffu, C0, o);
            W o1 = __shfl_xor_sync(0xffffffffu, C1, o);
            combine(mo, C0, C1, o0, o1);
        }
        if (lane == 0) partials[g - part_base] = make_ulonglong2((unsigned long long)C0, (unsigned long long)C1);
        __syncwarp();
    }
}


// ---------------------------------------------------------------- lane mode
// Lane mode (sorted prime lists, class 0): a warp item is (group of 32 consecutive
// primes of one test, slice q of Q).  Lane l owns record (32g + l, test) and
// evaluates slice q of every sum of its congruence: for sum j with n_j terms the
// slice is [floor(q n_j / Q), floor((q+1) n_j / Q)).  Neighbouring primes share
// the congruence and have nearly equal n_j, so each sum is one warp-uniform loop:
// min-count unpredicated steps, then a short predicated tail up to the max count.
// One record per lane removes the per-boundary lockstep breaks of chunk mode.
template <class M, class R, int E>
__device__ __forceinline__ void lane_slice_work(const M &mo, const ModD &md, const Cong &cg, uint64_t p, bool valid,
                                                uint64_t q, uint64_t Q, typename M::W &C0, typename M::W &C1) {
    using W = typename M::W;
    const uint32_t m = valid ? cg.m : 0;
    const uint32_t mmax = __reduce_max_sync(0xffffffffu, m);
    uint32_t rb = R::kFP ? (E == 3 ? md.rb3 : md.rb2) : 0xffffffffu;
    if (R::kFP) rb = __reduce_min_sync(0xffffffffu, valid ? rb : 0xffffffffu);
    R run;
    for (uint32_t j = 0; j < mmax; j++) {
        uint32_t cnt = 0;
        uint64_t s0 = 1;
        if (j < m) {
            uint64_t f, n;
            sum_bounds(p, c_terms[cg.off + j], &f, &n);
            const uint64_t a = n * q / Q, b = n * (q + 1) / Q;
            cnt = (uint32_t)(b - a);
            s0 = f + a;
        }
        const uint32_t kmax = __reduce_max_sync(0xffffffffu, cnt);
        if (kmax == 0) continue;
        const uint32_t kmin = __reduce_min_sync(0xffffffffu, cnt ? cnt : 0xffffffffu);
        run.setup(mo, md, s0);
        uint32_t i = 0, since = 0;
        while (i < kmin) {
            const uint32_t kk0 = kmin - i;
            const uint32_t kk = kk0 < rb - since ? kk0 : rb - since;
            uint32_t x = 0;
            #pragma unroll 1
            for (; x + 4 <= kk; x += 4) {
                run.step(mo, md); run.step(mo, md); run.step(mo, md); run.step(mo, md);
            }
            for (; x < kk; x++) run.step(mo, md);
            i += kk;
            if (R::kFP) {
                since += kk;
                if (since == rb) { run.reduce(md); since = 0; }
            }
        }
        for (; i < kmax; i++) {
            run.step_masked(mo, md, i < cnt);
            if (R::kFP && ++since == rb) { run.reduce(md); since = 0; }
        }
        if (cnt) {
            W c0, c1;
            run.result(mo, md, c0, c1);
            c1 = mo.mul(c1, mo.mul((W)coef_mod(c_terms[cg.off + j], p), mo.r2));   // fold a_j
            combine(mo, C0, C1, c0, c1);
        }
    }
}

// items it in [item_lo, item_lo + nitems) processed largest-first (groups ascend in p);
// gstart = exclusive scan of gq over group-tests; start = per-record partial slots.
template <class M, int CLASS, int ENGINE>
__global__ void __launch_bounds__(RES_THREADS)
residue_lane_kernel(const Rec *__restrict__ recs, const uint64_t *__restrict__ start,
                    const uint64_t *__restrict__ gstart, const uint64_t *__restrict__ gq, uint64_t ngt,
                    uint64_t item_lo, uint64_t nitems_host, const uint64_t *__restrict__ nitems_dev, uint32_t ntests,
                    uint64_t K, uint64_t part_base, ulonglong2 *__restrict__ partials,
                    unsigned long long *__restrict__ counter,
                    unsigned long long *__restrict__ /*term_count: the plan counts this kernel's terms*/,
                    uint32_t /*allsl_mode: lane2 only*/, const unsigned long long *__restrict__ /*slice_counts*/) {
    const uint64_t nitems = nitems_dev ? *nitems_dev - item_lo : nitems_host;
    using W = typename M::W;
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned long long it = 0;
        if (lane == 0) it = atomicAdd(counter, 1ull);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= nitems) break;
        const uint64_t item = item_lo + nitems - 1 - it;
        const uint64_t gt = find_rec(gstart, 0, ngt, item);
        const uint64_t q = item - gstart[gt], Q = gq[gt];
        const uint64_t g = gt / ntests, t = gt % ntests;
        const uint64_t k = (32 * g + lane) * ntests + t;
        Rec r;
        r.p = 0;
        if (k < K) r = recs[k];
        const bool valid = r.p != 0 && prime_class(r.p) == CLASS;
        const Cong &cg = c_cong[valid ? r.cid : 0];
        M mo;
        mo.init(valid ? r.p : 7);
        W C0 = mo.r1, C1 = 0;
        ModD md;
        const uint32_t e = __reduce_max_sync(0xffffffffu, valid ? cg.e : 0);   // one test per item
        if (ENGINE == 1) {
            md.init(valid ? r.p : 7);
            if (e == 3) lane_slice_work<M, RunD<M, 3>, 3>(mo, md, cg, r.p, valid, q, Q, C0, C1);
            else lane_slice_work<M, RunD<M, 2>, 2>(mo, md, cg, r.p, valid, q, Q, C0, C1);
        } else {
            if (e == 3) lane_slice_work<M, Run<M, 3>, 3>(mo, md, cg, r.p, valid, q, Q, C0, C1);
            else lane_slice_work<M, Run<M, 2>, 2>(mo, md, cg, r.p, valid, q, Q, C0, C1);
        }
        if (valid) partials[start[k] + q - part_base] = make_ulonglong2((unsigned long long)C0, (unsigned long long)C1);
    }
}

// One thread per record in [klo, khi): merge the record's chunk pairs, invert, store.
template <class M>
__device__ __forceinline__ void finalize_one(const Rec &r, const uint64_t *start, uint64_t k, uint64_t part_base,
                                             const ulonglong2 *partials, uint64_t *res_w, uint64_t *res_v) {
    using W = typename M::W;
    M mo;
    mo.init(r.p);
    W C0 = mo.r1, C1 = 0;
    const uint64_t s = start[k], e = start[k + 1];
    for (uint64_t g = s; g < e; g++) {
        const ulonglong2 v = partials[g - part_base];
        combine(mo, C0, C1, (W)v.x, (W)v.y);
    }
    const Cong &cg = c_cong[r.cid];
    const W Lm = mo.mul((W)left_mod(cg, r.p), mo.r2);
    const W den = mo.mul(C0, Lm);
    const W X = mo.mul(C1, mont_inv(mo, den));
    const uint64_t x = mo.canon(X);
    if (r.test == 0) res_w[r.idx] = x; else res_v[r.idx] = x;
}

__global__ void finalize_kernel(const Rec *__restrict__ recs, const uint64_t *__restrict__ start,
                                uint64_t klo, uint64_t khi, uint64_t part_base,
                                const ulonglong2 *__restrict__ partials,
                                uint64_t *__restrict__ res_w, uint64_t *__restrict__ res_v) {
    for (uint64_t k = klo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < khi;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const Rec r = recs[k];
        if (r.p == 0) continue;                     // padding record (beyond n primes)
        if (r.p < WIDTH32_MAX) finalize_one<Mont32>(r, start, k, part_base, partials, res_w, res_v);
        else finalize_one<Mont64>(r, start, k, part_base, partials, res_w, res_v);
    }
}

// ---------------------------------------------------------------- checksum / hits
__host__ __device__ __forceinline__ uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {   // splitmix64 finaliser
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t checksum_term(uint64_t p, uint64_t rw, uint64_t rv) {
    return mix64(p ^ rotl64(rw, 21) ^ rotl64(rv, 42));
}

__global__ void flags_kernel(const uint64_t *__restrict__ primes, const uint64_t *__restrict__ n_dev,
                             uint64_t n_host, uint64_t kmax, uint64_t *__restrict__ res_w,
                             uint64_t *__restrict__ res_v, uint32_t mode, uint32_t *__restrict__ flags,
                             unsigned long long *__restrict__ checksum) {
    const uint64_t n = n_dev ? *n_dev : n_host;
    uint64_t acc = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < kmax;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t f = 0;
        if (i < n) {
            uint64_t rw = ~0ull, rv = ~0ull;
            if (mode & 1) rw = res_w[i]; else res_w[i] = ~0ull;
            if (mode & 2) rv = res_v[i]; else res_v[i] = ~0ull;
            f = (rw == 0 ? 1u : 0u) | (rv == 0 ? 2u : 0u);
            acc += checksum_term(primes[i], rw, rv);
        }
        if (flags) flags[i] = f ? 1u : 0u;
    }
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && checksum) atomicAdd(checksum, (unsigned long long)acc);
}

struct HitOut { uint64_t p; uint32_t flags; uint32_t reserved; };

// ---------------------------------------------------------------- near misses / histograms (NEXT-1)
struct NearOut { uint64_t p; int64_t symres; uint32_t test; uint32_t reserved; };

__device__ __forceinline__ void near_one(uint64_t p, uint64_t r, uint32_t test, uint64_t bound, NearOut *out,
                                         uint64_t cap, unsigned long long *count, unsigned long long *hist) {
    if (r == ~0ull) return;
    const bool neg = r > (p - 1) / 2;                    // <r> = r - p  if r > (p-1)/2
    const uint64_t mag = neg ? p - r : r;
    if (mag < bound) {
        const unsigned long long slot = atomicAdd(count, 1ull);
        if (slot < cap) out[slot] = NearOut{p, neg ? -(int64_t)mag : (int64_t)mag, test, 0};
    }
    if (hist) {
        // x = 2<r> + p in [1, 2p-1];  bin = floor(1000 x / p)  in [0, 1999]
        const uint64_t x = neg ? 2 * r - p : 2 * r + p;  // 2(r - p) + p = 2r - p for negative <r>
        const unsigned __int128 num = (unsigned __int128)x * 1000u;
        const uint32_t bin = (uint32_t)(num / p);
        atomicAdd(&hist[bin < 2000 ? bin : 1999], 1ull);
    }
}

__global__ void nearmiss_kernel(const uint64_t *__restrict__ primes, uint64_t n, const uint64_t *__restrict__ res_w,
                                const uint64_t *__restrict__ res_v, uint64_t bound, NearOut *__restrict__ out,
                                uint64_t cap, unsigned long long *__restrict__ count,
                                unsigned long long *__restrict__ hist_w, unsigned long long *__restrict__ hist_v) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t p = primes[i];
        near_one(p, res_w[i], 1, bound, out, cap, count, hist_w);
        near_one(p, res_v[i], 2, bound, out, cap, count, hist_v);
    }
}

__global__ void hits_scatter_kernel(const uint64_t *__restrict__ primes, const uint64_t *__restrict__ n_dev,
                                    uint64_t kmax, const uint64_t *__restrict__ res_w,
                                    const uint64_t *__restrict__ res_v, const uint32_t *__restrict__ flags,
                                    const uint64_t *__restrict__ pos, HitOut *__restrict__ hits) {
    const uint64_t n = *n_dev;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < kmax && i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (!flags[i]) continue;
        HitOut h;
        h.p = primes[i];
        h.flags = (res_w[i] == 0 ? 1u : 0u) | (res_v[i] == 0 ? 2u : 0u);
        h.reserved = 0;
        hits[pos[i]] = h;
    }
}

struct ResOut { uint64_t p, rw, rv; };
__global__ void pack_residues_kernel(const uint64_t *__restrict__ primes, uint64_t n,
                                     const uint64_t *__restrict__ res_w, const uint64_t *__restrict__ res_v,
                                     ResOut *__restrict__ out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = ResOut{primes[i], res_w[i], res_v[i]};
}

// first item of the first 64-bit record, and the batch boundaries
__global__ void split_kernel(const uint64_t *__restrict__ start, uint64_t K, const unsigned long long *first,
                             uint64_t *__restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        for (int c = 0; c < 2; c++) {              // class boundaries 2^30 and 2^44
            unsigned long long k = first[c];
            out[2 * c] = (k >= K) ? start[K] : start[k];   // start has K+1 entries (start[K] = total)
            out[2 * c + 1] = (k >= K) ? K : k;
        }
    }
}

// For batch b (1 <= b < nb): record index kb[b] = largest k with start[k] <= b * step (k in [0, K]);
// kb[nb + 1 + b] = start[kb[b]] (the batch's first item).
// Batch b of the partial-pair buffer: records [kb[b], kb[b + 1]), partial slots from kb[nb + 1 + b]
// (= start[kb[b]]).  Record boundaries are multiples of `align` (lane mode: whole groups of 32 primes x
// ntests, so a lane item never straddles two batches) or K; with gstart (lane mode) kb[2 (nb + 1) + b]
// is the first lane item of the batch (gstart at the boundary's group-test).
__global__ void batch_bounds_kernel(const uint64_t *__restrict__ start, uint64_t K, uint64_t step, uint64_t nb,
                                    uint64_t *__restrict__ kb, uint64_t align, const uint64_t *__restrict__ gstart,
                                    uint32_t ntests) {
    const uint64_t ng = (K + align - 1) / align;                  // aligned boundaries g * align, g <= ng
    for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t g;
        if (b == 0) {
            g = 0;
        } else if (b == nb) {
            g = ng;
        } else {
            const uint64_t target = b * step;
            uint64_t lo = 0, hi = ng + 1;                          // largest g with start[min(g align, K)] <= target
            while (hi - lo > 1) {
                const uint64_t mid = (lo + hi) >> 1;
                const uint64_t k = mid * align < K ? mid * align : K;
                if (start[k] <= target) lo = mid; else hi = mid;
            }
            g = lo;
        }
        const uint64_t k = g * align < K ? g * align : K;
        kb[b] = k;
        kb[nb + 1 + b] = start[k];
        if (gstart) kb[2 * (nb + 1) + b] = gstart[g * ntests];
    }
}

}  // namespace wv
