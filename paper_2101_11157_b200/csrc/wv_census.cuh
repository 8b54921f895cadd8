// wv_census.cuh -- SURVEY.md 8(f) NEXT-3: general-index residues B_{2k}, E_{2k} mod p for every
// even index 2 <= 2k <= p-3 of every prime p in a window (the irregular / E-irregular pair census
// of P:L88-103), on sm_100a.
//
// The paper's congruences hold for every k with p-1 not dividing 2k:
//   B:  C_k(3,4,6) B_{2k} == S_{2k-1}(1/6, 1/4)                      eqnSV
//   E:  (-1)^k 4^{2k-1} E_{p-1-2k} == S_{p-1-2k}(0, 1/4)             eqnE1   (reading R10)
// with S_l(x, y) = sum_{xp<s<yp} s^l mod p and C_k(a,b,c) = (a^{p-2k} + b^{p-2k} - c^{p-2k} - 1)/(4k).
// Finite differences do not apply to s^l for large l, so all exponents of one prime are walked
// together over the multiplicative group: with g a primitive root and s_j = g^j,
//     S_l(I) = sum_{0<=j<(p-1)/2} [s'_j in I] sigma_j (g^l)^j,   s'_j = min(s_j, p - s_j),
// sigma_j = 1 if s'_j = s_j else (-1)^l (s_{j+(p-1)/2} = -s_j, so each pair {s, p-s} is visited
// once).  One lane owns one exponent l; the membership codes of s'_j are shared by the warp, and
// the sum over j is a polynomial in h = g^l with coefficients in {0, +1, -1}, evaluated by Horner
// over blocks of 16 steps with table lookups inside a block (see census_walk_kernel).  Every index
// of a prime costs (p-1)/2 steps.
//
// Where C_k(3,4,6) == 0 (mod p) the finalize kernel queues (p, l) for a fix-up that evaluates the
// first congruence of a fixed list with a unit C_k directly (per-term powers; rare: ~1/p of the B
// indices): VOR (2,3,4) P:L245-249, (4,5,8) P:L263-268, eqnVandiver (2,5,6) P:L171-175, eqnTW1
// with b = 2, 4, 6, 7, then b = 8, 9, ....
#pragma once
#include <stdint.h>
#include "wv_mont.cuh"
#include "wv_residue.cuh"

namespace wv {

constexpr uint32_t CEN_SEG = 4096;             // walk steps per work item
constexpr uint32_t CEN_TG = 8;                 // exponent tiles (of 32) per work item
constexpr uint32_t CEN_TW_BMAX = 1024;         // fix-up: eqnTW1 parameters b <= this
constexpr uint32_t CEN_THREADS = 128;
constexpr uint32_t CEN_WARPS = CEN_THREADS / 32;
constexpr uint64_t CEN_HI_MAX = 1ull << 26;    // lazy bounds of the Horner walk

// Montgomery power: b in Montgomery form, result in Montgomery form ([0, 2p))
__device__ __forceinline__ uint32_t cen_pow(const Mont32 &mo, uint32_t b, uint64_t e) {
    uint32_t r = mo.r1;
    while (e) {
        if (e & 1) r = mo.mul(r, b);
        b = mo.mul(b, b);
        e >>= 1;
    }
    return r;
}

// number of exponents per prime for the mode: 3 -> l = 1..p-3; 1 -> odd l (B); 2 -> even l (E)
__host__ __device__ __forceinline__ uint64_t cen_nexp(uint64_t p, uint32_t mode) {
    return mode == 3 ? p - 3 : (p - 3) / 2;
}
// exponent of enumeration position q (0-based)
__device__ __forceinline__ uint64_t cen_exp(uint64_t q, uint32_t mode) {
    return mode == 3 ? q + 1 : (mode == 1 ? 2 * q + 1 : 2 * q + 2);
}

// one thread per prime: primitive root (smallest g with g^{(p-1)/q} != 1 for all primes q | p-1),
// number of exponents and of work items (groups of CEN_TG exponent tiles of 32 x walk segments
// of CEN_SEG steps)
__global__ void census_plan_kernel(const uint64_t *__restrict__ primes, uint64_t n, uint32_t mode,
                                   uint32_t *__restrict__ groot, uint64_t *__restrict__ nexp,
                                   uint64_t *__restrict__ nitems) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = (uint32_t)primes[i];
        uint32_t q[10], nq = 0, m = p - 1;
        for (uint32_t d = 2; d * d <= m; d += (d == 2 ? 1 : 2)) {
            if (m % d == 0) {
                q[nq++] = d;
                while (m % d == 0) m /= d;
            }
        }
        if (m > 1) q[nq++] = m;
        Mont32 mo;
        mo.init(p);
        uint32_t g = 2;
        for (;; g++) {
            const uint32_t gm = mo.to(g);
            bool ok = true;
            for (uint32_t t = 0; t < nq && ok; t++) ok = mo.canon(cen_pow(mo, gm, (p - 1) / q[t])) != 1;
            if (ok) break;
        }
        groot[i] = g;
        const uint64_t ne = cen_nexp(p, mode);
        const uint64_t half = (p - 1) / 2, tiles = (mode == 3 ? 2 : 1) * (((p - 3) / 2 + 31) / 32);
        nexp[i] = ne;
        nitems[i] = ((tiles + CEN_TG - 1) / CEN_TG) * ((half + CEN_SEG - 1) / CEN_SEG);
    }
}

// Persistent walk.  Items: (prime i, group of CEN_TG exponent tiles, walk segment of CEN_SEG
// steps).  A tile is 32 exponents of one parity (B: odd l, E: even l), one per lane, so the
// membership codes are warp-uniform.  Per segment the warp writes three bit masks (B with
// sigma = +1, B with sigma = -1, E) of its steps j; per tile each lane evaluates
//     sum_j c_j h^j  (h = g^l, c_j in {0, +1, -1})
// by Horner over blocks of 16 steps from the last block down:  acc <- acc h^16 + inner_J, with
// inner_J = sum_{d<16} c_{16J+d} h^d read from per-lane subset-sum tables of {h^{4n+b}: b < 4}
// (4 nibbles x 16 entries, shared memory, uniform index) -- 4 (E) or 8 (B) table reads and one
// Montgomery step per 16 walk steps.  Lazy bounds (p < 2^26): table entries < 4p, inner < 32p,
// acc < 40p, REDC(acc H + inner R) < 40p.
constexpr uint32_t CEN_WORDS = CEN_SEG / 32;

__device__ __forceinline__ uint32_t cen_lds(uint32_t addr) {     // 32-bit shared load, shared address
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint32_t cen_horner(const Mont32 &mo, uint32_t acc, uint32_t H, uint32_t in) {
    // REDC(acc H + in 2^32): T = acc H + (in << 32); m = T_lo pinv; (T + m p) >> 32 -- three IMADs
    uint32_t r;
    asm("{\n\t.reg .u64 t, z;\n\t.reg .u32 lo, m, hi;\n\t"
        "mov.b64 z, {0, %4};\n\t"
        "mad.wide.u32 t, %1, %2, z;\n\t"
        "cvt.u32.u64 lo, t;\n\t"
        "mul.lo.u32 m, lo, %3;\n\t"
        "mad.wide.u32 t, m, %5, t;\n\t"
        "mov.b64 {lo, hi}, t;\n\t"
        "mov.u32 %0, hi;\n\t}"
        : "=r"(r) : "r"(acc), "r"(H), "r"(mo.pinv), "r"(in), "r"(mo.p));
    return r;
}

__global__ void __launch_bounds__(CEN_THREADS)
census_walk_kernel(const uint64_t *__restrict__ primes, const uint32_t *__restrict__ groot,
                   const uint64_t *__restrict__ istart, const uint64_t *__restrict__ ebase, uint64_t i_lo,
                   uint64_t i_hi, uint32_t mode, unsigned long long *__restrict__ acc_out,
                   unsigned long long *__restrict__ counter) {
    __shared__ uint32_t s_bp[CEN_WARPS][CEN_WORDS], s_bn[CEN_WARPS][CEN_WORDS], s_e[CEN_WARPS][CEN_WORDS];
    // per-warp tables [4][16][32] (8 KB), placed at an 8 KB-aligned shared address at run time so a
    // table address is  base | (nibble << 7) | (n << 11)  -- one LOP3, no add (the static
    // attribute alone does not fix the absolute shared address)
    __shared__ uint32_t s_tabraw[CEN_WARPS * 2048 + 2048];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t g_lo = istart[i_lo], g_hi = istart[i_hi];
    const uint32_t raw = (uint32_t)__cvta_generic_to_shared(s_tabraw);
    const uint32_t al = (raw + 8191u) & ~8191u;
    uint32_t *tabw = s_tabraw + (al - raw) / 4 + wid * 2048;          // [n][x][lane] = tabw[(16 n + x) 32 + lane]
    const uint32_t tb = al + wid * 8192u + lane * 4u;
    const uint32_t t0 = tb, t1 = tb | 0x800u, t2 = tb | 0x1000u, t3 = tb | 0x1800u;
    for (;;) {
        unsigned long long gi = 0;
        if (lane == 0) gi = atomicAdd(counter, 1ull);
        gi = __shfl_sync(0xffffffffu, gi, 0);
        const uint64_t g = g_lo + gi;
        if (g >= g_hi) break;
        const uint64_t i = find_rec_warp(istart, i_lo, i_hi, g);
        const uint32_t p = (uint32_t)primes[i];
        const uint64_t c = g - istart[i];
        const uint32_t half = (p - 1) / 2;
        const uint32_t nseg = (half + CEN_SEG - 1) / CEN_SEG;
        const uint64_t grp = c / nseg;
        const uint32_t seg = (uint32_t)(c % nseg);
        const uint32_t j0 = seg * CEN_SEG;
        const uint32_t len = half - j0 < CEN_SEG ? half - j0 : CEN_SEG;
        Mont32 mo;
        mo.init(p);
        const uint32_t gm = mo.to(groot[i]);
        // codes of s_j = g^{j0 + j}, j < len (s kept plain: mul(s, g R) = s g mod p)
        const uint32_t nwords = (len + 31) / 32;
        {
            const uint32_t g1024 = cen_pow(mo, gm, 1024);
            uint32_t s0 = (uint32_t)mo.canon(cen_pow(mo, gm, (uint64_t)j0 + 32 * lane));
            for (uint32_t wd = lane; wd < nwords; wd += 32) {
                uint32_t s = s0, bp = 0, bn = 0, be = 0;
                #pragma unroll 8
                for (uint32_t b = 0; b < 32; b++) {
                    if (32 * wd + b < len) {
                        const uint32_t sp = s <= p - s ? s : p - s;
                        const bool q4 = 4ull * sp < p, inb = q4 && 6ull * sp > p;
                        bp |= (uint32_t)(inb && sp == s) << b;
                        bn |= (uint32_t)(inb && sp != s) << b;
                        be |= (uint32_t)q4 << b;
                    }
                    s = mo.mul(s, gm);
                    s = s >= p ? s - p : s;
                }
                s_bp[wid][wd] = bp;
                s_bn[wid][wd] = bn;
                s_e[wid][wd] = be;
                s0 = mo.mul(s0, g1024);
                s0 = s0 >= p ? s0 - p : s0;
            }
        }
        __syncwarp();
        const uint64_t nhalf = (p - 3) / 2;                 // exponents per parity
        const uint64_t tB = mode == 2 ? 0 : (nhalf + 31) / 32, tE = mode == 1 ? 0 : (nhalf + 31) / 32;
        const uint32_t nblk = (len + 15) / 16;
        for (uint32_t tt = 0; tt < CEN_TG; tt++) {
            const uint64_t t = grp * CEN_TG + tt;
            if (t >= tB + tE) break;                         // warp-uniform
            const bool isB = t < tB;
            const uint64_t u = (isB ? t : t - tB) * 32 + lane;
            const bool valid = u < nhalf;
            const uint64_t l = isB ? 2 * u + 1 : 2 * u + 2;
            const uint64_t q = mode == 3 ? l - 1 : u;
            const uint32_t h = cen_pow(mo, gm, valid ? l : 1);
            // h^d, d < 16 (canonical Montgomery form), subset-sum tables, H = h^16
            uint32_t hp[16];
            hp[0] = mo.r1;
            #pragma unroll
            for (int d = 1; d < 16; d++) {
                const uint32_t x = mo.mul(hp[d - 1], h);
                hp[d] = x >= p ? x - p : x;
            }
            uint32_t H = mo.mul(hp[15], h);
            H = H >= p ? H - p : H;
            __syncwarp();
            #pragma unroll
            for (int n = 0; n < 4; n++) {
                uint32_t v[16];
                v[0] = 0;
                #pragma unroll
                for (int x = 1; x < 16; x++) v[x] = v[x & (x - 1)] + hp[4 * n + ((x & 1) ? 0 : (x & 2) ? 1 : (x & 4) ? 2 : 3)];
                #pragma unroll
                for (int x = 0; x < 16; x++) tabw[(16 * n + x) * 32 + lane] = v[x];
            }
            __syncwarp();
            uint32_t acc = 0;
            const uint32_t p16 = 16 * p;
            // blocks J = nblk-1 .. 0, two per code word (block 2w: low half, 2w+1: high half)
            if (isB) {
                int J = (int)nblk - 1;
                if (!(J & 1)) {                                  // odd count: the lone top block first
                    const uint32_t bp = s_bp[wid][J >> 1], bn = s_bn[wid][J >> 1];
                    acc = cen_horner(mo, acc, H, cen_lds(t0 | ((bp << 7) & 0x780u)) + cen_lds(t1 | ((bp << 3) & 0x780u)) +
                                                 cen_lds(t2 | ((bp >> 1) & 0x780u)) + cen_lds(t3 | ((bp >> 5) & 0x780u)) +
                                                 p16 - (cen_lds(t0 | ((bn << 7) & 0x780u)) + cen_lds(t1 | ((bn << 3) & 0x780u)) +
                                                        cen_lds(t2 | ((bn >> 1) & 0x780u)) + cen_lds(t3 | ((bn >> 5) & 0x780u))));
                    J--;
                }
                for (; J > 0; J -= 2) {
                    const uint32_t wp = s_bp[wid][J >> 1], wn = s_bn[wid][J >> 1];
                    {
                        const uint32_t bp = wp >> 16, bn = wn >> 16;
                        acc = cen_horner(mo, acc, H, cen_lds(t0 | ((bp << 7) & 0x780u)) + cen_lds(t1 | ((bp << 3) & 0x780u)) +
                                                     cen_lds(t2 | ((bp >> 1) & 0x780u)) + cen_lds(t3 | ((bp >> 5) & 0x780u)) +
                                                     p16 - (cen_lds(t0 | ((bn << 7) & 0x780u)) + cen_lds(t1 | ((bn << 3) & 0x780u)) +
                                                            cen_lds(t2 | ((bn >> 1) & 0x780u)) + cen_lds(t3 | ((bn >> 5) & 0x780u))));
                    }
                    {
                        const uint32_t bp = wp, bn = wn;
                        acc = cen_horner(mo, acc, H, cen_lds(t0 | ((bp << 7) & 0x780u)) + cen_lds(t1 | ((bp << 3) & 0x780u)) +
                                                     cen_lds(t2 | ((bp >> 1) & 0x780u)) + cen_lds(t3 | ((bp >> 5) & 0x780u)) +
                                                     p16 - (cen_lds(t0 | ((bn << 7) & 0x780u)) + cen_lds(t1 | ((bn << 3) & 0x780u)) +
                                                            cen_lds(t2 | ((bn >> 1) & 0x780u)) + cen_lds(t3 | ((bn >> 5) & 0x780u))));
                    }
                }
            } else {
                int J = (int)nblk - 1;
                if (!(J & 1)) {
                    const uint32_t be = s_e[wid][J >> 1];
                    acc = cen_horner(mo, acc, H, cen_lds(t0 | ((be << 7) & 0x780u)) + cen_lds(t1 | ((be << 3) & 0x780u)) +
                                                 cen_lds(t2 | ((be >> 1) & 0x780u)) + cen_lds(t3 | ((be >> 5) & 0x780u)));
                    J--;
                }
                for (; J > 0; J -= 2) {
                    const uint32_t we = s_e[wid][J >> 1];
                    const uint32_t bh = we >> 16;
                    acc = cen_horner(mo, acc, H, cen_lds(t0 | ((bh << 7) & 0x780u)) + cen_lds(t1 | ((bh << 3) & 0x780u)) +
                                                 cen_lds(t2 | ((bh >> 1) & 0x780u)) + cen_lds(t3 | ((bh >> 5) & 0x780u)));
                    acc = cen_horner(mo, acc, H, cen_lds(t0 | ((we << 7) & 0x780u)) + cen_lds(t1 | ((we << 3) & 0x780u)) +
                                                 cen_lds(t2 | ((we >> 1) & 0x780u)) + cen_lds(t3 | ((we >> 5) & 0x780u)));
                }
            }
            if (valid) {
                // times h^{j0} (segment offset), canonical
                const uint32_t w0 = cen_pow(mo, h, j0);
                const uint32_t r = (uint32_t)(((uint64_t)mo.mul(acc, w0)) % p);
                atomicAdd(acc_out + (ebase[i] - ebase[i_lo]) + q, (unsigned long long)r);
            }
        }
        __syncwarp();
    }
}

struct CenPair { uint64_t p; uint32_t index; uint32_t kind; };   // = wv_pair
struct CenFix { uint64_t i; uint64_t e; };                         // prime index, batch entry

__host__ __device__ __forceinline__ uint64_t cen_checksum_term(uint64_t p, uint32_t index, uint32_t kind,
                                                               uint64_t res) {
    return mix64(p ^ ((uint64_t)index << 32) ^ rotl64(res, 17) ^ ((uint64_t)kind << 62));
}

// outputs of one index residue: residue array, zero -> pair list; the checksum term is added to
// the caller's register sum (flushed once per warp by cen_flush: one global atomic per warp)
__device__ __forceinline__ void cen_emit(uint64_t p, uint32_t index, uint32_t kind, uint64_t res, uint64_t e,
                                         uint64_t *__restrict__ res_out, CenPair *__restrict__ pairs,
                                         uint64_t pair_cap, unsigned long long *__restrict__ misc, uint64_t &chk) {
    if (res_out) res_out[e] = res;
    if (res == 0) {
        const unsigned long long k = atomicAdd(misc + 0, 1ull);
        if (k < pair_cap) pairs[k] = CenPair{p, index, kind};
    }
    chk += cen_checksum_term(p, index, kind, res);
}
__device__ __forceinline__ void cen_flush(uint64_t chk, unsigned long long *__restrict__ misc) {
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) chk += __shfl_xor_sync(0xffffffffu, chk, o);
    if ((threadIdx.x & 31) == 0 && chk) atomicAdd(misc + 1, (unsigned long long)chk);
}

// C_k(3,4,6) numerator 3^t + 4^t - 6^t - 1 (t = p - 2k), canonical
__device__ __forceinline__ uint32_t cen_cnum(const Mont32 &mo, uint32_t a, uint32_t b, uint32_t c, uint64_t t) {
    const uint32_t pa = cen_pow(mo, mo.to(a), t), pb = cen_pow(mo, mo.to(b), t), pc = cen_pow(mo, mo.to(c), t);
    uint32_t x = mo.add(pa, pb);
    x = mo.add(x, mo.p2 - (pc >= mo.p2 ? pc - mo.p2 : pc));
    x = mo.add(x, mo.p2 - mo.r1);
    return (uint32_t)mo.canon(x);
}

// One block per prime (grid-stride over the batch's primes), thread tid takes positions
// q = tid, tid + CEN_FIN_T, ... of that prime, so its exponents l advance by a fixed step dl:
//   odd l = 2k-1:  B_{2k} = S (4k) / N,  N = 3^t + 4^t - 6^t - 1,  t = p - 2k     (eqnSV)
//   even l:        E_l = (-1)^k 4^{p-2k} S,  2k = p - 1 - l                       (eqnE1, R10)
// The powers 3^t, 4^t, 6^t (t falls by dl) and 4^{p-2k} (rises by dl) are advanced by one product
// each; the B inverses are batched 8 at a time per thread (one Fermat inverse per batch).
constexpr uint32_t CEN_FIN_T = 256;
constexpr int CEN_FIN_BATCH = 8;

__global__ void __launch_bounds__(CEN_FIN_T)
census_finalize_kernel(const uint64_t *__restrict__ primes, const uint64_t *__restrict__ ebase,
                       uint64_t i_lo, uint64_t i_hi, uint32_t mode, const unsigned long long *__restrict__ acc,
                       uint64_t *__restrict__ res_out, CenPair *__restrict__ pairs, uint64_t pair_cap,
                       CenFix *__restrict__ fix, uint64_t fix_cap, unsigned long long *__restrict__ misc) {
    const uint32_t tid = threadIdx.x;
    uint64_t chk = 0;
    for (uint64_t i = i_lo + blockIdx.x; i < i_hi; i += gridDim.x) {
        const uint32_t p = (uint32_t)primes[i];
        const uint64_t base = ebase[i] - ebase[i_lo], ne = ebase[i + 1] - ebase[i];
        if (tid >= ne) continue;
        Mont32 mo;
        mo.init(p);
        const uint64_t l0 = cen_exp(tid, mode);
        const uint64_t dl = (mode == 3 ? 1 : 2) * (uint64_t)CEN_FIN_T;      // exponent step per iteration
        const uint64_t dlm = dl % (p - 1);
        if (l0 & 1) {                                    // B entries (odd l)
            const uint64_t t0 = p - (l0 + 1);           // t = p - 2k, falls by dl
            const uint64_t back = (p - 1) - dlm;         // x^{-dl} = x^{(p-1) - dl mod (p-1)}
            const uint32_t m3 = mo.to(3), m4 = mo.to(4), m6 = mo.to(6);
            uint32_t p3 = cen_pow(mo, m3, t0), p4 = cen_pow(mo, m4, t0), p6 = cen_pow(mo, m6, t0);
            const uint32_t s3 = cen_pow(mo, m3, back), s4 = cen_pow(mo, m4, back), s6 = cen_pow(mo, m6, back);
            uint32_t pend_x[CEN_FIN_BATCH], pend_n[CEN_FIN_BATCH];  // S (4k) and N (Montgomery form)
            uint64_t pend_q[CEN_FIN_BATCH];
            int np = 0;
            for (uint64_t q = tid; q < ne; q += CEN_FIN_T) {
                const uint64_t l = cen_exp(q, mode), k2 = l + 1;
                uint32_t N = mo.add(p3, p4);
                N = mo.add(N, mo.p2 - p6);
                N = mo.add(N, mo.p2 - mo.r1);
                p3 = mo.mul(p3, s3); p4 = mo.mul(p4, s4); p6 = mo.mul(p6, s6);
                const uint32_t Sm = (uint32_t)(acc[base + q] % p);
                if (mo.canon(N) == 0) {                  // C_k(3,4,6) == 0: another congruence
                    const unsigned long long f = atomicAdd(misc + 2, 1ull);
                    if (f < fix_cap) fix[f] = CenFix{i, base + q};
                    continue;
                }
                pend_x[np] = mo.mul(Sm, mo.to(2 * k2));
                pend_n[np] = N;
                pend_q[np] = q;
                np++;
                const bool last = q + CEN_FIN_T >= ne;
                if (np == CEN_FIN_BATCH || last) {
                    // Montgomery's trick: one inverse for the batch
                    uint32_t pre[CEN_FIN_BATCH];
                    uint32_t run = mo.r1;
                    #pragma unroll
                    for (int u = 0; u < CEN_FIN_BATCH; u++) {
                        if (u < np) { pre[u] = run; run = mo.mul(run, pend_n[u]); }
                    }
                    uint32_t inv = cen_pow(mo, run, p - 2);
                    #pragma unroll
                    for (int u = CEN_FIN_BATCH - 1; u >= 0; u--) {
                        if (u < np) {
                            const uint32_t iu = mo.mul(inv, pre[u]);         // 1 / N_u
                            inv = mo.mul(inv, pend_n[u]);
                            const uint64_t lq = cen_exp(pend_q[u], mode);
                            cen_emit(p, (uint32_t)(lq + 1), 1, mo.canon(mo.mul(pend_x[u], iu)), base + pend_q[u],
                                     res_out, pairs, pair_cap, misc, chk);
                        }
                    }
                    np = 0;
                }
            }
            if (np) {                                    // (only when the last entries were fix-ups)
                uint32_t pre[CEN_FIN_BATCH];
                uint32_t run = mo.r1;
                #pragma unroll
                for (int u = 0; u < CEN_FIN_BATCH; u++) {
                    if (u < np) { pre[u] = run; run = mo.mul(run, pend_n[u]); }
                }
                uint32_t inv = cen_pow(mo, run, p - 2);
                #pragma unroll
                for (int u = CEN_FIN_BATCH - 1; u >= 0; u--) {
                    if (u < np) {
                        const uint32_t iu = mo.mul(inv, pre[u]);
                        inv = mo.mul(inv, pend_n[u]);
                        const uint64_t lq = cen_exp(pend_q[u], mode);
                        cen_emit(p, (uint32_t)(lq + 1), 1, mo.canon(mo.mul(pend_x[u], iu)), base + pend_q[u],
                                 res_out, pairs, pair_cap, misc, chk);
                    }
                }
            }
        } else {                                         // E entries (even l): 4^{p-2k} = 4^{l+1}
            const uint32_t m4 = mo.to(4);
            uint32_t f = cen_pow(mo, m4, l0 + 1);
            const uint32_t sf = cen_pow(mo, m4, dlm);
            for (uint64_t q = tid; q < ne; q += CEN_FIN_T) {
                const uint64_t l = cen_exp(q, mode), k = (p - 1 - l) / 2;
                const uint32_t Sm = (uint32_t)(acc[base + q] % p);
                uint64_t v = mo.canon(mo.mul(Sm, f));
                f = mo.mul(f, sf);
                if ((k & 1) && v) v = p - v;
                cen_emit(p, (uint32_t)l, 2, v, base + q, res_out, pairs, pair_cap, misc, chk);
            }
        }
    }
    cen_flush(chk, misc);
}

// fallback congruences for B_{2k} where C_k(3,4,6) == 0 (mod p): C_k(a,b,c) B_{2k} == sum of
// S_{2k-1} over the intervals (VOR P:L245-249; (4,5,8) P:L263-268; eqnVandiver P:L171-175;
// eqnTW1 b = 2, 4, 6, 7 P:L185-189)
struct CenAlt { uint32_t a, b, c, min_p, n; uint32_t iv[3][4]; };
__constant__ CenAlt c_cen_alt[7] = {
    {2, 3, 4, 5, 1, {{1, 4, 1, 3}}},
    {4, 5, 8, 7, 2, {{1, 8, 1, 5}, {3, 8, 2, 5}}},
    {2, 5, 6, 7, 2, {{1, 6, 1, 5}, {1, 3, 2, 5}}},
    {2, 2, 3, 5, 1, {{1, 3, 1, 2}}},
    {2, 4, 5, 7, 2, {{1, 5, 1, 4}, {2, 5, 1, 2}}},
    {2, 6, 7, 11, 3, {{1, 7, 1, 6}, {2, 7, 1, 3}, {3, 7, 1, 2}}},
    {2, 7, 8, 11, 3, {{1, 8, 1, 7}, {2, 8, 2, 7}, {3, 8, 3, 7}}},
};

// one warp per queued entry: the first fallback with a unit C_k, its sums by per-term powers
__global__ void census_fixup_kernel(const uint64_t *__restrict__ primes, const uint64_t *__restrict__ ebase,
                                    uint64_t i_lo, uint32_t mode, const CenFix *__restrict__ fix, uint64_t nfix,
                                    uint64_t *__restrict__ res_out, CenPair *__restrict__ pairs, uint64_t pair_cap,
                                    unsigned long long *__restrict__ misc) {
    const int lane = threadIdx.x & 31;
    uint64_t chk = 0;
    const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t f = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; f < nfix; f += nwarps) {
        const CenFix fx = fix[f];
        const uint32_t p = (uint32_t)primes[fx.i];
        const uint64_t q = fx.e - (ebase[fx.i] - ebase[i_lo]);
        const uint64_t l = cen_exp(q, mode), k2 = l + 1;
        Mont32 mo;
        mo.init(p);
        bool done = false;
        // the table, then eqnTW1 for b = 8, 9, ... (p > b + 1): C_k(2,b,b+1) B_{2k} ==
        // sum_{m=1}^{floor(b/2)} S_{2k-1}(m/(b+1), m/b).  All small-base numerators vanish together
        // where a^{t-1} is a character of small order (e.g. t = (p+1)/2 with 2, 3, 5, 7 quadratic
        // residues); a base b + 1 outside its kernel ends that (b <= 28 for every p < 30000).
        for (uint32_t a = 0; a < 7 + CEN_TW_BMAX && !done; a++) {
            uint32_t ca, cb, cc, n;
            if (a < 7) {
                const CenAlt &A = c_cen_alt[a];
                if (p < A.min_p) continue;
                ca = A.a; cb = A.b; cc = A.c; n = A.n;
            } else {
                const uint32_t b = a + 1;
                if (p <= b + 1) break;
                ca = 2; cb = b; cc = b + 1; n = b / 2;
            }
            const uint32_t N = cen_cnum(mo, ca, cb, cc, p - k2);
            if (N == 0) continue;
            uint32_t S = 0;
            for (uint32_t t = 0; t < n; t++) {
                uint32_t xn, xd, yn, yd;
                if (a < 7) {
                    xn = c_cen_alt[a].iv[t][0]; xd = c_cen_alt[a].iv[t][1];
                    yn = c_cen_alt[a].iv[t][2]; yd = c_cen_alt[a].iv[t][3];
                } else {
                    xn = t + 1; xd = cc; yn = t + 1; yd = cb;        // (m/(b+1), m/b)
                }
                const uint64_t s_lo = (uint64_t)xn * p / xd + 1;                      // x p < s
                const uint64_t yp = (uint64_t)yn * p;                                  // s < y p
                const uint64_t s_hi = yp % yd ? yp / yd : yp / yd - 1;
                for (uint64_t s = s_lo + lane; s <= s_hi; s += 32) S = mo.add(S, cen_pow(mo, mo.to(s), l));
            }
            #pragma unroll
            for (int o = 16; o > 0; o >>= 1) S = mo.add(S, __shfl_xor_sync(0xffffffffu, S, o));
            uint32_t r = mo.mul(S, mo.to(2 * k2));
            r = mo.mul(r, cen_pow(mo, mo.to(N), p - 2));
            if (lane == 0) cen_emit(p, (uint32_t)k2, 1, mo.canon(r), fx.e, res_out, pairs, pair_cap, misc, chk);
            done = true;
        }
        if (!done && lane == 0) atomicAdd(misc + 3, 1ull);   // unresolved (reported as an error)
    }
    cen_flush(chk, misc);
}

}  // namespace wv
