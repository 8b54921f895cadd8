// wv_mont.cuh -- Montgomery arithmetic mod p for the residue kernels (sm_100a).
//
// The paper multiplies mod p with native 64-bit products for p < 2^32 and a
// split 32-bit product + '%' beyond (eqnMultiply).  Here every
// product is a Montgomery product (BASELINE.json north_star): no division in
// the hot loop, only IMAD / IMAD.WIDE / IMAD.HI.
//
// Both widths keep values "lazy" in [0, 2p):
//   Mont32: R = 2^32, p < 2^30  (4p^2 + 3pR < 2^64 for the fused multiply-add)
//   Mont64: R = 2^64, p < 2^62  (4p < R)
// REDC(T) = (T + m p)/R with m = T * (-p^{-1}) mod R;  for a, b < 2p,
// REDC(a b) < (4p^2 + pR)/R < 2p.
#pragma once
#include <stdint.h>

namespace wv {

struct Mont32 {
    using W = uint32_t;
    uint32_t p, pinv, p2, r1, r2;   // pinv = -p^{-1} mod 2^32; r1 = R mod p; r2 = R^2 mod p

    __device__ __forceinline__ void init(uint64_t p64) {
        p = (uint32_t)p64;
        p2 = 2u * p;
        uint32_t inv = p;                       // p*p == 1 (mod 8): 3 correct bits
        #pragma unroll
        for (int i = 0; i < 4; i++) inv *= 2u - p * inv;   // Newton: 3 -> 48 bits
        pinv = 0u - inv;
        r1 = (uint32_t)(0x100000000ull % p);
        r2 = (uint32_t)(((uint64_t)r1 * r1) % p);
    }
    // a, b < 2p  ->  a b R^{-1} mod p, in [0, 2p)
    __device__ __forceinline__ uint32_t mul(uint32_t a, uint32_t b) const {
        uint64_t T = (uint64_t)a * b;
        uint32_t m = (uint32_t)T * pinv;
        return (uint32_t)((T + (uint64_t)m * p) >> 32);
    }
    // a b R^{-1} + c mod p, in [0, 2p):  REDC(a b + c R), then one lazy subtract.
    __device__ __forceinline__ uint32_t muladd(uint32_t a, uint32_t b, uint32_t c) const {
        uint64_t T = (uint64_t)a * b + ((uint64_t)c << 32);
        uint32_t m = (uint32_t)T * pinv;
        uint32_t t = (uint32_t)((T + (uint64_t)m * p) >> 32);   // < 4p
        return min(t, t - p2);
    }
    __device__ __forceinline__ uint32_t add(uint32_t a, uint32_t b) const {
        uint32_t s = a + b;                     // < 4p < 2^32
        return min(s, s - p2);
    }
    // (a b + c d) R^{-1} mod p in [0, 2p) with one REDC: a, b, c < 2p and d < 4p, so
    // T < 12p^2 and T + m p < 3 2^62 + 2^62 = 2^64; the REDC output is < 4p.
    __device__ __forceinline__ uint32_t mul2add(uint32_t a, uint32_t b, uint32_t c, uint32_t d) const {
        uint64_t T = (uint64_t)a * b + (uint64_t)c * d;
        uint32_t m = (uint32_t)T * pinv;
        uint32_t t = (uint32_t)((T + (uint64_t)m * p) >> 32);
        return min(t, t - p2);
    }
    __device__ __forceinline__ uint32_t to(uint64_t x) const { return mul((uint32_t)(x % p), r2); }
    __device__ __forceinline__ uint64_t canon(uint32_t x) const {  // Montgomery -> [0, p)
        uint32_t r = mul(x, 1u);                // <= p
        return r >= p ? r - p : r;
    }
};

struct Mont64 {
    using W = uint64_t;
    uint64_t p, pinv, p2, r1, r2;

    __device__ __forceinline__ void init(uint64_t p64) {
        p = p64;
        p2 = 2 * p;
        uint64_t inv = p;
        #pragma unroll
        for (int i = 0; i < 5; i++) inv *= 2 - p * inv;      // 3 -> 96 bits
        pinv = 0 - inv;
        r1 = (0 - p) % p;                       // 2^64 mod p
        uint64_t x = r1;
        for (int i = 0; i < 64; i++) { x <<= 1; if (x >= p) x -= p; }   // r1 * 2^64 mod p
        r2 = x;
    }
    __device__ __forceinline__ uint64_t mul(uint64_t a, uint64_t b) const {
        uint64_t lo = a * b, hi = __umul64hi(a, b);
        uint64_t m = lo * pinv;
        return hi + __umul64hi(m, p) + (lo != 0);   // low words sum to 0 or R
    }
    __device__ __forceinline__ uint64_t muladd(uint64_t a, uint64_t b, uint64_t c) const {
        uint64_t lo = a * b, hi = __umul64hi(a, b);
        uint64_t m = lo * pinv;
        uint64_t t = hi + c + __umul64hi(m, p) + (lo != 0);     // < 4p
        return min(t, t - p2);
    }
    __device__ __forceinline__ uint64_t add(uint64_t a, uint64_t b) const {
        uint64_t s = a + b;
        return min(s, s - p2);
    }
    // (a b + c d) R^{-1} mod p: two REDCs (a 128-bit double product would not fit the lazy bound)
    __device__ __forceinline__ uint64_t mul2add(uint64_t a, uint64_t b, uint64_t c, uint64_t d) const {
        return add(mul(a, b), mul(c, d));
    }
    __device__ __forceinline__ uint64_t to(uint64_t x) const { return mul(x % p, r2); }
    __device__ __forceinline__ uint64_t canon(uint64_t x) const {
        uint64_t r = mul(x, 1);
        return r >= p ? r - p : r;
    }
};

// Exact modular arithmetic on the FP64 pipe (p < 2^44), a second engine beside
// the IMAD path.  Values are doubles holding integers; a product uses the
// error-free transform  a b = h + l  (h = fl(a b), l = fma(a, b, -h) exact),
// q = rint(h / p) via fma(h, 1/p, 1.5*2^52) - 1.5*2^52, and
//     a b - q p = fma(-q, p, h) + l        (both steps exact),
// so the result is congruent to a b mod p with |result| <= p whenever
// |a| <= 2p and |b| <= 2^49 (then q < 2^51, |q - h/p| <= 0.875 and
// |l| <= 2^-53 |h| <= p/8).  Residues stay "balanced" (signed) -- no
// conditional corrections in the hot loop.  All operations use _rn
// intrinsics so the compiler cannot re-associate or contract them.
struct ModD {
    double p, pinv;
    uint32_t rb2, rb3;      // reduction intervals (terms) for e = 2 and e = 3
    static constexpr double MAGIC = 6755399441055744.0;   // 1.5 * 2^52

    __device__ __forceinline__ void init(uint64_t p64) {
        p = (double)p64;
        pinv = __drcp_rn(p);
        const int lg = 64 - __clzll(p64);                  // p < 2^lg
        // e = 2: u grows by < p per term from <= p:      u <= (1 + j) p + j^2  <= 2^49
        // e = 3: d1 grows by < 3p+6j, u by d1:           u <= (1 + j + 4.5 j^2) p <= 2^49
        const int k2 = 48 - lg, k3 = (46 - lg) / 2;
        rb2 = k2 >= 20 ? (1u << 20) : (k2 < 1 ? 1u : (1u << k2));
        rb3 = k3 >= 20 ? (1u << 20) : (k3 < 1 ? 1u : (1u << k3));
    }
    __device__ __forceinline__ double rnd(double x) const {   // rint(x / p) for |x| < 2^51 p
        return __dadd_rn(__fma_rn(x, pinv, MAGIC), -MAGIC);
    }
    __device__ __forceinline__ double mul(double a, double b) const {
        const double h = __dmul_rn(a, b);
        const double l = __fma_rn(a, b, -h);
        const double q = rnd(h);
        return __dadd_rn(__fma_rn(-q, p, h), l);
    }
    __device__ __forceinline__ double reduce(double x) const { return __fma_rn(-rnd(x), p, x); }
    __device__ __forceinline__ uint64_t canon(double x) const {
        double r = reduce(x);
        if (r < 0) r = __dadd_rn(r, p);
        if (r >= p) r = __dadd_rn(r, -p);
        return (uint64_t)r;
    }
};

// signed integer -> residue in [0, p)   (no division when |a| < p)
__device__ __forceinline__ uint64_t smod(int64_t a, uint64_t p) {
    uint64_t m = a >= 0 ? (uint64_t)a : (uint64_t)(-a);
    if (m >= p) m %= p;
    return a >= 0 ? m : (m ? p - m : 0);
}

// x^(p-2) in Montgomery form (Fermat inverse of a unit x, lazy in / lazy out)
template <class M>
__device__ __forceinline__ typename M::W mont_inv(const M &mo, typename M::W x) {
    uint64_t e = mo.p - 2;
    typename M::W r = mo.r1;
    int top = 63 - __clzll(e);
    for (int i = top; i >= 0; i--) {
        r = mo.mul(r, r);
        if ((e >> i) & 1) r = mo.mul(r, x);
    }
    return r;
}

}  // namespace wv
