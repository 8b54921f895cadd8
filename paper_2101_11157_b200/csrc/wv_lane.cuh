// wv_lane.cuh -- class-0 lane-mode residue kernel (sorted prime lists, 5 <= p < 2^30).
//
// A warp item is (group of 32 consecutive primes of one test, slice q of Q).  Lane l owns
// record (32 g + l, test) and walks every sum j of its congruence.
// Neighbouring primes share the congruence and have nearly equal term counts, so all lanes cross
// sum boundaries together: per sum one unmasked loop of min-count steps, then a short masked tail.
// (The chunk kernel splits one record over 64 lane streams instead; with C2-size primes and ~90-sum
// congruences its streams cross sum boundaries at different times and the lockstep loop breaks
// every ~8 terms.)
//
// Arithmetic: everything in Montgomery form x R mod p (R = 2^32), lazy in [0, 2p), with the
// subtractive REDC  m = T_lo p^{-1} mod R,  REDC(T) = T_hi - hi(m p) + p  -- the low words cancel
// exactly, so no carry is propagated -- which lies in (0, p + T_hi].
//
// The sum of inverses is the ratio a1/a0 of eqnComputeS, advanced K terms at a time:
//     1/u_0 + ... + 1/u_{K-1} = N / D,   D = prod u_i,  N = sum_i prod_{j != i} u_j,  u_i = (s+i)^e,
//     a1 <- REDC(a1 D + a0 N),   a0 <- REDC(a0 D)          (ratio += N/D; one REDC for both products)
// D(s), N(s) are polynomials in s (degree Ke, (K-1)e) advanced by step-K forward differences with
// modular adds only.  K = 4 for both tests (LaneRun2Q, LaneRunP<3,4>); the pair step with
// u = s^3 by unit differences (LaneRun3) serves e = 3 outside chain mode.
// Chain mode (lane2_chain_item): the sums, sorted by left endpoint, form chains of adjacent
// intervals whose terms are consecutive integers, so one table runs through a chain.
// At the end of a sum: c1 <- a_j c1 (fold) and (C0, C1) (+) (c0, c1) (eqnCombinePairs).
#pragma once
#include <stdint.h>
#include <type_traits>
#include "wv_residue.cuh"

namespace wv {

// first s and count of x p < s < y p (strict) for p < 2^32: exact.
__device__ __forceinline__ void lane_bounds(uint32_t p, const Term &t, double2 rr, uint64_t &first, uint32_t &cnt) {
    const uint64_t f = fdiv((uint64_t)t.xn * p, t.xd, rr.x) + 1;                  // floor(x p) + 1
    const uint64_t l = fdiv((uint64_t)t.yn * p + t.yd - 1, t.yd, rr.y) - 1;       // ceil(y p) - 1
    first = f;
    cnt = l >= f ? (uint32_t)(l - f + 1) : 0u;
}

struct MontS {      // p < 2^30, R = 2^32, values lazy in [0, 2p)
    uint32_t p, pinv, p2, r1, r2;        // pinv = p^{-1} mod 2^32 (positive); r1 = R mod p; r2 = R^2 mod p
    __device__ __forceinline__ void init(uint32_t p_) {
        p = p_;
        p2 = 2u * p;
        uint32_t inv = p;                                    // p p == 1 mod 8
        #pragma unroll
        for (int i = 0; i < 4; i++) inv *= 2u - p * inv;     // 3 -> 48 bits
        pinv = inv;
        r1 = (uint32_t)(0x100000000ull % p);
        r2 = (uint32_t)(((uint64_t)r1 * r1) % p);
    }
    // T R^{-1} mod p, in (0, p + T_hi]
    __device__ __forceinline__ uint32_t redc(uint64_t T) const {
        const uint32_t m = (uint32_t)T * pinv;
        return (uint32_t)(T >> 32) - __umulhi(m, p) + p;
    }
    // a, b < 2p: a b < 4p^2 < p 2^32, result in (0, 2p)
    __device__ __forceinline__ uint32_t mul(uint32_t a, uint32_t b) const { return redc((uint64_t)a * b); }
    // (a b + c d) R^{-1}: BIG (p < 2^30, all < 2p): T < 8p^2, REDC in (0, 3p), one lazy subtract;
    // !BIG (p < 2^28, a, b, c < 2p, d < 4p): T < 12 p^2 < p 2^32, REDC already in (0, 2p).
    template <bool BIG>
    __device__ __forceinline__ uint32_t mul2add(uint32_t a, uint32_t b, uint32_t c, uint32_t d) const {
        const uint32_t t = redc((uint64_t)a * b + (uint64_t)c * d);
        return BIG ? min(t, t - p2) : t;
    }
    // l < 2^32, r < 2p: T < 2^33 p, REDC in (0, 3p) -> [0, 2p)
    __device__ __forceinline__ uint32_t mulw(uint32_t l, uint32_t r) const {
        const uint32_t t = redc((uint64_t)l * r);
        return min(t, t - p2);
    }
    __device__ __forceinline__ uint32_t add(uint32_t a, uint32_t b) const {
        const uint32_t s = a + b;
        return min(s, s - p2);
    }
    __device__ __forceinline__ uint32_t sub(uint32_t a, uint32_t b) const {
        const uint32_t s = a - b + p2;                       // (0, 4p)
        return min(s, s - p2);
    }
};

// a_j R mod p from the 128-bit magnitude (4 limbs) and sign; rho[i] = R^{i+2} mod p
__device__ __forceinline__ uint32_t lane_coef(const MontS &mo, const Term &t, const uint32_t rho[4]) {
    uint32_t a = mo.mulw((uint32_t)t.a_lo, rho[0]);
    if (t.a_lo >> 32) a = mo.add(a, mo.mulw((uint32_t)(t.a_lo >> 32), rho[1]));
    if (t.a_hi) {
        a = mo.add(a, mo.mulw((uint32_t)t.a_hi, rho[2]));
        a = mo.add(a, mo.mulw((uint32_t)(t.a_hi >> 32), rho[3]));
    }
    if (t.neg) a = mo.sub(0u, a);
    return a;
}

// e = 3 run: u = s^3 and its unit-step differences (3s^2+3s+1, 6s+6, 6), Montgomery form.
struct LaneRun3 {
    static constexpr uint32_t K = 2;
    uint32_t u, d1, d2, d3, a0, a1;
    __device__ __forceinline__ void setup(const MontS &mo, uint32_t x) {
        const uint32_t xt = mo.mul(x, mo.r2);
        const uint32_t xx = mo.mul(xt, xt);
        u = mo.mul(xx, xt);
        const uint32_t r3 = mo.add(mo.add(mo.r1, mo.r1), mo.r1);
        const uint32_t x3 = mo.add(mo.add(xt, xt), xt);
        d1 = mo.add(mo.add(mo.add(xx, xx), xx), mo.add(x3, mo.r1));
        d3 = mo.add(r3, r3);
        d2 = mo.add(mo.add(x3, x3), d3);
        a0 = mo.r1;
        a1 = 0;
    }
    template <bool BIG, bool MASK>
    __device__ __forceinline__ void pair(const MontS &mo, bool act) {
        const uint32_t u2 = mo.add(u, d1);
        d1 = mo.add(d1, d2);
        d2 = mo.add(d2, d3);
        const uint32_t N = BIG ? mo.add(u, u2) : u + u2;
        const uint32_t D = mo.mul(u, u2);
        u = mo.add(u2, d1);
        d1 = mo.add(d1, d2);
        d2 = mo.add(d2, d3);
        const uint32_t n1 = mo.mul2add<BIG>(a1, D, a0, N);
        const uint32_t n0 = mo.mul(a0, D);
        a1 = (!MASK || act) ? n1 : a1;
        a0 = (!MASK || act) ? n0 : a0;
    }
    // one term s = x (x < p), masked; u is recomputed (masked pair steps advanced it for every lane)
    template <bool BIG>
    __device__ __forceinline__ void single(const MontS &mo, uint32_t x, bool act) {
        const uint32_t xt = mo.mul(x, mo.r2);
        const uint32_t w = mo.mul(mo.mul(xt, xt), xt);
        const uint32_t n1 = mo.mul2add<BIG>(a1, w, a0, mo.r1);
        const uint32_t n0 = mo.mul(a0, w);
        a1 = act ? n1 : a1;
        a0 = act ? n0 : a0;
    }
    static __device__ __forceinline__ uint32_t term_w(const MontS &mo, uint32_t x) {   // x^3 R
        const uint32_t xt = mo.mul(x, mo.r2);
        return mo.mul(mo.mul(xt, xt), xt);
    }
    // table + accumulators advance only where act (masked steps of chain mode keep tables aligned)
    template <bool BIG>
    __device__ __forceinline__ void pair_all(const MontS &mo, bool act) {
        const auto old = *this;
        pair<BIG, false>(mo, true);
        if (!act) *this = old;
    }
    // the table advances one step where act; the accumulators are left alone
    template <bool BIG>
    __device__ __forceinline__ void advance(const MontS &mo, bool act) {
        const auto old = *this;
        pair<BIG, false>(mo, true);
        a0 = old.a0;
        a1 = old.a1;
        if (!act) *this = old;
    }
};

// e = 2 run, four terms per step: 1/u0 + 1/u1 + 1/u2 + 1/u3 = N / D with
//     D(s) = (s (s+1) (s+2) (s+3))^2                      (degree 8)
//     N(s) = u1 u2 u3 + u0 u2 u3 + u0 u1 u3 + u0 u1 u2       (degree 6),  u_i = (s+i)^2,
// advanced by step-4 forward differences: per four terms the same 2 products (3 wide multiplies,
// one shared REDC) as a pair step, plus 14 modular adds.  The tables are set up from D and N at
// 9 and 7 points, N = P01 (u2 + u3) + P23 (u0 + u1) with P01 = u0 u1, P23 = u2 u3.
struct LaneRun2Q {
    static constexpr uint32_t K = 4;
    uint32_t D0, D1, D2, D3, D4, D5, D6, D7, Dc, N0, N1, N2, N3, N4, N5, Nc, a0, a1;
    __device__ __forceinline__ void setup(const MontS &mo, uint32_t x) {   // x < p
        const uint32_t xt = mo.mul(x, mo.r2);
        uint32_t u = mo.mul(xt, xt);                                        // s^2 R at s = x
        uint32_t d1 = mo.add(mo.add(xt, xt), mo.r1);                        // (2s + 1) R
        const uint32_t d2 = mo.add(mo.r1, mo.r1);                           // 2 R
        uint32_t v[9], w[7];
        #pragma unroll
        for (int i = 0; i < 9; i++) {
            uint32_t q[4];
            #pragma unroll
            for (int k = 0; k < 4; k++) {
                q[k] = u;
                u = mo.add(u, d1);
                d1 = mo.add(d1, d2);
            }
            const uint32_t P01 = mo.mul(q[0], q[1]), P23 = mo.mul(q[2], q[3]);
            v[i] = mo.mul(P01, P23);
            if (i < 7) w[i] = mo.mul2add<true>(P01, mo.add(q[2], q[3]), P23, mo.add(q[0], q[1]));
        }
        #pragma unroll
        for (int k = 1; k < 9; k++) {
            #pragma unroll
            for (int i = 8; i >= k; i--) v[i] = mo.sub(v[i], v[i - 1]);
        }
        #pragma unroll
        for (int k = 1; k < 7; k++) {
            #pragma unroll
            for (int i = 6; i >= k; i--) w[i] = mo.sub(w[i], w[i - 1]);
        }
        D0 = v[0]; D1 = v[1]; D2 = v[2]; D3 = v[3]; D4 = v[4]; D5 = v[5]; D6 = v[6]; D7 = v[7]; Dc = v[8];
        N0 = w[0]; N1 = w[1]; N2 = w[2]; N3 = w[3]; N4 = w[4]; N5 = w[5]; Nc = w[6];
        a0 = mo.r1;
        a1 = 0;
    }
    template <bool BIG, bool MASK>
    __device__ __forceinline__ void pair(const MontS &mo, bool act) {       // one step = four terms
        const uint32_t n1 = mo.mul2add<BIG>(a1, D0, a0, N0);
        const uint32_t n0 = mo.mul(a0, D0);
        a1 = (!MASK || act) ? n1 : a1;
        a0 = (!MASK || act) ? n0 : a0;
        D0 = mo.add(D0, D1); D1 = mo.add(D1, D2); D2 = mo.add(D2, D3); D3 = mo.add(D3, D4);
        D4 = mo.add(D4, D5); D5 = mo.add(D5, D6); D6 = mo.add(D6, D7); D7 = mo.add(D7, Dc);
        N0 = mo.add(N0, N1); N1 = mo.add(N1, N2); N2 = mo.add(N2, N3); N3 = mo.add(N3, N4);
        N4 = mo.add(N4, N5); N5 = mo.add(N5, Nc);
    }
    template <bool BIG>
    __device__ __forceinline__ void single(const MontS &mo, uint32_t x, bool act) {
        const uint32_t xt = mo.mul(x, mo.r2);
        const uint32_t w = mo.mul(xt, xt);
        const uint32_t n1 = mo.mul2add<BIG>(a1, w, a0, mo.r1);
        const uint32_t n0 = mo.mul(a0, w);
        a1 = act ? n1 : a1;
        a0 = act ? n0 : a0;
    }
    static __device__ __forceinline__ uint32_t term_w(const MontS &mo, uint32_t x) {   // x^2 R
        const uint32_t xt = mo.mul(x, mo.r2);
        return mo.mul(xt, xt);
    }
    // table + accumulators advance only where act (masked steps of chain mode keep tables aligned)
    template <bool BIG>
    __device__ __forceinline__ void pair_all(const MontS &mo, bool act) {
        const auto old = *this;
        pair<BIG, false>(mo, true);
        if (!act) *this = old;
    }
    // the table advances one step where act; the accumulators are left alone
    template <bool BIG>
    __device__ __forceinline__ void advance(const MontS &mo, bool act) {
        const auto old = *this;
        pair<BIG, false>(mo, true);
        a0 = old.a0;
        a1 = old.a1;
        if (!act) *this = old;
    }
};

// General K-term run for e = 2 or 3 (Montgomery form): D(s) = prod_{i<K} (s+i)^e (degree Ke) and
// N(s) = sum_i prod_{j != i} (s+j)^e (degree (K-1)e), step-K forward differences.  The tables are set
// up from D and N at Ke + 1 and (K-1)e + 1 points, each from K consecutive u = s^e (unit-step
// differences) with prefix / suffix products.  LaneRun2Q is the hand-written e = 2, K = 4 case.
template <int EE, int KK>
struct LaneRunP {
    static constexpr uint32_t K = KK;
    static constexpr int DD = KK * EE, DN = (KK - 1) * EE;
    uint32_t D[DD + 1], N[DN + 1], a0, a1;
    __device__ __forceinline__ void setup(const MontS &mo, uint32_t x) {   // x < p
        const uint32_t xt = mo.mul(x, mo.r2);
        const uint32_t xx = mo.mul(xt, xt);
        uint32_t u, d1, d2, d3 = 0;
        if (EE == 3) {
            const uint32_t r3 = mo.add(mo.add(mo.r1, mo.r1), mo.r1);
            const uint32_t x3 = mo.add(mo.add(xt, xt), xt);
            u = mo.mul(xx, xt);                                             // x^3
            d1 = mo.add(mo.add(mo.add(xx, xx), xx), mo.add(x3, mo.r1));     // 3x^2 + 3x + 1
            d3 = mo.add(r3, r3);                                            // 6
            d2 = mo.add(mo.add(x3, x3), d3);                                // 6x + 6
        } else {
            u = xx;                                                         // x^2
            d1 = mo.add(mo.add(xt, xt), mo.r1);                             // 2x + 1
            d2 = mo.add(mo.r1, mo.r1);                                      // 2
        }
        #pragma unroll
        for (int i = 0; i <= DD; i++) {
            uint32_t q[KK], pre[KK + 1], suf[KK + 1];
            #pragma unroll
            for (int k = 0; k < KK; k++) {
                q[k] = u;
                u = mo.add(u, d1);
                d1 = mo.add(d1, d2);
                if (EE == 3) d2 = mo.add(d2, d3);
            }
            pre[1] = q[0];
            #pragma unroll
            for (int k = 1; k < KK; k++) pre[k + 1] = mo.mul(pre[k], q[k]);
            D[i] = pre[KK];
            if (i <= DN) {
                suf[KK - 1] = q[KK - 1];
                #pragma unroll
                for (int k = KK - 2; k >= 1; k--) suf[k] = mo.mul(suf[k + 1], q[k]);
                uint32_t n = mo.add(suf[1], pre[KK - 1]);                   // prod_{j != 0} + prod_{j != K-1}
                #pragma unroll
                for (int k = 1; k < KK - 1; k++) n = mo.add(n, mo.mul(pre[k], suf[k + 1]));
                N[i] = n;
            }
        }
        #pragma unroll
        for (int k = 1; k <= DD; k++) {
            #pragma unroll
            for (int i = DD; i >= k; i--) D[i] = mo.sub(D[i], D[i - 1]);
        }
        #pragma unroll
        for (int k = 1; k <= DN; k++) {
            #pragma unroll
            for (int i = DN; i >= k; i--) N[i] = mo.sub(N[i], N[i - 1]);
        }
        a0 = mo.r1;
        a1 = 0;
    }
    template <bool BIG, bool MASK>
    __device__ __forceinline__ void pair(const MontS &mo, bool act) {       // one step = K terms
        const uint32_t n1 = mo.mul2add<BIG>(a1, D[0], a0, N[0]);
        const uint32_t n0 = mo.mul(a0, D[0]);
        a1 = (!MASK || act) ? n1 : a1;
        a0 = (!MASK || act) ? n0 : a0;
        #pragma unroll
        for (int i = 0; i < DD; i++) D[i] = mo.add(D[i], D[i + 1]);
        #pragma unroll
        for (int i = 0; i < DN; i++) N[i] = mo.add(N[i], N[i + 1]);
    }
    static __device__ __forceinline__ uint32_t term_w(const MontS &mo, uint32_t x) {   // x^e R
        const uint32_t xt = mo.mul(x, mo.r2);
        const uint32_t x2 = mo.mul(xt, xt);
        return EE == 3 ? mo.mul(x2, xt) : x2;
    }
    template <bool BIG>
    __device__ __forceinline__ void single(const MontS &mo, uint32_t x, bool act) {
        const uint32_t w = term_w(mo, x);
        const uint32_t n1 = mo.mul2add<BIG>(a1, w, a0, mo.r1);
        const uint32_t n0 = mo.mul(a0, w);
        a1 = act ? n1 : a1;
        a0 = act ? n0 : a0;
    }
    template <bool BIG>
    __device__ __forceinline__ void pair_all(const MontS &mo, bool act) {
        const auto old = *this;
        pair<BIG, false>(mo, true);
        if (!act) *this = old;
    }
    template <bool BIG>
    __device__ __forceinline__ void advance(const MontS &mo, bool act) {
        const auto old = *this;
        pair<BIG, false>(mo, true);
        a0 = old.a0;
        a1 = old.a1;
        if (!act) *this = old;
    }
};

// One item: every sum of the lane's congruence, slice q of Q.  Returns the merged (C0, C1).
template <class Run, bool BIG>
__device__ __forceinline__ void lane2_item(const MontS &mo, const Cong &cg, bool valid, uint64_t q, uint64_t Q,
                                           double rQ, uint32_t &C0, uint32_t &C1, uint64_t &nterms) {
    const uint32_t m = valid ? cg.m : 0u;
    const uint32_t mmax = __reduce_max_sync(0xffffffffu, m);
    uint32_t rho[4];
    rho[0] = mo.r2;
    rho[1] = mo.mul(mo.r2, mo.r2);
    rho[2] = mo.mul(rho[1], mo.r2);
    rho[3] = mo.mul(rho[2], mo.r2);
    for (uint32_t j = 0; j < mmax; j++) {
        uint32_t cnt = 0;
        uint64_t s0 = 1;
        Term tm;
        if (j < m) {
            tm = c_terms[cg.off + j];
            uint64_t f;
            uint32_t n;
            lane_bounds(mo.p, tm, c_termr[cg.off + j], f, n);
            uint64_t a = 0, b = n;
            if (Q > 1) {
                a = fdiv((uint64_t)n * q, (uint32_t)Q, rQ);
                b = fdiv((uint64_t)n * (q + 1), (uint32_t)Q, rQ);
            }
            cnt = (uint32_t)(b - a);
            s0 = f + a;
        }
        const bool act = cnt != 0;
        nterms += cnt;
        const uint32_t np = cnt / Run::K;                        // steps of K terms, then cnt % K singles
        const uint32_t kmin = __reduce_min_sync(0xffffffffu, act ? np : 0xffffffffu);
        if (kmin == 0xffffffffu) continue;                       // no lane has terms in this sum
        const uint32_t kmax = __reduce_max_sync(0xffffffffu, act ? np : 0u);
        const uint32_t rem = act ? cnt - np * Run::K : 0u;
        Run run;
        run.setup(mo, (uint32_t)s0);
        uint32_t i = 0;
        #pragma unroll 1
        for (; i + 4 <= kmin; i += 4) {
            run.template pair<BIG, false>(mo, true);
            run.template pair<BIG, false>(mo, true);
            run.template pair<BIG, false>(mo, true);
            run.template pair<BIG, false>(mo, true);
        }
        #pragma unroll 1
        for (; i < kmin; i++) run.template pair<BIG, false>(mo, true);
        #pragma unroll 1
        for (; i < kmax; i++) run.template pair<BIG, true>(mo, i < np);
        const uint32_t rmax = __reduce_max_sync(0xffffffffu, rem);
        #pragma unroll 1
        for (uint32_t r = 0; r < rmax; r++)
            run.template single<BIG>(mo, (uint32_t)(s0 + (uint64_t)Run::K * np + r), r < rem);
        if (act) {
            const uint32_t c1 = mo.mul(run.a1, lane_coef(mo, tm, rho));          // fold a_j
            const uint32_t n1 = mo.mul2add<true>(C0, c1, C1, run.a0);            // eqnCombinePairs
            C0 = mo.mul(C0, run.a0);
            C1 = n1;
        }
    }
}


__constant__ uint32_t c_lane_chain = 5u;   // bit 0: chain mode for e = 2; bit 2: chain mode with four-term steps
                                           // for e = 3 (else pair steps per sum) (WV_LANE_CHAIN)

// Chain mode: the sums of a congruence sorted by left endpoint fall into chains of adjacent intervals
// (x_{j+1} = y_j, flagged in Term.pad): for p >= 7 their terms are consecutive integers (R5), so one
// difference table and ONE accumulator run through the whole chain, and the sums are separated by
// summation by parts (Abel):  with P_j the running sum of s^-e through the end of sum j,
//     sum_j a_j S_j = a_J P_J - sum_{j < J} (a_{j+1} - a_j) P_j .
// At the end of sum j the lane takes a snapshot P_j = the accumulator plus the r < K terms of sum j
// that do not fill a whole K-term step (single terms, u recomputed, on a copy), folds it with
// a_j - a_{j+1} (a_J for the last sum) and merges it into (C0, C1); the r terms stay pending and
// enter the accumulator with the next step.  Per sum: bounds, coefficient, < K singles, one fold +
// merge -- no table set-up and no accumulator restart.  (The generated congruences have 91 / 87 sums
// in 47 / 24 chains (BG_SML / EG_SML), 3534 / 3535 in 1192 / 1065 (BG_BIG / EG_BIG).)
// Every lane of the warp must have the same congruence (the caller checks).  Slices cut the lane's
// terms of all chains, concatenated in chain order, into Q pieces (prefix sums over the slice's terms;
// the identity holds for any P sequence).  A lane whose next sum does not start where its previous one ended (p < 7, R5) absorbs
// its pending terms and realigns its table there; a realignment sets up every lane's table at its
// own position (accumulators kept).
template <class Run, bool BIG, bool SL>     // SL: the item is a slice (Q > 1); Q == 1 compiles without the cut
__device__ __forceinline__ void lane2_chain_item(const MontS &mo, const Cong &cg, bool valid, uint64_t q, uint64_t Q,
                                                 double rQ, uint32_t &C0, uint32_t &C1, uint64_t &nterms) {
    constexpr uint32_t K = Run::K;
    const uint32_t m = cg.m;
    uint32_t rho[4];
    rho[0] = mo.r2;
    rho[1] = mo.mul(mo.r2, mo.r2);
    rho[2] = mo.mul(rho[1], mo.r2);
    rho[3] = mo.mul(rho[2], mo.r2);
    // slice q of Q: the lane's terms of all chains, concatenated in chain order, cut into Q pieces
    // [g_lo, g_hi), so a slice sets up tables only for the chains it overlaps
    uint64_t g_lo = 0, g_hi = 0, base = 0;
    if (SL) {
        uint64_t tot = 0;
        if (valid) {
            for (uint32_t a = 0; a < m;) {
                uint32_t b = a;
                while (b + 1 < m && (c_terms[cg.off + b].pad & 1u)) b++;
                uint64_t f0, f1;
                uint32_t n0, n1;
                lane_bounds(mo.p, c_terms[cg.off + a], c_termr[cg.off + a], f0, n0);
                lane_bounds(mo.p, c_terms[cg.off + b], c_termr[cg.off + b], f1, n1);
                tot += f1 + n1 > f0 ? f1 + n1 - f0 : 0;
                a = b + 1;
            }
        }
        g_lo = fdiv(tot * q, (uint32_t)Q, rQ);
        g_hi = fdiv(tot * (q + 1), (uint32_t)Q, rQ);
    }
    uint32_t j = 0;
    while (j < m) {
        if (SL && __all_sync(0xffffffffu, !valid || base >= g_hi)) break;   // past every lane's slice
        uint32_t je = j;
        while (je + 1 < m && (c_terms[cg.off + je].pad & 1u)) je++;
        uint64_t F = 1, E = 1;
        uint64_t fc = 1;                              // bounds of the chain's current sum (computed once)
        uint32_t nc = 0;
        if (valid) {
            uint64_t f1;
            uint32_t n1;
            lane_bounds(mo.p, c_terms[cg.off + j], c_termr[cg.off + j], fc, nc);
            lane_bounds(mo.p, c_terms[cg.off + je], c_termr[cg.off + je], f1, n1);
            F = fc;
            E = f1 + n1 > F ? f1 + n1 : F;
        }
        uint64_t lo = F, hi = E;
        if (SL) {
            const uint64_t w = E - F;
            const uint64_t a = g_lo > base ? g_lo - base : 0, b = g_hi > base ? g_hi - base : 0;
            lo = F + (a < w ? a : w);
            hi = F + (b < w ? b : w);
            base += valid ? w : 0;
        }
        if (!__any_sync(0xffffffffu, valid && lo < hi)) {
            j = je + 1;
            continue;
        }
        // a slice (Q > 1) starts inside the chain: its sums that end before every lane's slice start add
        // nothing (empty running sum), so only their bounds are computed
        uint32_t j0 = j;
        while (SL && j0 < je && !__any_sync(0xffffffffu, valid && fc + nc > lo)) {
            j0++;
            if (valid) lane_bounds(mo.p, c_terms[cg.off + j0], c_termr[cg.off + j0], fc, nc);
        }
        Run run;
        run.setup(mo, (uint32_t)lo);
        uint64_t t = lo, tp = lo;                     // accumulator covers [lo, t); the table sits at tp
        uint32_t coef = valid ? lane_coef(mo, c_terms[cg.off + j0], rho) : 0u;
        bool done = false;                            // this lane's slice ended in an earlier sum
        for (uint32_t jj = j0; jj <= je; jj++) {
            const bool act = valid && !done;
            const uint64_t f = fc;
            const uint32_t n = nc;
            uint32_t coef_n = 0;
            if (jj < je && act) {
                lane_bounds(mo.p, c_terms[cg.off + jj + 1], c_termr[cg.off + jj + 1], fc, nc);
                coef_n = lane_coef(mo, c_terms[cg.off + jj + 1], rho);
            }
            if (__any_sync(0xffffffffu, act && t != tp)) {            // realign every lane's table at t
                const uint32_t s0 = run.a0, s1 = run.a1;
                run.setup(mo, (uint32_t)(act ? t : 1));
                run.a0 = s0;
                run.a1 = s1;
                tp = t;
            }
            // this sum's end within the slice; steps of K while they fit, r < K terms left over
            uint64_t b = f + n < hi ? f + n : hi;
            if (b < t) b = t;
            const uint32_t cnt = act ? (uint32_t)(b - t) : 0u;
            const uint32_t ns = cnt / K, r = cnt - ns * K;
            // over the lanes still working: a lane whose slice ended (done) has no terms left and never reads
            // its run state again, so the unmasked steps may advance it
            const uint32_t kmin = __reduce_min_sync(0xffffffffu, act ? ns : 0xffffffffu);
            const uint32_t kmax = __reduce_max_sync(0xffffffffu, act ? ns : 0u);
            uint32_t i = 0;
            #pragma unroll 1
            for (; i + 4 <= kmin; i += 4) {
                run.template pair<BIG, false>(mo, true);
                run.template pair<BIG, false>(mo, true);
                run.template pair<BIG, false>(mo, true);
                run.template pair<BIG, false>(mo, true);
            }
            #pragma unroll 1
            for (; i < kmin; i++) run.template pair<BIG, false>(mo, true);
            #pragma unroll 1
            for (; i < kmax; i++) run.template pair_all<BIG>(mo, i < ns);
            t += (uint64_t)K * ns;
            tp += (uint64_t)K * ns;
            // snapshot P_jj = accumulator + the r pending terms [t, t + r)
            uint32_t s0 = run.a0, s1 = run.a1;
            const uint32_t rmax = __reduce_max_sync(0xffffffffu, r);
            #pragma unroll 1
            for (uint32_t k = 0; k < rmax; k++) {
                const uint32_t w = Run::term_w(mo, (uint32_t)(t + k));
                const uint32_t n1 = mo.mul2add<BIG>(s1, w, s0, mo.r1);
                const uint32_t n0 = mo.mul(s0, w);
                const bool act = k < r;
                s1 = act ? n1 : s1;
                s0 = act ? n0 : s0;
            }
            // the slice ends in this sum (or the chain does): every later running sum equals this one,
            // so their Abel weights telescope to a_jj and the lane is done with the chain
            const bool last = jj == je || (SL && f + n >= hi);
            if (act) {
                nterms += (uint64_t)K * ns + (last ? r : 0u);         // pending terms count where absorbed
                // Abel weight: a_jj - a_{jj+1} inside the chain, a_jj where the slice or chain ends
                const uint32_t wgt = last ? coef : mo.sub(coef, coef_n);
                const uint32_t c1 = mo.mul(s1, wgt);
                const uint32_t m1 = mo.mul2add<true>(C0, c1, C1, s0);            // eqnCombinePairs
                C0 = mo.mul(C0, s0);
                C1 = m1;
                done = last;
            }
            if (SL && __all_sync(0xffffffffu, !valid || done)) break;
            coef = coef_n;
            // next sum not contiguous for this lane: absorb the pending terms and continue at the next
            // sum's first term (its table is realigned above)
            if (jj < je && act && fc != t + r) {
                run.a0 = s0;
                run.a1 = s1;
                nterms += r;
                if (t + r >= hi) {                      // the slice ended: nothing left to step
                    t = tp = hi;
                } else {
                    t = fc > t + r ? fc : t + r;
                }
            }
        }
        j = je + 1;
    }
}

// items it in [item_lo, item_lo + nitems) processed largest-first (groups ascend in p); gstart = exclusive scan of
// gq (slices per group-test); start = per-record partial slots.
// Step widths in chain mode (terms per step) for W (e = 3) and V (e = 2); build-time choices.
#ifndef WV_LANE_KW
#define WV_LANE_KW 4
#endif
#ifndef WV_LANE_KV
#define WV_LANE_KV 4
#endif
using RunW = LaneRunP<3, WV_LANE_KW>;
using RunV = std::conditional<WV_LANE_KV == 4, LaneRun2Q, LaneRunP<2, WV_LANE_KV>>::type;   // K = 4: hand-written

// Resident blocks per SM the register allocation targets: 2 (up to 128 registers, 16 warps/SM).
// Measured on C2 (residue ms): 4 blocks (64 registers, spills in the per-sum code) 12.18, 3: 11.59,
// 2: 11.13, 1: 11.05; 2 keeps more warps for small windows.
#ifndef WV_LANE2_MINB
#define WV_LANE2_MINB 2
#endif
__global__ void __launch_bounds__(RES_THREADS, WV_LANE2_MINB)
residue_lane2_kernel(const Rec *__restrict__ recs, const uint64_t *__restrict__ start,
                     const uint64_t *__restrict__ gstart, const uint64_t *__restrict__ gq, uint64_t ngt,
                     uint64_t item_lo, uint64_t nitems_host, const uint64_t *__restrict__ nitems_dev, uint32_t ntests,
                     uint64_t K, uint64_t part_base, ulonglong2 *__restrict__ partials,
                     unsigned long long *__restrict__ counter, unsigned long long *__restrict__ term_count,
                     uint32_t allsl_mode, const unsigned long long *__restrict__ slice_counts) {
    // item count: from the host, or (asynchronous launches) the device-side total gstart[ngt]
    const uint64_t nitems = nitems_dev ? *nitems_dev - item_lo : nitems_host;
    // allsl_mode 0 / 1: forced; 2: most lane group-tests sliced (slice_counts[0] of slice_counts[1])
    const bool all_sliced = allsl_mode == 2 ? 2 * slice_counts[0] > slice_counts[1] : allsl_mode != 0;
    const uint32_t chain_mask = c_lane_chain;          // bit 0: chain mode for e = 2, bit 2: for e = 3
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned long long it = 0;
        if (lane == 0) it = atomicAdd(counter, 1ull);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= nitems) break;
        const uint64_t item = item_lo + nitems - 1 - it;          // this batch's items [item_lo, item_lo + nitems)
        const uint64_t gt = find_rec(gstart, 0, ngt, item);
        const uint64_t q = item - gstart[gt], Q = gq[gt];
        const uint64_t g = gt / ntests, t = gt % ntests;
        const uint64_t k = (32 * g + lane) * ntests + t;
        Rec r;
        r.p = 0;
        if (k < K) r = recs[k];
        const bool valid = r.p != 0 && r.p < WIDTH32_MAX;
        const Cong &cg = c_cong[valid ? r.cid : 0];
        MontS mo;
        mo.init(valid ? (uint32_t)r.p : 7u);
        uint32_t C0 = mo.r1, C1 = 0;
        const double rQ = 1.0 / (double)Q;
        const uint32_t e = __reduce_max_sync(0xffffffffu, valid ? cg.e : 0u);   // one test per item
        const bool big = __any_sync(0xffffffffu, valid && r.p >= (1ull << 28));
        uint64_t nterms = 0;
        // chain mode when every valid lane has the same congruence (all but groups at a tier threshold)
        const uint32_t vm = __ballot_sync(0xffffffffu, valid);
        const uint32_t cid0 = __shfl_sync(0xffffffffu, r.cid, vm ? __ffs(vm) - 1 : 0);
        const bool chain = vm && __all_sync(0xffffffffu, !valid || r.cid == cid0) &&
                           ((chain_mask >> (e == 3 ? 2 : 0)) & 1u);
        // the sliced chain variant (SL) for slices, and for whole groups too when most groups of the launch
        // are sliced: one hot code path per test instead of two (N-way shards of C2: instruction-fetch
        // stalls fell from 22 % of the samples; the result is the same, a whole group is slice 0 of 1)
        const bool sl = Q > 1 || all_sliced;
        if (chain) {
            const Cong &cu = c_cong[cid0];
            // (six-term steps, LaneRunP<3, 6> / <2, 6>, measured slower: C2 residue 17.3 / 15.7 ms vs 13.1)
            // (chains with W pair steps measured slower than without: C2 residue 13.64 vs 13.29 ms; no longer built)
            if (e == 3) {                                  // four-term W steps
                if (sl) {
                    if (big) lane2_chain_item<RunW, true, true>(mo, cu, valid, q, Q, rQ, C0, C1, nterms);
                    else lane2_chain_item<RunW, false, true>(mo, cu, valid, q, Q, rQ, C0, C1, nterms);
                } else {
                    if (big) lane2_chain_item<RunW, true, false>(mo, cu, valid, q, Q, rQ, C0, C1, nterms);
                    else lane2_chain_item<RunW, false, false>(mo, cu, valid, q, Q, rQ, C0, C1, nterms);
                }
            } else {
                if (sl) {
                    if (big) lane2_chain_item<RunV, true, true>(mo, cu, valid, q, Q, rQ, C0, C1, nterms);
                    else lane2_chain_item<RunV, false, true>(mo, cu, valid, q, Q, rQ, C0, C1, nterms);
                } else {
                    if (big) lane2_chain_item<RunV, true, false>(mo, cu, valid, q, Q, rQ, C0, C1, nterms);
                    else lane2_chain_item<RunV, false, false>(mo, cu, valid, q, Q, rQ, C0, C1, nterms);
                }
            }
        } else if (e == 3) {
            if (big) lane2_item<LaneRun3, true>(mo, cg, valid, q, Q, rQ, C0, C1, nterms);
            else lane2_item<LaneRun3, false>(mo, cg, valid, q, Q, rQ, C0, C1, nterms);
        } else {
            if (big) lane2_item<LaneRun2Q, true>(mo, cg, valid, q, Q, rQ, C0, C1, nterms);
            else lane2_item<LaneRun2Q, false>(mo, cg, valid, q, Q, rQ, C0, C1, nterms);
        }
        if (valid) partials[start[k] + q - part_base] = make_ulonglong2(C0, C1);
        if (term_count) {                                   // executed terms (stats; the plan skips them)
            uint64_t w = nterms;
            #pragma unroll
            for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
            if (lane == 0) atomicAdd(term_count, (unsigned long long)w);
        }
    }
}

}  // namespace wv
