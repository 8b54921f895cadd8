/*
 * oracle/wv_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU reference for the quantities the
 * GPU path computes: B_{p-3} mod p (Wolstenholme test) and E_{p-3} mod p
 * (Vandiver test, secant convention).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this file's
 * shared object.  It shares no code, header, table or constant with
 * paper_2101_11157_b200/ (the product), and the product never calls it.
 *
 * Citations: "P:Lnnn" = /root/reference/PAPER.md line nnn (+ section /
 * equation label).  The oracle does not implement the paper's reduced
 * congruences (eqnBB*, eqnEE*) that the GPU path uses; it uses the plain
 * definitions and the classical O(p) formulas instead:
 *
 *   tier A (definition, O(p^2)):
 *     B_m mod p from the generating function z/(e^z-1) (P:L54-58,
 *       section 1) through its standard recurrence sum_{j<=m} C(m+1,j)B_j = 0;
 *     E_{2n} mod p from sec z (section 1) through
 *       sec z * cos z = 1.
 *   tier B (classical, O(p)):
 *     W: the first congruence of eqnWolst in its exact mod-p^2
 *        form  sum_{0<k<p} k^{-2} == (2/3) p B_{p-3}  (mod p^2)  (Glaisher;
 *        the "strengthening" equivalence stated at P:L45-50 with the
 *        residue made explicit by eqnGlaisher).  For p < 2^32 the
 *        residues mod p^2 fit one 64-bit word; for 2^32 <= p < 2^62 they are
 *        held as two base-p digits (schoolbook long multiplication, below).
 *        This is the W oracle for every p > 2000.
 *     W (pin only): eqnGlaisher itself with h = 2,
 *        C(2p-1, p-1) == 1 - (2/3) p^3 B_{p-3}  (mod p^4); p < 2^31.
 *     V: Glaisher's quarter-range formula eqnE1 at k = 1 (P:L748-756,
 *        section 4), with the sign reading of DESIGN.md "Readings" R1:
 *        -4 E_{p-3} == sum_{0<s<p/4} s^{-2}  (mod p).
 *   tier C (cross-check pin only, never dispatched): the Stafford-Vandiver
 *        congruence eqnSV at k = (p-3)/2, i.e. eqnBB1:
 *        21 B_{p-3} == sum_{p/6<s<p/4} s^{-3}  (mod p).  It is one of the
 *        paper's own reduced congruences, so it is kept only to be compared
 *        with tier B (tests), not as the oracle of any prime.
 *
 * Sums of inverses are accumulated as one fraction num/den, adding 1/u by
 * num/den + 1/u = (num*u + den)/(den*u) (all mod the modulus), with a single
 * modular inverse at the end: the schoolbook rule for adding fractions.
 *
 * Arithmetic is exact: unsigned 64-bit residues, 128-bit products, '%' and
 * '/' (for p^2 >= 2^64: base-p digit pairs, products by long multiplication).
 * Functions return UINT64_MAX when an argument is outside their domain.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
typedef uint64_t u64;

#define BAD UINT64_MAX

/* ------------------------------------------------------------------ */
/* modular helpers (modulus m < 2^64)                                  */
/* ------------------------------------------------------------------ */
static u64 mulmod(u64 a, u64 b, u64 m) { return (u64)(((u128)a * b) % m); }
static u64 addmod(u64 a, u64 b, u64 m) { return (u64)(((u128)a + b) % m); }
static u64 submod(u64 a, u64 b, u64 m) { a %= m; b %= m; return a >= b ? a - b : a + (m - b); }

/* inverse of a modulo m by the extended Euclidean algorithm; 0 if gcd != 1 */
static u64 invmod(u64 a, u64 m)
{
    __int128 t = 0, newt = 1;
    __int128 r = m, newr = a % m;
    while (newr != 0) {
        __int128 q = r / newr, tmp;
        tmp = t - q * newt; t = newt; newt = tmp;
        tmp = r - q * newr; r = newr; newr = tmp;
    }
    if (r != 1) return 0;
    if (t < 0) t += m;
    return (u64)t;
}

u64 oracle_invmod(u64 a, u64 m) { return invmod(a, m); }
u64 oracle_mulmod(u64 a, u64 b, u64 m) { return mulmod(a, b, m); }

/* ------------------------------------------------------------------ */
/* primes: sieve of Eratosthenes over [lo, hi), plain segmented form    */
/* ------------------------------------------------------------------ */
/* Writes the primes q with lo <= q < hi, ascending, into out (if out != NULL
 * and room remains); returns how many there are.  hi <= 2^40. */
u64 oracle_primes(u64 lo, u64 hi, u64 *out, u64 cap)
{
    if (hi <= lo || hi > ((u64)1 << 40)) return 0;
    u64 root = 1;
    while ((root + 1) * (root + 1) < hi) root++;
    /* small primes up to root by the textbook sieve */
    char *small = calloc(root + 2, 1);
    for (u64 i = 2; i <= root; i++) small[i] = 1;
    for (u64 i = 2; i * i <= root; i++)
        if (small[i])
            for (u64 j = i * i; j <= root; j += i) small[j] = 0;
    u64 count = 0;
    const u64 SEG = (u64)1 << 20;
    char *seg = malloc(SEG);
    for (u64 a = lo; a < hi; a += SEG) {
        u64 b = a + SEG < hi ? a + SEG : hi;
        memset(seg, 1, b - a);
        for (u64 q = 2; q <= root; q++) {
            if (!small[q]) continue;
            if (q * q >= b) break;
            u64 start = (a + q - 1) / q * q;
            if (start < q * q) start = q * q;
            for (u64 j = start; j < b; j += q) seg[j - a] = 0;
        }
        for (u64 n = a; n < b; n++) {
            if (n < 2 || !seg[n - a]) continue;
            if (out && count < cap) out[count] = n;
            count++;
        }
    }
    free(seg);
    free(small);
    return count;
}

/* ------------------------------------------------------------------ */
/* tier A: the definitions                                            */
/* ------------------------------------------------------------------ */

/* B_{n} mod p for 0 <= n <= p-3 from z/(e^z - 1) = sum B_k z^k/k!
 * (P:L54-58).  Multiplying by (e^z - 1)/z gives, for m >= 1,
 *     sum_{j=0}^{m} C(m+1, j) B_j = 0,
 * so B_m = -(m+1)^{-1} sum_{j<m} C(m+1, j) B_j.  Every B_j with j <= p-3 is
 * p-integral (von Staudt-Clausen) and m+1 <= p-2 is invertible mod p.
 * Writes B_0..B_n into out[0..n] (out may be NULL); returns B_n mod p.
 * Cost O(n^2) -- intended for p up to a few 10^4. */
u64 oracle_bernoulli_mod_p(u64 p, u64 n, u64 *out)
{
    if (p < 5 || n > p - 3) return BAD;
    u64 *B = malloc((n + 1) * sizeof(u64));
    u64 *row = calloc(n + 3, sizeof(u64)); /* row[j] = C(N, j) mod p */
    B[0] = 1;
    row[0] = 1; row[1] = 1;                /* N = 1 */
    u64 N = 1;
    for (u64 m = 1; m <= n; m++) {
        /* advance Pascal's row to N = m + 1 (in place, right to left) */
        while (N < m + 1) {
            N++;
            row[N] = 1;
            for (u64 j = N - 1; j >= 1; j--) row[j] = addmod(row[j], row[j - 1], p);
        }
        u64 acc = 0;
        for (u64 j = 0; j < m; j++) acc = addmod(acc, mulmod(row[j], B[j], p), p);
        B[m] = submod(0, mulmod(invmod((m + 1) % p, p), acc, p), p);
    }
    u64 r = B[n];
    if (out) memcpy(out, B, (n + 1) * sizeof(u64));
    free(B); free(row);
    return r;
}

/* E_{2n} mod p (secant convention: sec z = sum E_k z^k/k!, so
 * E_2 = 1, E_4 = 5) for 0 <= 2n <= p-3.  From sec z * cos z = 1 with
 * cos z = sum (-1)^j z^{2j}/(2j)!: for n >= 1,
 *     sum_{k=0}^{n} (-1)^{n-k} C(2n, 2k) E_{2k} = 0,
 * so E_{2n} = sum_{k<n} (-1)^{n-k+1} C(2n, 2k) E_{2k}.
 * Writes E_0, E_2, ..., E_{2n} into out[0..n]; returns E_{2n} mod p. */
u64 oracle_euler_mod_p(u64 p, u64 twon, u64 *out)
{
    if (p < 5 || (twon & 1) || twon > p - 3) return BAD;
    u64 n = twon / 2;
    u64 *E = malloc((n + 1) * sizeof(u64));
    u64 *row = calloc(twon + 3, sizeof(u64));
    E[0] = 1;
    row[0] = 1;
    u64 N = 0;
    for (u64 i = 1; i <= n; i++) {
        while (N < 2 * i) {
            N++;
            row[N] = 1;
            for (u64 j = N - 1; j >= 1; j--) row[j] = addmod(row[j], row[j - 1], p);
        }
        u64 acc = 0;
        for (u64 k = 0; k < i; k++) {
            u64 t = mulmod(row[2 * k], E[k], p);
            if ((i - k + 1) % 2 == 0) acc = addmod(acc, t, p);   /* (-1)^{i-k+1} = +1 */
            else acc = submod(acc, t, p);                         /* = -1 */
        }
        E[i] = acc;
    }
    u64 r = E[n];
    if (out) memcpy(out, E, (n + 1) * sizeof(u64));
    free(E); free(row);
    return r;
}

/* ------------------------------------------------------------------ */
/* tier B, W: harmonic sum of squares mod p^2                          */
/* ------------------------------------------------------------------ */
/* H2 = sum_{0<k<p} k^{-2} mod p^2 (the first form of eqnWolst).
 * Glaisher: H2 == (2/3) p B_{p-3} (mod p^2), so p | H2 and
 * B_{p-3} == (3/2) (H2 / p) (mod p).  Requires 5 <= p < 2^32 (p^2 < 2^64). */
u64 oracle_wolstenholme_h2(u64 p)
{
    if (p < 5 || p >= ((u64)1 << 32)) return BAD;
    u64 m = p * p;
    u64 num = 0, den = 1;              /* running fraction num/den */
    for (u64 k = 1; k < p; k++) {
        u64 u = k * k;                 /* k^2 < p^2: already reduced */
        num = addmod(mulmod(num, u, m), den, m);
        den = mulmod(den, u, m);
    }
    return mulmod(num, invmod(den, m), m);
}

u64 oracle_B_harmonic(u64 p)
{
    u64 h2 = oracle_wolstenholme_h2(p);
    if (h2 == BAD) return BAD;
    if (h2 % p != 0) return BAD;       /* Wolstenholme's theorem fails: impossible */
    u64 q = (h2 / p) % p;
    return mulmod(mulmod(q, 3, p), invmod(2, p), p);
}

/* ------------------------------------------------------------------ */
/* tier B, W for 2^32 <= p < 2^62: the same sum mod p^2 in base p       */
/* ------------------------------------------------------------------ */
/* A residue x mod p^2 is held as its two base-p digits, x = d0 + d1 p with
 * 0 <= d0, d1 < p.  Long multiplication in base p, dropping the p^2 column:
 *   (a0 + a1 p)(b0 + b1 p) = a0 b0 + (a0 b1 + a1 b0) p + a1 b1 p^2
 *                          == c0 + ((c1 + a0 b1 + a1 b0) mod p) p   (mod p^2),
 * where a0 b0 = c1 p + c0 (quotient and remainder).  For p < 2^62 every
 * intermediate is below 2p^2 + p < 2^126: exact in unsigned 128-bit. */
typedef struct { u64 d0, d1; } p2num;

static p2num p2_from(u128 x, u64 p)            /* x < p^2 */
{
    p2num r = { (u64)(x % p), (u64)(x / p) };
    return r;
}

static p2num p2_mul(p2num a, p2num b, u64 p)
{
    u128 t = (u128)a.d0 * b.d0;
    u64 c1 = (u64)(t / p);
    u64 c0 = (u64)(t - (u128)c1 * p);
    u128 col1 = (u128)a.d0 * b.d1 + (u128)a.d1 * b.d0 + c1;
    p2num r = { c0, (u64)(col1 % p) };
    return r;
}

static p2num p2_add(p2num a, p2num b, u64 p)    /* digit-wise with carry */
{
    u64 d0 = a.d0 + b.d0, carry = 0;
    if (d0 >= p) { d0 -= p; carry = 1; }
    u64 d1 = a.d1 + b.d1 + carry;
    if (d1 >= p) d1 -= p;
    p2num r = { d0, d1 };
    return r;
}

/* exported for the pins: (a0 + a1 p)(b0 + b1 p) mod p^2 as digits */
int oracle_p2_mul(u64 a0, u64 a1, u64 b0, u64 b1, u64 p, u64 *r0, u64 *r1)
{
    if (p < 2 || p >= ((u64)1 << 62) || a0 >= p || a1 >= p || b0 >= p || b1 >= p) return -1;
    p2num a = { a0, a1 }, b = { b0, b1 };
    p2num r = p2_mul(a, b, p);
    *r0 = r.d0; *r1 = r.d1;
    return 0;
}

static u128 invmod128(u128 a, u128 m);

/* H2 = sum_{0<k<p} k^{-2} mod p^2 for 5 <= p < 2^62, as digits (d0, d1).
 * The same running fraction as oracle_wolstenholme_h2: k^2 < p^2 is reduced
 * already; the single inverse of den (a unit mod p^2) is by Euclid on 128-bit
 * integers. */
int oracle_wolstenholme_h2_wide(u64 p, u64 *d0, u64 *d1)
{
    if (p < 5 || p >= ((u64)1 << 62)) return -1;
    p2num num = { 0, 0 }, den = { 1, 0 };
    for (u64 k = 1; k < p; k++) {
        p2num u = p2_from((u128)k * k, p);
        num = p2_add(p2_mul(num, u, p), den, p);
        den = p2_mul(den, u, p);
    }
    u128 m = (u128)p * p;
    u128 den_v = (u128)den.d1 * p + den.d0;
    u128 inv = invmod128(den_v, m);
    if (inv == 0) return -1;
    p2num h = p2_mul(num, p2_from(inv, p), p);
    *d0 = h.d0; *d1 = h.d1;
    return 0;
}

/* B_{p-3} mod p from H2 == (2/3) p B_{p-3} (mod p^2): p | H2 (Wolstenholme,
 * digit d0 = 0) and B_{p-3} == (3/2) d1 (mod p). */
u64 oracle_B_harmonic_wide(u64 p)
{
    u64 d0, d1;
    if (oracle_wolstenholme_h2_wide(p, &d0, &d1) != 0) return BAD;
    if (d0 != 0) return BAD;           /* Wolstenholme's theorem fails: impossible */
    return mulmod(mulmod(d1, 3, p), invmod(2, p), p);
}

/* ------------------------------------------------------------------ */
/* tier B, W (pin): Glaisher's binomial congruence mod p^4            */
/* ------------------------------------------------------------------ */
/* a*b mod m for m < 2^127, by shift-and-add (schoolbook binary method). */
static u128 mulmod128(u128 a, u128 b, u128 m)
{
    u128 r = 0;
    a %= m;
    int top = 127;
    while (top >= 0 && !((b >> top) & 1)) top--;
    for (int i = top; i >= 0; i--) {
        r <<= 1;
        if (r >= m) r -= m;
        if ((b >> i) & 1) { r += a; if (r >= m) r -= m; }
    }
    return r;
}

static u128 invmod128(u128 a, u128 m)
{
    /* Euclid on unsigned values with the Bezout coefficient kept mod m */
    u128 r0 = m, r1 = a % m, t0 = 0, t1 = 1;
    while (r1 != 0) {
        u128 q = r0 / r1, tmp;
        tmp = r0 - q * r1; r0 = r1; r1 = tmp;
        /* t0 - q*t1 mod m */
        u128 qt = mulmod128(q % m, t1, m);
        tmp = t0 >= qt ? t0 - qt : t0 + (m - qt);
        t0 = t1; t1 = tmp;
    }
    return r0 == 1 ? t0 : 0;
}

/* C(2p-1, p-1) mod p^4 = prod_{k=1}^{p-1} (p+k)/k  (eqnGlaisher with h = 2,
 * P:L59-64); returns the low and high 64-bit halves through lo/hi. */
int oracle_binom_2p_1_mod_p4(u64 p, u64 *lo, u64 *hi)
{
    if (p < 5 || p >= ((u64)1 << 31)) return -1;
    u128 m = (u128)p * p * p * p;
    u128 num = 1, den = 1;
    for (u64 k = 1; k < p; k++) {
        num = mulmod128(num, (u128)(p + k), m);
        den = mulmod128(den, (u128)k, m);
    }
    u128 c = mulmod128(num, invmod128(den, m), m);
    *lo = (u64)c; *hi = (u64)(c >> 64);
    return 0;
}

/* B_{p-3} mod p from C(2p-1,p-1) == 1 - (h(h-1)/3) p^3 B_{p-3} (mod p^4),
 * h = 2:  B_{p-3} == -(3/2) (C - 1)/p^3  (mod p). */
u64 oracle_B_glaisher(u64 p)
{
    u64 lo, hi;
    if (oracle_binom_2p_1_mod_p4(p, &lo, &hi) != 0) return BAD;
    u128 c = ((u128)hi << 64) | lo;
    u128 p3 = (u128)p * p * p;
    u128 d = c - 1;                     /* c >= 1 since c == 1 mod p^3 */
    if (d % p3 != 0) return BAD;        /* Wolstenholme mod p^3 */
    u64 q = (u64)((d / p3) % p);
    u64 t = mulmod(mulmod(q, 3, p), invmod(2, p), p);
    return submod(0, t, p);
}

/* ------------------------------------------------------------------ */
/* tier B, V: Glaisher's quarter sum                                   */
/* ------------------------------------------------------------------ */
/* Q = sum_{0<s<p/4} s^{-2} mod p (eqnE1, at k = 1: the
 * right side S_{p-3}(0, 1/4) == sum s^{-2}).  Valid for p < 2^63. */
u64 oracle_quarter_sum(u64 p)
{
    if (p < 5 || p >= ((u64)1 << 63)) return BAD;
    u64 last = p / 4;                  /* s < p/4 <=> s <= floor(p/4) (p odd, p/4 not an integer) */
    u64 num = 0, den = 1;
    for (u64 s = 1; s <= last; s++) {
        u64 u = mulmod(s, s, p);
        num = addmod(mulmod(num, u, p), den, p);
        den = mulmod(den, u, p);
    }
    return mulmod(num, invmod(den, p), p);
}

/* E_{p-3} mod p (secant convention): -4 E_{p-3} == Q (mod p)  (reading R1). */
u64 oracle_E_quarter(u64 p)
{
    u64 q = oracle_quarter_sum(p);
    if (q == BAD) return BAD;
    u64 t = mulmod(q, invmod(4, p), p);
    return submod(0, t, p);
}

/* ------------------------------------------------------------------ */
/* tier C, W: Stafford-Vandiver (eqnSV at k=(p-3)/2 == eqnBB1)          */
/* ------------------------------------------------------------------ */
/* 21 B_{p-3} == sum_{p/6 < s < p/4} s^{-3}  (mod p), P:L518 (from eqnSV,
 * P:L163-169, with C_k(3,4,6) == (6^3-3^3-4^3+1)/6 = 21 by P:L506-507).
 * Valid for p >= 5, p != 7; intended for 2^32 <= p < 2^62. */
u64 oracle_B_stafford_vandiver(u64 p)
{
    if (p < 5 || p == 7 || p >= ((u64)1 << 62)) return BAD;
    u64 first = p / 6 + 1;             /* s > p/6 */
    u64 last = p / 4;                  /* s < p/4 */
    u64 num = 0, den = 1;
    for (u64 s = first; s <= last; s++) {
        u64 u = mulmod(mulmod(s, s, p), s, p);
        num = addmod(mulmod(num, u, p), den, p);
        den = mulmod(den, u, p);
    }
    u64 S = mulmod(num, invmod(den, p), p);
    return mulmod(S, invmod(21, p), p);
}

/* ------------------------------------------------------------------ */
/* tier dispatch                                                       */
/* ------------------------------------------------------------------ */
#define TIER_A_MAX 2000u

u64 oracle_residue_B(u64 p)
{
    if (p < 5) return BAD;
    if (p <= TIER_A_MAX) return oracle_bernoulli_mod_p(p, p - 3, NULL);
    if (p < ((u64)1 << 32)) return oracle_B_harmonic(p);
    return oracle_B_harmonic_wide(p);
}

u64 oracle_residue_E(u64 p)
{
    if (p < 5) return BAD;
    if (p <= TIER_A_MAX) return oracle_euler_mod_p(p, p - 3, NULL);
    return oracle_E_quarter(p);
}
