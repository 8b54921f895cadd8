/*
 * wv.h -- C ABI of libwv.so, the B200 (sm_100a) Wolstenholme / Vandiver
 * residue search (Hathi, Mossinghoff, Trudgian, arXiv:2101.11157).
 *
 * Citations: "P:Lnnn" = /root/reference/PAPER.md line nnn with its section /
 * equation label; readings R1..R6 are listed in DESIGN.md.
 *
 * What the library computes (BASELINE.json north_star):
 * for every prime p with lo <= p < hi and p >= 5,
 *   W:  B_{p-3} mod p   (Bernoulli, z/(e^z-1) convention), via
 *       L_W B_{p-3} == sum_i a_i sum_{x_i p < s < y_i p} s^{-3}   (mod p)
 *       -- eqnBB1/2/6/9/16/22/30, eqnV12 at p = 7;
 *   V:  E_{p-3} mod p   (Euler, sec z convention; reading R1), via
 *       L_V E_{p-3} == sum_i a_i sum_{x_i p < s < y_i p} s^{-2}   (mod p)
 *       -- eqnEE3/5/9/16/24/33;
 * each inner sum evaluated by the (c0, c1) product recurrence eqnComputeS
 * and partial pairs merged by eqnCombinePairs.
 * A prime is a hit when its residue is 0 (Wolstenholme prime: p | B_{p-3},
 * P:L59-66; Vandiver prime: p | E_{p-3}).
 *
 * Conventions for every entry point:
 *  - integers are host-endian; residues are canonical in [0, p);
 *    WV_RES_NONE marks a test that was not requested;
 *  - ranges are half-open [lo, hi); primes < 5 are skipped; hi <= 2^62; one call handles
 *    windows with fewer than 2^32 primes (WV_EINVAL otherwise: sweep in blocks);
 *  - outputs are sorted ascending by p and identical for every shard count,
 *    block size and internal partition (the combine is exact);
 *  - the library never keeps caller pointers after a call returns;
 *  - all device work runs on the current CUDA device; device entry points
 *    run on the caller's stream, host entry points on an internal stream;
 *  - on a non-OK return, wv_last_error() gives a thread-local message.
 * There is no CPU fallback: without a usable sm_100 GPU every compute entry
 * point returns WV_ECUDA.
 */
#ifndef WV_H
#define WV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- codes */
#define WV_MODE_W    1u   /* Wolstenholme test: B_{p-3} mod p */
#define WV_MODE_V    2u   /* Vandiver test:     E_{p-3} mod p */
#define WV_MODE_BOTH 3u

#define WV_OK        0
#define WV_EINVAL   (-1)  /* lo >= hi, hi > 2^62, mode not in {1,2,3}, shard >= nshards, bad id */
#define WV_ENOSPC   (-2)  /* a caller capacity is too small; the *n_ outputs hold the sizes needed */
#define WV_ECUDA    (-3)  /* CUDA error (message in wv_last_error) */
#define WV_ENOMEM   (-4)  /* device allocation failed */

#define WV_RES_NONE UINT64_MAX
#define WV_HI_MAX   (UINT64_C(1) << 62)

#define WV_HIT_W 1u       /* p | numerator of B_{p-3}: Wolstenholme prime */
#define WV_HIT_V 2u       /* p | E_{p-3}: Vandiver prime */

typedef struct { uint64_t p; uint32_t flags; uint32_t reserved; } wv_hit;
typedef struct { uint64_t p; uint64_t res_w; uint64_t res_v; } wv_residue;

/* --------------------------------------------------------- host buffers */

/* wv_search: the whole hot path over [lo, hi) on the current device.
 *   out_hits[0..*n_hits)       primes with a zero residue and which test(s);
 *   out_residues[0..*n_primes) every prime with its residues (may be NULL:
 *                              then res_cap is ignored and only hits are returned).
 * Buffers are caller-owned host memory (pinned or pageable).  Two-call sizing:
 * if hits_cap < hits or (out_residues && res_cap < primes), returns WV_ENOSPC
 * with *n_hits / *n_primes set to the required counts and writes nothing else.
 * Device scratch is allocated (stream-ordered) and freed inside the call. */
int wv_search(uint64_t lo, uint64_t hi, uint32_t mode,
              wv_hit *out_hits, size_t hits_cap, size_t *n_hits,
              wv_residue *out_residues, size_t res_cap, size_t *n_primes);

/* wv_search_shard: as wv_search, restricted to this shard's blocks.  [lo, hi)
 * is cut into blocks of `block` integers (0 = default: a power of two giving
 * every shard >= 32 blocks, at least 2^15;
 * any block must be a multiple of 2^15, the sieve segment); block b = [lo + b*block, ...)
 * is dealt to shards in rounds of nshards, alternating direction ("snake"
 * interleave: round j gives block j*N + s - pad for even j and j*N + N-1-s - pad
 * for odd j to shard s, where pad = (-nblocks) mod N virtual empty blocks sit
 * below block 0 so that the rounds align with the top of the window and the one
 * partial round holds the lightest blocks), which balances the growth of
 * per-prime work with p.  *checksum
 * receives this shard's order-independent 64-bit checksum (wv_checksum_term
 * summed mod 2^64), so shard checksums add up to the unsharded one.
 * checksum may be NULL. */
int wv_search_shard(uint64_t lo, uint64_t hi, uint32_t mode,
                    uint32_t shard, uint32_t nshards, uint64_t block,
                    wv_hit *out_hits, size_t hits_cap, size_t *n_hits,
                    wv_residue *out_residues, size_t res_cap, size_t *n_primes,
                    uint64_t *checksum);

/* ------------------------------------------------------- device buffers */

/* Device-resident form of the same path (what bench.py's `value` times).
 * wv_device_workspace_bytes: bytes of device workspace wv_search_device needs
 * for these arguments (an upper bound fixed by (lo, hi, mode, shard, nshards,
 * block); it does not depend on the data) and the prime capacity the outputs
 * must have (*prime_cap, an upper bound on the primes in this shard from the
 * Montgomery-Vaughan bound pi(x+y)-pi(x) < 2y/log y). */
int wv_device_workspace_bytes(uint64_t lo, uint64_t hi, uint32_t mode,
                              uint32_t shard, uint32_t nshards, uint64_t block,
                              size_t *workspace_bytes, size_t *prime_cap);

/* wv_search_device: all pointers are device pointers (e.g. torch tensors).
 *   d_primes[prime_cap]   uint64 primes, ascending;
 *   d_res_w[prime_cap]    uint64 B_{p-3} mod p   (WV_RES_NONE if not requested);
 *   d_res_v[prime_cap]    uint64 E_{p-3} mod p   (WV_RES_NONE if not requested);
 *   d_hits[prime_cap]     wv_hit, ascending (may be NULL);
 *   d_checksum[1]         uint64 checksum of this shard (may be NULL);
 *   d_workspace           >= wv_device_workspace_bytes(...) bytes, 256-byte aligned
 *                         (NULL: the library allocates it stream-ordered);
 *   stream                a cudaStream_t (NULL = legacy default stream).
 * n_primes (host, may be NULL): the prime count (known after the plan step; the
 * call waits once for it).  n_hits (host, may be NULL): the hit count; the stream
 * is then synchronised.  With both NULL the call may return without waiting at all:
 * for a window whose primes are all < 2^30 under the default schedule (no
 * override, stats off) nothing is read back, the item counts stay on the device,
 * and the call returns once the last kernel is enqueued (hits, residues and
 * checksum are complete when the stream reaches that point); otherwise it waits
 * once after the plan step.  Returns WV_ENOSPC if prime_cap or workspace_bytes is
 * too small (nothing written). */
int wv_search_device(uint64_t lo, uint64_t hi, uint32_t mode,
                     uint32_t shard, uint32_t nshards, uint64_t block,
                     uint64_t *d_primes, uint64_t *d_res_w, uint64_t *d_res_v,
                     wv_hit *d_hits, uint64_t *d_checksum, size_t prime_cap,
                     void *d_workspace, size_t workspace_bytes, void *stream,
                     size_t *n_primes, size_t *n_hits);

/* wv_residues_device: the residue step alone for a caller-supplied list of
 * primes d_primes[0..n) (each >= 5, < 2^62, need not be sorted or distinct;
 * composite inputs give meaningless values).  Writes d_res_w[i], d_res_v[i]
 * as above.  Workspace as for wv_search_device, sized by
 * wv_residues_workspace_bytes(n, max_p, mode, ...). */
int wv_residues_workspace_bytes(size_t n, uint64_t max_p, uint32_t mode, size_t *workspace_bytes);
int wv_residues_device(const uint64_t *d_primes, size_t n, uint32_t mode,
                       uint64_t *d_res_w, uint64_t *d_res_v,
                       void *d_workspace, size_t workspace_bytes, void *stream);

/* wv_sieve_device: the sieve step alone: primes q with
 * max(lo,5) <= q < hi into d_primes[0..*n) ascending.  Returns WV_ENOSPC with
 * *n = count if cap is too small. */
int wv_sieve_device(uint64_t lo, uint64_t hi, uint64_t *d_primes, size_t cap, size_t *n,
                    void *d_workspace, size_t workspace_bytes, void *stream);

/* Near misses and histograms.
 * For residues already on the device (e.g. the outputs of wv_search_device):
 *   symmetric residue <r>_p in (-p/2, p/2];
 *   near miss: |<r>_p| < bound  -> d_out[] entries (unordered), *n_out = count
 *     (if the count exceeds cap, only cap entries are written and WV_ENOSPC
 *      is returned with *n_out = the full count);
 *   histogram: 2000 equal bins of <r>_p / p over (-1/2, 1/2],
 *     bin = floor(2000 (<r>_p + p/2) / p) computed exactly; d_hist_w/v[2000]
 *     uint64 counts are ADDED to (zero them first); either may be NULL.
 * Tests whose residue array holds WV_RES_NONE are skipped.  Synchronises the stream. */
typedef struct { uint64_t p; int64_t symres; uint32_t test; uint32_t reserved; } wv_nearmiss;  /* test 1=W, 2=V */
int wv_near_misses_device(const uint64_t *d_primes, const uint64_t *d_res_w, const uint64_t *d_res_v, size_t n,
                          uint64_t bound, wv_nearmiss *d_out, size_t cap, size_t *n_out,
                          uint64_t *d_hist_w, uint64_t *d_hist_v, void *d_workspace, void *stream);

/* wv_prime_count: number of primes q with max(lo,5) <= q < hi, counted by the
 * same segmented sieve without materialising them (used to pin the sieve to
 * the paper's counts).  Device scratch is internal. */
int wv_prime_count(uint64_t lo, uint64_t hi, uint64_t *count);

/* wv_shard_blocks: host-only (no GPU) description of the interleaved partition
 * used by wv_search_shard: writes the integer ranges [lo_i, hi_i) of this
 * shard's blocks (clipped to [lo, hi), empty ones skipped) into out[2*i],
 * out[2*i+1] for i < cap, sets *n to their number and *block_used to the block
 * size actually used (the default when block == 0).  WV_ENOSPC if cap < *n. */
int wv_shard_blocks(uint64_t lo, uint64_t hi, uint32_t shard, uint32_t nshards, uint64_t block,
                    uint64_t *out, size_t cap, size_t *n, uint64_t *block_used);

/* ------------------------------------------------------ small utilities */

/* Checksum term of one prime (reading R6 in DESIGN.md):
 * mix64(p ^ rotl(res_w, 21) ^ rotl(res_v, 42)), mix64 = splitmix64 finaliser.
 * Checksums are sums of terms mod 2^64. */
uint64_t wv_checksum_term(uint64_t p, uint64_t res_w, uint64_t res_v);

/* Congruence table (host copy of the constants the kernels use).
 * id 0..wv_congruence_count()-1.  Each congruence states
 *   L * X == sum_{j<m} a_j * S(xn_j/xd_j, yn_j/yd_j)  (mod p),
 * S(x,y) = sum_{xp<s<yp} s^{-e}; X = B_{p-3} (e = 3) or E_{p-3} (e = 2).
 * Valid for p >= min_p and p != excluded_p.  Returns WV_EINVAL for a bad id. */
typedef struct { int64_t a; uint32_t xn, xd, yn, yd; } wv_term;
typedef struct {
    char     name[8];       /* "BB30", "EE33", "VOR12", ... */
    int64_t  L;             /* left factor */
    uint32_t e;             /* 3: B_{p-3} (s^-3);  2: E_{p-3} (s^-2) */
    uint32_t m;             /* number of sums */
    uint32_t min_p;
    uint32_t excluded_p;    /* 0 = none */
    wv_term  t[33];
} wv_congruence;
int wv_congruence_count(void);
int wv_congruence_get(int id, wv_congruence *out);   /* WV_EINVAL if m > 33 or |a| >= 2^63 */

/* Any congruence, including the generated many-sum ones (NEXT-2): coefficients and the
 * left factor are sign + 128-bit magnitude (hi * 2^64 + lo).  seg = 1 means the kernels
 * cut its work into sum-aligned chunks. */
typedef struct {
    char name[8];
    uint64_t L_lo, L_hi;
    uint32_t L_neg, e, m, min_p, excluded_p, seg;
} wv_cong_header;
typedef struct { uint64_t a_lo, a_hi; uint32_t neg, xn, xd, yn, yd; } wv_term128;
int wv_congruence_header(int id, wv_cong_header *out);
int wv_congruence_term(int id, uint32_t j, wv_term128 *out);

/* Schedule override for tests and benchmarking (process-global, not
 * thread-safe): force congruence ids for W and V (-1 restores the default
 * schedule).  The caller must respect validity (min_p / excluded_p); an
 * invalid forced choice for some p gives WV_EINVAL from the search. */
int wv_set_schedule_override(int w_id, int v_id);
/* Default schedule (each p takes the tier with the largest threshold <= p):
 *   W: p = 5 BB1, p = 7 VOR12, 11 <= p < 4096 BB1, 4096 <= p < 2^17 BB30,
 *      2^17 <= p < 2^24 "BG_SML", 2^24 <= p < 2^30 "BG_XL", p >= 2^30 "BG_BIG";
 *   V: p < 4096 EE3, 4096 <= p < 2^17 EE33, 2^17 <= p < 2^21 "EG_SML",
 *      2^21 <= p < 2^24 "EG_MID", 2^24 <= p < 2^30 "EG_XL", p >= 2^30 "EG_BIG";
 * the quoted names are the generated congruences of congruences_gen.inc (greedy continuations of
 * BB30 / EE33, and of eqnVandiver / eqnEMac2 for the many-sum tiers).  "BG_MID" is built but in no
 * default range; WV_TH_<name> (read once) sets any generated tier's threshold (0 disables it).
 * Returns the id used. */
int wv_schedule(uint64_t p, uint32_t test /* WV_MODE_W or WV_MODE_V */);

/* Measurement hooks (process-wide, for bench.py / profiling).  When enabled,
 * every residue-kernel launch is bracketed by CUDA events on its stream and
 * the elapsed times are accumulated at the call's final synchronisation.
 *   terms      algorithmic terms evaluated (sum over (prime,test) of the
 *              congruence's term count);
 *   residue_ms summed device time of residue-kernel launches;
 *   residue_launches, records ((prime,test) pairs), chunks (warp work items). */
typedef struct {
    uint64_t terms;
    uint64_t terms32;          /* of which class 0: p < 2^30 (Mont32 combine) */
    uint64_t terms_fp;         /* of which class 1: 2^30 <= p < 2^44 (FP64 engine) */
    uint64_t residue_launches;
    uint64_t records;
    uint64_t chunks;
    double   residue_ms;
    double   residue32_ms;     /* class-0 kernel time */
    double   residue_fp_ms;    /* class-1 kernel time */
} wv_stats;
int wv_stats_enable(int on);
int wv_stats_get(wv_stats *out);
int wv_stats_reset(void);

/* Residue-kernel variants (benchmarking / tests; process-global, not
 * thread-safe).  Primes fall in three classes: 0: p < 2^30 (32-bit
 * Montgomery), 1: 2^30 <= p < 2^44 (FP64 engine by default), 2: p >= 2^44
 * (64-bit Montgomery).  A variant fixes the kernel: for class 0 the lane-mode
 * kernel ("c0 lane2", default; one prime per lane, sorted prime lists from the
 * sieve) or a chunk kernel (engine, interleaved term streams per lane); for
 * class 1 the K-term FP64 steps ("c1 fp tuples K2/K3", default 6/6) or the
 * term-by-term FP64 / IMAD engines; for class 2 the K-term 64-bit Montgomery
 * steps with lazy difference tables ("c2 int tuples K2/K3", default 8/8) or the
 * term-by-term Mont64 engine ("c2 int s1/1").  wv_kernel_variant_info returns the name
 * and class of variant id (WV_EINVAL past the end); wv_set_kernel_variant
 * selects it for its class (-1 restores the default).  Results are identical
 * for every variant.  Environment knobs read per call (benchmarking only; the
 * results never change): WV_VARIANT0/1/2 (default variant per class, read once),
 * WV_LANE_ITEMS (lane-mode slices: items per resident warp, default 2),
 * WV_LANE_CHAIN (lane-mode chain mode, bit 0: e = 2, bit 2: e = 3 with
 * four-term steps (else pair steps per sum); default 5), WV_TH_<tier> (schedule threshold of a generated tier, read once). */
int wv_kernel_variant_info(int id, char *name, size_t name_cap, int *cls);
int wv_set_kernel_variant(int cls, int id);

/* ------------------------------------------- general-index residues (NEXT-3)
 * The irregular-pair census of P:L88-103: for every prime p in [lo, hi)
 * (p >= 5, hi <= 2^26) and every even index 2 <= 2k <= p-3,
 *   B_{2k} mod p  (mode bit 1) from eqnSV for general k,
 *       C_k(3,4,6) B_{2k} == S_{2k-1}(1/6, 1/4)  (mod p),
 *       C_k(a,b,c) = (a^{p-2k} + b^{p-2k} - c^{p-2k} - 1)/(4k);
 *     where C_k(3,4,6) == 0 (mod p), from the first of VOR (2,3,4),
 *     (4,5,8), eqnVandiver, eqnTW1 b = 2, 4, 6, 7,
 *     8, 9, ... whose C_k is a unit (WV_ECUDA "no unit C_k" if
 *     none up to b = 1031: not seen for any p < 30000, where b <= 28 suffices);
 *   E_{2k} mod p  (mode bit 2, secant convention) from eqnE1
 *     read as  (-1)^j 4^{2j-1} E_{p-1-2j} == S_{p-1-2j}(0, 1/4)  (reading R10,
 *     the printed sign (-1)^{(p-1)/2-j} is wrong for half the j).
 * All exponents of a prime are evaluated together by a walk over the
 * multiplicative group (powers of a primitive root): (p-1)/2 walk steps
 * per index, i.e. ~p^2/2 per prime for both kinds -- a census workload for
 * p up to ~10^6, not for the frontier primes.
 *
 * wv_census: p | B_{2k} ("irregular pair (p, 2k)", kind 1) and p | E_{2k}
 * ("E-irregular pair", kind 2) into out[0..cap), sorted by (p, kind, index);
 * *n_pairs = their number (WV_ENOSPC if > cap, nothing written past cap);
 * *n_primes = primes in the window; *checksum = sum mod 2^64 over every
 * computed (p, index, kind, residue) of wv_census_checksum_term.  Any
 * out-pointer may be NULL.  Runs on the library's device stream; synchronous.
 * Errors: WV_EINVAL (lo >= hi, hi > 2^26, mode not in {1,2,3}), WV_ENOMEM,
 * WV_ECUDA. */
typedef struct { uint64_t p; uint32_t index; uint32_t kind; } wv_pair;
int wv_census(uint64_t lo, uint64_t hi, uint32_t mode, wv_pair *out, size_t cap, size_t *n_pairs,
              size_t *n_primes, uint64_t *checksum);
/* wv_census_residues: the residues themselves, one record per (p, index),
 * p ascending then index = 2, 4, ..., p-3; res_b / res_e = UINT64_MAX for a
 * kind not requested.  *n = sum over primes of (p-3)/2; WV_ENOSPC (nothing
 * computed) if cap < *n. */
typedef struct { uint64_t p; uint32_t index; uint32_t reserved; uint64_t res_b; uint64_t res_e; } wv_index_residue;
int wv_census_residues(uint64_t lo, uint64_t hi, uint32_t mode, wv_index_residue *out, size_t cap, size_t *n);
/* mix64(p ^ (index << 32) ^ rotl(res, 17) ^ (kind << 62)), mix64 = splitmix64 finaliser */
uint64_t wv_census_checksum_term(uint64_t p, uint32_t index, uint32_t kind, uint64_t res);

/* Counters: kernels launched by this library since load (process-wide). */
uint64_t wv_launch_count(void);
/* Library / device info string (build flags, sm, ...). */
const char *wv_version(void);
const char *wv_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* WV_H */
