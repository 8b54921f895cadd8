// wv_api.cu -- host runtime and C ABI of libwv.so (declared in include/wv.h).
//
// Host-side responsibilities only: argument checks, workspace layout, the
// launch sequence (sieve -> plan -> scan -> residue -> finalize -> flags/hits),
// batching of the partial-pair buffer, and host<->device copies for the
// host-buffer entry points.  Every arithmetic step of the method runs in the
// kernels of wv_sieve.cuh / wv_residue.cuh.
#include <cuda_runtime.h>
#include <math.h>
#include <nvtx3/nvToolsExt.h>   // NVTX v3, header-only: ranges cost nothing unless a profiler is attached
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <vector>

#include "../../include/wv.h"
#include "wv_mont.cuh"
#include "wv_residue.cuh"
#include "wv_lane.cuh"
#include "wv_scan.cuh"
#include "wv_sieve.cuh"
#include "wv_census.cuh"

using namespace wv;

// ------------------------------------------------------------------ constants
// default schedule: the printed congruences, plus generated many-sum ones (if present) for large p;
// finalised in sched_init() once the generated table is known
static Sched g_sched = {{{0, 4096}, {0, 4096}}, {{C_BB1, C_BB30}, {C_EE3, C_EE33}}, {2, 2}, -1, -1};
// printed congruences of the paper (int64 coefficients, <= 33 sums)
struct SmallTerm { int64_t a; uint32_t xn, xd, yn, yd; };
struct SmallCong { char name[8]; int64_t L; uint32_t e, m, min_p, excluded_p; SmallTerm t[33]; };
#define WV_CONG(NAME, L, E, M, MINP, EXCL, ...) {NAME, (int64_t)(L), E, M, MINP, EXCL, __VA_ARGS__},
static const SmallCong h_small[] = {
#include "congruences.inc"
};
#undef WV_CONG
static const int NSMALL = sizeof h_small / sizeof h_small[0];

// generated congruences (scripts/gen_congruences.py -> congruences_gen.inc): 128-bit coefficients
struct GenCong { const char *name; uint32_t L_neg; uint64_t L_hi, L_lo; uint32_t e, m, min_p, excluded_p, seg; };
struct GenTerm { uint32_t neg; uint64_t hi, lo; uint32_t xn, xd, yn, yd; };
#include "congruences_gen.inc"

// generated-congruence tiers (name, test, threshold): names from congruences_gen.inc
struct GenTier { const char *name; int test; uint64_t th; };
// th = 0: not in the default schedule (BG_MID, p/34.3 with 305 sums, measured slower than BG_SML / BG_XL
// everywhere); WV_TH_<name> enables or moves a tier.  The schedule uses, for each p,
// the tier with the largest threshold <= p (sched_init sorts them).
static GenTier kGenTiers[] = {
    {"BG_SML", 0, 1ull << 17}, {"BG_MID", 0, 0}, {"BG_XL", 0, 1ull << 24}, {"BG_BIG", 0, 1ull << 30},
    {"EG_SML", 1, 1ull << 17}, {"EG_MID", 1, 1ull << 21}, {"EG_XL", 1, 1ull << 24}, {"EG_BIG", 1, 1ull << 30},
};

// uniform host copy of every congruence: headers + one term array (uploaded per device)
struct Table {
    std::vector<Cong> hdr;
    std::vector<Term> terms;
    Table() {
        for (int i = 0; i < NSMALL; i++) {
            const SmallCong &s = h_small[i];
            Cong c{};
            memcpy(c.name, s.name, 8);
            c.L_lo = (uint64_t)(s.L < 0 ? -s.L : s.L);
            c.L_hi = 0;
            c.L_neg = s.L < 0;
            c.e = s.e; c.m = s.m; c.min_p = s.min_p; c.excluded_p = s.excluded_p;
            c.seg = 0;
            c.off = (uint32_t)terms.size();
            for (uint32_t j = 0; j < s.m; j++) {
                const SmallTerm &t = s.t[j];
                terms.push_back(Term{(uint64_t)(t.a < 0 ? -t.a : t.a), 0, t.a < 0 ? 1u : 0u, t.xn, t.xd, t.yn, t.yd, 0});
            }
            hdr.push_back(c);
        }
        uint32_t k = 0;
        for (int i = 0; i < NGEN; i++) {
            const GenCong &g = kGenCong[i];
            Cong c{};
            strncpy(c.name, g.name, 7);
            c.L_lo = g.L_lo; c.L_hi = g.L_hi; c.L_neg = g.L_neg;
            c.e = g.e; c.m = g.m; c.min_p = g.min_p; c.excluded_p = g.excluded_p; c.seg = g.seg;
            c.off = (uint32_t)terms.size();
            for (uint32_t j = 0; j < g.m; j++, k++) {
                const GenTerm &t = kGenTerms[k];
                terms.push_back(Term{t.lo, t.hi, t.neg, t.xn, t.xd, t.yn, t.yd, 0});
            }
            hdr.push_back(c);
        }
    }
};
static void sched_init(const Table &t);
static const Table &table() {
    static Table t;
    static bool once = false;
    if (!once) {
        once = true;
        sched_init(t);
    }
    return t;
}
static void sched_init(const Table &t) {
    // benchmarking knob: WV_SML_TH_W / WV_SML_TH_V override the small-tier thresholds (0 disables)
    const char *ew = getenv("WV_SML_TH_W"), *ev = getenv("WV_SML_TH_V");
    for (GenTier &g : kGenTiers) {
        if (!strcmp(g.name, "BG_SML") && ew) g.th = strtoull(ew, nullptr, 0);
        if (!strcmp(g.name, "EG_SML") && ev) g.th = strtoull(ev, nullptr, 0);
        char key[32];                                     // WV_TH_<tier name>: any tier's threshold
        snprintf(key, sizeof key, "WV_TH_%s", g.name);
        if (const char *e = getenv(key)) g.th = strtoull(e, nullptr, 0);
    }
    std::vector<GenTier> tiers(std::begin(kGenTiers), std::end(kGenTiers));
    std::stable_sort(tiers.begin(), tiers.end(), [](const GenTier &a, const GenTier &b) { return a.th < b.th; });
    for (const GenTier &g : tiers) {
        if (g.th == 0) continue;
        for (size_t i = NSMALL; i < t.hdr.size(); i++) {
            if (strncmp(t.hdr[i].name, g.name, 7) != 0) continue;
            int &n = g_sched.n[g.test];
            if (n >= SCHED_TIERS) {   // cannot happen with the built-in table (static_assert below)
                fprintf(stderr, "libwv: schedule holds %d tiers per test; %s dropped\n", SCHED_TIERS, g.name);
                continue;
            }
            if (g_sched.th[g.test][n - 1] >= g.th) continue;   // at or below an earlier threshold: dropped
            g_sched.th[g.test][n] = g.th;
            g_sched.id[g.test][n] = (int)i;
            n++;
        }
    }
}
static_assert(sizeof kGenTiers / sizeof kGenTiers[0] / 2 + 2 <= SCHED_TIERS, "schedule tier capacity");

// odd primes below 256: the bootstrap list that sieves [3, 65536)
static const uint32_t h_boot[] = {3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61, 67,
                                  71, 73, 79, 83, 89, 97, 101, 103, 107, 109, 113, 127, 131, 137, 139,
                                  149, 151, 157, 163, 167, 173, 179, 181, 191, 193, 197, 199, 211, 223,
                                  227, 229, 233, 239, 241, 251};
static const uint64_t BASE0_HI = 65536;

// ------------------------------------------------------------------ NVTX ranges (nsys / ncu --nvtx)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

// ------------------------------------------------------------------ errors
static thread_local char g_err[1024] = "";
static std::atomic<uint64_t> g_launches{0};

// measurement hooks
static std::atomic<int> g_stats_on{0};
static std::mutex g_stats_mu;
static wv_stats g_stats;
struct EvPair { cudaEvent_t a, b; int cls; };

static int set_err(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

#define CK(x)                                                                                        \
    do {                                                                                             \
        cudaError_t e_ = (x);                                                                        \
        if (e_ != cudaSuccess)                                                                       \
            return set_err(e_ == cudaErrorMemoryAllocation ? WV_ENOMEM : WV_ECUDA, "%s:%d %s: %s",   \
                           __FILE__, __LINE__, #x, cudaGetErrorString(e_));                          \
    } while (0)
#define TRY(x)                       \
    do {                             \
        int r_ = (x);                \
        if (r_ != WV_OK) return r_;  \
    } while (0)
#define LAUNCH(kern, grid, block, st, ...)                          \
    do {                                                            \
        kern<<<(grid), (block), 0, (st)>>>(__VA_ARGS__);            \
        g_launches.fetch_add(1, std::memory_order_relaxed);         \
        CK(cudaGetLastError());                                     \
    } while (0)

// ------------------------------------------------------------------ residue kernel variants
// (prime class, engine, streams per lane for e = 2 / e = 3 sums); selected per class by the
// env vars WV_VARIANT0/1/2 (index into this table) for benchmarking; defaults below.
typedef void (*ResKern)(const Rec *, const uint64_t *, uint64_t, uint64_t, uint64_t, uint64_t, uint64_t, ulonglong2 *,
                        unsigned long long *, uint32_t, const uint32_t *, uint32_t);
typedef void (*LaneKern)(const Rec *, const uint64_t *, const uint64_t *, const uint64_t *, uint64_t, uint64_t, uint64_t,
                         const uint64_t *, uint32_t, uint64_t, uint64_t, ulonglong2 *, unsigned long long *,
                         unsigned long long *, uint32_t, const unsigned long long *);
struct Variant { const char *name; int cls; ResKern fn; LaneKern lane; };
static const Variant kVariants[] = {
    {"c0 int s1/1", 0, residue_kernel<Mont32, 0, 0, 1, 1>, nullptr},
    {"c0 int s2/2", 0, residue_kernel<Mont32, 0, 0, 2, 2>, nullptr},
    {"c0 int s3/2", 0, residue_kernel<Mont32, 0, 0, 3, 2>, nullptr},
    {"c0 int s3/3", 0, residue_kernel<Mont32, 0, 0, 3, 3>, nullptr},
    {"c0 fp s1/1", 0, residue_kernel<Mont32, 0, 1, 1, 1>, nullptr},
    {"c1 fp s1/1", 1, residue_kernel<Mont64, 1, 1, 1, 1>, nullptr},
    {"c1 fp s2/2", 1, residue_kernel<Mont64, 1, 1, 2, 2>, nullptr},
    {"c1 int s1/1", 1, residue_kernel<Mont64, 2, 0, 1, 1>, nullptr},
    {"c2 int s1/1", 2, residue_kernel<Mont64, 2, 0, 1, 1>, nullptr},
    {"c2 int s2/2", 2, residue_kernel<Mont64, 2, 0, 2, 2>, nullptr},
    {"c0 lane int", 0, nullptr, residue_lane_kernel<Mont32, 0, 0>},   // lane mode (sorted lists)
    {"c0 lane fp", 0, nullptr, residue_lane_kernel<Mont32, 0, 1>},
    {"c0 int s1/1 pairs", 0, residue_kernel<Mont32, 0, 0, 1, 1, true>, nullptr},
    {"c0 int s2/2 pairs", 0, residue_kernel<Mont32, 0, 0, 2, 2, true>, nullptr},
    {"c2 int s1/1 pairs", 2, residue_kernel<Mont64, 2, 0, 1, 1, true>, nullptr},
    {"c0 lane2", 0, nullptr, residue_lane2_kernel},                   // lane mode v2 (sorted lists)
    // K-term FP64 steps for sum-aligned congruences (K for e = 2 / e = 3); measured on C4/C5 heads:
    // 4/4 620/371 ms, 6/4 621/352, 6/5 583/342, 8/4 628/347, 8/5 594/337, 6/6 565/340, 8/6 560/334,
    // 8/7 578/365, 10/6 560/379 (register spills beyond 6/6) (term-by-term: 880/552)
    {"c1 fp tuples 4/4", 1, residue_kernel<Mont64, 1, 1, 4, 4, true>, nullptr},
    {"c1 fp tuples 6/6", 1, residue_kernel<Mont64, 1, 1, 6, 6, true>, nullptr},
    // Mont64 K-term steps with lazy tables (class 2, sum-aligned congruences); also selectable for class 1
    {"c2 int tuples 4/4", 2, residue_kernel<Mont64, 2, 0, 4, 4, true>, nullptr},   // 18
    {"c2 int tuples 6/6", 2, residue_kernel<Mont64, 2, 0, 6, 6, true>, nullptr},
    {"c2 int tuples 8/8", 2, residue_kernel<Mont64, 2, 0, 8, 8, true>, nullptr},   // 20 (class-2 default)
    {"c2 int tuples 8/6", 2, residue_kernel<Mont64, 2, 0, 8, 6, true>, nullptr},
    {"c1 int tuples 4/4", 1, residue_kernel<Mont64, 2, 0, 4, 4, true>, nullptr},

};
static const int NVAR = sizeof kVariants / sizeof kVariants[0];
static_assert(NVAR <= 32, "DevCtx::occ holds 32 variants");
// measured best (scripts/variant_sweep.py; class 2: scripts/class2_timing.py, first primes above 2^44, W+V:
// s1/1 2.48e11, tuples 4/4 4.72e11, 6/6 6.10e11, 8/6 6.65e11, 8/8 7.09e11 terms/s)
static const int kDefaultVariant[3] = {15, 17, 20};
static int g_variant[3] = {15, 17, 20};             // per class
static const int kChunkFallback0 = 13;             // class-0 chunk variant when lane mode is unusable
static void read_variant_env() {
    static bool done = false;
    if (done) return;
    done = true;
    const char *names[3] = {"WV_VARIANT0", "WV_VARIANT1", "WV_VARIANT2"};
    for (int c = 0; c < 3; c++) {
        const char *e = getenv(names[c]);
        if (!e) continue;
        int v = atoi(e);
        if (v >= 0 && v < NVAR && kVariants[v].cls == c) g_variant[c] = v;
    }
}

// ------------------------------------------------------------------ device context
struct DevCtx {
    bool ready = false;
    int sms = 0;
    int occ[32] = {};            // residue-kernel blocks per SM per kernel variant
    int occ_census = 1;          // census walk blocks per SM
    uint32_t *d_base0 = nullptr;   // odd primes < 65536
    uint32_t nbase0 = 0;
    cudaStream_t stream = nullptr; // internal stream for the host-buffer API
};
static DevCtx g_ctx[64];
static std::mutex g_mu;

static int ctx_get(DevCtx **out) {
    int dev = -1;
    CK(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return set_err(WV_ECUDA, "device index %d out of range", dev);
    DevCtx &c = g_ctx[dev];
    std::lock_guard<std::mutex> lk(g_mu);
    if (!c.ready) {
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, dev));
        if (prop.major != 10)
            return set_err(WV_ECUDA, "libwv.so is built for sm_100a; device %d is sm_%d%d", dev, prop.major, prop.minor);
        c.sms = prop.multiProcessorCount;
        {
            const Table &T = table();
            if (T.hdr.size() > (size_t)NCONG_MAX) return set_err(WV_ECUDA, "too many congruences");
            const int nc = (int)T.hdr.size();
            CK(cudaMemcpyToSymbol(c_cong, T.hdr.data(), T.hdr.size() * sizeof(Cong)));
            CK(cudaMemcpyToSymbol(c_ncong, &nc, sizeof nc));
            // device copy: each congruence's sums sorted by left endpoint, bit 0 of pad set where the next
            // interval starts where this one ends (x_{j+1} = y_j): consecutive integers, one run (wv_lane.cuh)
            std::vector<Term> dev = T.terms;
            for (const Cong &c : T.hdr) {
                Term *b = dev.data() + c.off, *e = b + c.m;
                std::sort(b, e, [](const Term &u, const Term &v) {
                    return (unsigned __int128)u.xn * v.xd < (unsigned __int128)v.xn * u.xd;
                });
                for (Term *t = b; t < e; t++)
                    t->pad = (t + 1 < e && (unsigned __int128)t->yn * t[1].xd == (unsigned __int128)t[1].xn * t->yd) ? 1u : 0u;
            }
            Term *dt = nullptr;
            CK(cudaMalloc(&dt, dev.size() * sizeof(Term)));
            CK(cudaMemcpy(dt, dev.data(), dev.size() * sizeof(Term), cudaMemcpyHostToDevice));
            const Term *dtc = dt;
            CK(cudaMemcpyToSymbol(c_terms, &dtc, sizeof dtc));
            std::vector<double2> rr(dev.size());              // reciprocals of the endpoint denominators
            for (size_t i = 0; i < rr.size(); i++) rr[i] = make_double2(1.0 / dev[i].xd, 1.0 / dev[i].yd);
            double2 *dr = nullptr;
            CK(cudaMalloc(&dr, rr.size() * sizeof(double2)));
            CK(cudaMemcpy(dr, rr.data(), rr.size() * sizeof(double2), cudaMemcpyHostToDevice));
            const double2 *drc = dr;
            CK(cudaMemcpyToSymbol(c_termr, &drc, sizeof drc));

        }
        for (int v = 0; v < NVAR; v++) {
            if (kVariants[v].fn)
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ[v], kVariants[v].fn, RES_THREADS, 0));
            else
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ[v], kVariants[v].lane, RES_THREADS, 0));
            if (c.occ[v] < 1) c.occ[v] = 1;
        }
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ_census, census_walk_kernel, CEN_THREADS, 0));
        if (c.occ_census < 1) c.occ_census = 1;
        CK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, dev));
        uint64_t thr = UINT64_MAX;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        // level-0 base primes: odd primes in [3, 65536), sieved on the device
        const uint32_t nboot = sizeof h_boot / sizeof h_boot[0];
        uint32_t *d_boot, *d_bitmap;
        uint64_t *d_cnt, *d_off, *d_tiles;
        const uint64_t nseg = BASE0_HI / SIEVE_SPAN;  // segments of [0, 65536)
        const uint64_t nseg1 = nseg > 0 ? nseg : 1;
        CK(cudaMalloc(&d_boot, sizeof h_boot));
        CK(cudaMalloc(&d_bitmap, nseg1 * SIEVE_WORDS * 4));
        CK(cudaMalloc(&d_cnt, nseg1 * 8));
        CK(cudaMalloc(&d_off, (nseg1 + 1) * 8));
        CK(cudaMalloc(&d_tiles, 64));
        CK(cudaMemcpy(d_boot, h_boot, sizeof h_boot, cudaMemcpyHostToDevice));
        SegMap m{0, BASE0_HI, BASE0_HI, 0, 1, BASE0_HI / SIEVE_SPAN, 3, 0};
        cudaStream_t st = c.stream;
        LAUNCH(sieve_segments_kernel, (unsigned)nseg1, SIEVE_THREADS, st, m, d_boot, nboot, nullptr, d_bitmap, d_cnt);
        LAUNCH(scan_tile_totals<uint64_t>, 1, SCAN_THREADS, st, d_cnt, nseg1, d_tiles);
        LAUNCH(scan_tiles_single, 1, SCAN_THREADS, st, d_tiles, (uint64_t)1, d_off + nseg1);
        LAUNCH(scan_tile_apply<uint64_t>, 1, SCAN_THREADS, st, d_cnt, nseg1, d_tiles, d_off);
        uint64_t nb = 0;
        CK(cudaMemcpyAsync(&nb, d_off + nseg1, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        CK(cudaMalloc(&c.d_base0, nb * 4));
        LAUNCH(sieve_write_kernel<uint32_t>, (unsigned)nseg1, SIEVE_THREADS, st, m, d_bitmap, d_off, c.d_base0, nb);
        CK(cudaStreamSynchronize(st));
        c.nbase0 = (uint32_t)nb;
        cudaFree(d_boot); cudaFree(d_bitmap); cudaFree(d_cnt); cudaFree(d_off); cudaFree(d_tiles);
        if (nb != 6541) return set_err(WV_ECUDA, "base-prime sieve produced %llu primes < 65536 (want 6541)",
                                       (unsigned long long)nb);
        c.ready = true;
    }
    *out = &c;
    return WV_OK;
}

// ------------------------------------------------------------------ sizes
static uint64_t isqrt64(uint64_t x) {
    uint64_t r = (uint64_t)sqrtl((long double)x);
    while (r * r > x) r--;
    while ((r + 1) * (r + 1) <= x) r++;
    return r;
}

// upper bound on the primes in an interval of y integers: Montgomery-Vaughan
// pi(x+y) - pi(x) < 2y / log y, and trivially <= y/2 + 1 (odd numbers) + 1.
static uint64_t prime_bound(uint64_t y) {
    if (y == 0) return 0;
    uint64_t triv = y / 2 + 2;
    if (y < 64) return triv;
    uint64_t mv = (uint64_t)(2.0 * (double)y / log((double)y)) + 2;
    return mv < triv ? mv : triv;
}

static uint64_t ntiles(uint64_t n) { return (n + SCAN_TILE - 1) / SCAN_TILE + 1; }
static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

static const uint64_t PART_BUDGET = 1ull << 24;   // partial pairs per batch (256 MiB)
static const uint64_t PART_BUDGET_MIN = 1ull << 18;   // smallest WV_PART_BUDGET (tests: many batches)
// partial pairs per batch for this call: PART_BUDGET, or the WV_PART_BUDGET knob (tests of the batching)
static uint64_t part_budget() {
    const char *e = getenv("WV_PART_BUDGET");
    uint64_t b = e ? strtoull(e, nullptr, 0) : PART_BUDGET;
    return b < PART_BUDGET_MIN ? PART_BUDGET_MIN : (b > PART_BUDGET ? PART_BUDGET : b);
}

enum { M_NPRIMES = 0, M_ERR = 1, M_FIRST64 = 2 /* 2 slots: first k with p >= 2^30, >= 2^44 */,
       M_CNT = 4 /* 3 slots: work counters per class */, M_NHITS = 7, M_CHECKSUM = 8, M_NBASE1 = 9,
       M_SPLIT = 10 /* 4 slots */, M_TERMS = 14 /* 3 slots: terms per class */, M_LANE_T = 17,
       M_LANE_TERMS = 18 /* terms executed by the lane-mode v2 kernel (counted there) */,
       M_LANE_SLICED = 19 /* 2 slots: lane group-tests with Q > 1, all lane group-tests */, M_SLOTS = 24 };

struct Layout {
    // problem
    uint64_t lo, hi, block;
    uint32_t mode, shard, nshards, ntests;
    SegMap map, map1;
    uint64_t nseg, nseg1, nbase1_cap;
    bool need_l1;
    uint64_t prime_cap, K;
    // offsets into the workspace
    size_t o_misc, o_bitmap, o_segcnt, o_segoff, o_tiles, o_base1, o_recs, o_nch, o_start, o_part,
           o_flags, o_pos, o_kb, o_gq, o_gstart, total;
    uint64_t ngt;           // lane-mode group-tests: ceil(prime_cap / 32) * ntests
    uint64_t tiles_n;
    uint32_t segstride;     // coarse seg-chunk index entries per record (0: none)
    size_t o_segidx;
};

static void layout_tail(Layout &L) {
    size_t o = L.total;
    L.o_recs = o;  o += al(L.K * sizeof(Rec));
    L.o_nch = o;   o += al(L.K * 8);
    L.o_start = o; o += al((L.K + 1) * 8);
    L.o_part = o;  o += al(PART_BUDGET * sizeof(ulonglong2));
    L.o_kb = o;    o += al(3 * (L.K * CAP_CHUNKS / (PART_BUDGET_MIN / 2) + 4) * 8);
    L.ngt = (L.prime_cap + 31) / 32 * L.ntests;
    L.o_gq = o;     o += al((L.ngt + 1) * 8);
    L.o_gstart = o; o += al((L.ngt + 1) * 8);
    uint64_t t = ntiles(L.K + 1);
    if (ntiles(L.prime_cap) > t) t = ntiles(L.prime_cap);
    if (ntiles(L.ngt + 1) > t) t = ntiles(L.ngt + 1);
    if (L.tiles_n < t) L.tiles_n = t;
    L.o_tiles = o; o += al(L.tiles_n * 8);
    L.o_segidx = o; o += al(L.K * L.segstride * 4);   // last: a stride-0 layout is a prefix of this one
    L.total = o;
}

// Entries of the coarse seg-chunk index per record: max ceil(m / 32) over the sum-aligned (seg)
// congruences the current schedule (tiers + overrides) can pick for primes below hi.
static uint32_t seg_stride(uint64_t hi) {
    const Table &T = table();
    uint32_t s = 0;
    auto consider = [&](int id) {
        if (id >= 0 && id < (int)T.hdr.size() && T.hdr[id].seg) {
            const uint32_t r = (T.hdr[id].m + 31) / 32;
            if (r > s) s = r;
        }
    };
    for (int t = 0; t < 2; t++) {
        const int force = t == 0 ? g_sched.w_force : g_sched.v_force;
        if (force >= 0) { consider(force); continue; }
        for (int i = 0; i < g_sched.n[t]; i++)
            if (i == 0 || g_sched.th[t][i] < hi) consider(g_sched.id[t][i]);
    }
    return s;
}

static int make_layout(uint64_t lo, uint64_t hi, uint32_t mode, uint32_t shard, uint32_t nshards, uint64_t block,
                       Layout &L, bool records = true) {
    if (hi <= lo) return set_err(WV_EINVAL, "empty or inverted range [%llu, %llu)", (unsigned long long)lo,
                                 (unsigned long long)hi);
    if (hi > WV_HI_MAX) return set_err(WV_EINVAL, "hi > 2^62");
    if (mode < 1 || mode > 3) return set_err(WV_EINVAL, "mode %u not in {1,2,3}", mode);
    if (nshards == 0 || shard >= nshards) return set_err(WV_EINVAL, "shard %u of %u", shard, nshards);
    const uint64_t width = hi - lo;
    if (block == 0) {
        if (nshards == 1) {
            block = (width + SIEVE_SPAN - 1) / SIEVE_SPAN * SIEVE_SPAN;
        } else {
            uint64_t t = width / (32ull * nshards);
            block = SIEVE_SPAN;
            while (block * 2 <= t) block *= 2;
        }
    }
    if (block % SIEVE_SPAN != 0) return set_err(WV_EINVAL, "block %llu is not a multiple of %d",
                                                (unsigned long long)block, SIEVE_SPAN);
    memset(&L, 0, sizeof L);
    L.lo = lo; L.hi = hi; L.block = block; L.mode = mode; L.shard = shard; L.nshards = nshards;
    L.ntests = mode == 3 ? 2 : 1;
    const uint64_t nblocks = (width + block - 1) / block;
    // blocks j of this shard: shard_block(j, shard, nshards) - pad (rounds of nshards, snake order,
    // aligned to the top of the window; virtual blocks below 0 are empty)
    const uint64_t pad = shard_pad(nblocks, nshards);
    const uint64_t my_blocks = (nblocks + pad) / nshards;
    const uint64_t spb = block / SIEVE_SPAN;
    L.map = SegMap{lo, hi, block, shard, nshards, spb, 5, pad};
    L.nseg = my_blocks * spb;
    // primes in this shard: sum of per-block bounds
    uint64_t cap = 0;
    for (uint64_t j = 0; j < my_blocks; j++) {
        const uint64_t vb = shard_block(j, shard, nshards);
        if (vb < pad) continue;
        uint64_t bs = lo + (vb - pad) * block;
        uint64_t be = bs + block < hi ? bs + block : hi;
        cap += prime_bound(be - bs);
    }
    L.prime_cap = cap;
    if (records && cap >= (1ull << 32))   // record indices are 32-bit: split such windows into blocks / sweeps
        return set_err(WV_EINVAL, "window holds up to %llu primes (> 2^32): use smaller windows or wv_search_shard",
                       (unsigned long long)cap);
    L.K = cap * L.ntests;
    // base primes: q <= isqrt(hi - 1)
    const uint64_t r = isqrt64(hi - 1);
    L.need_l1 = r >= BASE0_HI;
    if (L.need_l1) {
        const uint64_t hi1 = r + 1;
        const uint64_t blk1 = (hi1 + SIEVE_SPAN - 1) / SIEVE_SPAN * SIEVE_SPAN;
        L.map1 = SegMap{0, hi1, blk1, 0, 1, blk1 / SIEVE_SPAN, 3, 0};
        L.nseg1 = blk1 / SIEVE_SPAN;
        L.nbase1_cap = prime_bound(hi1);
    }
    size_t o = 0;
    L.o_misc = o;   o += al(M_SLOTS * 8);
    const uint64_t nsegmax = L.nseg > L.nseg1 ? L.nseg : L.nseg1;
    L.o_bitmap = o; o += al(nsegmax * SIEVE_WORDS * 4);
    L.o_segcnt = o; o += al(nsegmax * 8);
    L.o_segoff = o; o += al((nsegmax + 1) * 8);
    L.o_base1 = o;  o += al(L.nbase1_cap * 4);
    L.o_flags = o;  o += al(L.prime_cap * 4);
    L.o_pos = o;    o += al((L.prime_cap + 1) * 8);
    L.tiles_n = ntiles(nsegmax + 1);
    L.total = o;
    L.segstride = records ? seg_stride(hi) : 0;
    layout_tail(L);
    return WV_OK;
}

// ------------------------------------------------------------------ lane-mode chain knob
// WV_LANE_CHAIN (benchmarking / tests: chain mode per exponent, default 5) lives in __constant__ memory of
// each device; it is rewritten only when the environment value changes, under a lock, stream-ordered
// before the launch (a value change waits for the stream, so no kernel still running can see it change).
static std::mutex g_knob_mu;
static int lane_chain_knob(cudaStream_t st) {
    static uint32_t cur[64];
    static bool init[64];
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return WV_OK;
    const char *ev = getenv("WV_LANE_CHAIN");
    const uint32_t cm = ev ? (uint32_t)strtoul(ev, nullptr, 0) : 5u;
    std::lock_guard<std::mutex> lk(g_knob_mu);
    if (!init[dev] || cur[dev] != cm) {
        CK(cudaDeviceSynchronize());              // no kernel of another stream may be reading the old value
        CK(cudaMemcpyToSymbolAsync(c_lane_chain, &cm, sizeof cm, 0, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
        cur[dev] = cm;
        init[dev] = true;
    }
    return WV_OK;
}

// ------------------------------------------------------------------ launch helpers
template <typename T>
static int scan_excl(const T *in, uint64_t n, uint64_t *out, uint64_t *total, uint64_t *tiles, cudaStream_t st) {
    const uint64_t nt = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (nt == 0) {
        CK(cudaMemsetAsync(total, 0, 8, st));
        return WV_OK;
    }
    LAUNCH(scan_tile_totals<T>, (unsigned)nt, SCAN_THREADS, st, in, n, tiles);
    LAUNCH(scan_tiles_single, 1, SCAN_THREADS, st, tiles, nt, total);
    LAUNCH(scan_tile_apply<T>, (unsigned)nt, SCAN_THREADS, st, in, n, tiles, out);
    return WV_OK;
}

static char *WS(void *ws, size_t off) { return (char *)ws + off; }

// sieve [map] with a base list -> out (T), count at *d_count
template <typename T>
static int run_sieve(const SegMap &map, uint64_t nseg, const uint32_t *base, uint32_t nbase_host,
                     const uint64_t *nbase_dev, T *out, uint64_t cap, uint64_t *d_count, void *ws,
                     const Layout &L, cudaStream_t st) {
    if (nseg == 0) {
        CK(cudaMemsetAsync(d_count, 0, 8, st));
        return WV_OK;
    }
    uint32_t *bitmap = (uint32_t *)WS(ws, L.o_bitmap);
    uint64_t *segcnt = (uint64_t *)WS(ws, L.o_segcnt);
    uint64_t *segoff = (uint64_t *)WS(ws, L.o_segoff);
    uint64_t *tiles = (uint64_t *)WS(ws, L.o_tiles);
    LAUNCH(sieve_segments_kernel, (unsigned)nseg, SIEVE_THREADS, st, map, base, nbase_host, nbase_dev, bitmap, segcnt);
    TRY(scan_excl<uint64_t>(segcnt, nseg, segoff, d_count, tiles, st));
    LAUNCH(sieve_write_kernel<T>, (unsigned)nseg, SIEVE_THREADS, st, map, bitmap, segoff, out, cap);
    return WV_OK;
}

// base list for the main sieve: level 0 (< 65536) or level 1 (<= isqrt(hi-1))
static int base_list(DevCtx *c, const Layout &L, void *ws, cudaStream_t st, const uint32_t **base,
                     uint32_t *nbase_host, const uint64_t **nbase_dev) {
    uint64_t *misc = (uint64_t *)WS(ws, L.o_misc);
    if (!L.need_l1) {
        *base = c->d_base0; *nbase_host = c->nbase0; *nbase_dev = nullptr;
        return WV_OK;
    }
    uint32_t *b1 = (uint32_t *)WS(ws, L.o_base1);
    TRY(run_sieve<uint32_t>(L.map1, L.nseg1, c->d_base0, c->nbase0, nullptr, b1, L.nbase1_cap, misc + M_NBASE1, ws,
                            L, st));
    *base = b1; *nbase_host = 0; *nbase_dev = misc + M_NBASE1;
    return WV_OK;
}

// plan + scan + residue + finalize for records [0, K) of the primes list.
// n_dev (device count) or n_host gives the number of valid primes.
// plan + scan + residue + finalize.  async_ok: the caller does not need the prime count on the host; then,
// for a window of class-0 primes only (lane mode, default schedule, no stats, the partial-pair bound fits
// one batch) nothing waits for the device: item counts and the sliced-code choice are read on the device.
static int run_residues(DevCtx *c, const uint64_t *primes, const uint64_t *n_dev, uint64_t n_host, uint64_t K,
                        uint32_t mode, bool sorted, uint64_t *res_w, uint64_t *res_v, void *ws, const Layout &L,
                        cudaStream_t st, uint64_t *n_primes_out, bool async_ok = false) {
    NvtxRange range("a2-a5 plan, residues, finalize");
    uint64_t *misc = (uint64_t *)WS(ws, L.o_misc);
    Rec *recs = (Rec *)WS(ws, L.o_recs);
    uint64_t *nch = (uint64_t *)WS(ws, L.o_nch);
    uint64_t *start = (uint64_t *)WS(ws, L.o_start);
    ulonglong2 *part = (ulonglong2 *)WS(ws, L.o_part);
    uint64_t *kb = (uint64_t *)WS(ws, L.o_kb);
    uint64_t *tiles = (uint64_t *)WS(ws, L.o_tiles);
    uint64_t *gq = (uint64_t *)WS(ws, L.o_gq);
    uint64_t *gstart = (uint64_t *)WS(ws, L.o_gstart);
    uint32_t *segidx = L.segstride ? (uint32_t *)WS(ws, L.o_segidx) : nullptr;
    read_variant_env();
    int var0 = g_variant[0];
    bool lane = sorted && kVariants[var0].lane != nullptr;
    if (!lane && kVariants[var0].lane) var0 = kChunkFallback0;
    const unsigned grid_plan = (unsigned)((K + 255) / 256 < (uint64_t)c->sms * 32 ? (K + 255) / 256 : c->sms * 32);
    // lane-mode slices per group: the v1 kernel cuts 8192-term slices; v2 keeps whole sums unless the
    // window has too few groups to fill the GPU (WV_LANE_ITEMS items per resident warp wanted)
    const bool lane2 = lane && kVariants[var0].lane == residue_lane2_kernel;
    double lane_items = 0;
    if (lane2) {
        const char *ev = getenv("WV_LANE_ITEMS");
        lane_items = (ev ? atof(ev) : 2.0) * (double)c->sms * c->occ[var0] * (RES_THREADS / 32);
    }
    uint64_t h[4] = {0, 0, 0, 0};   // n, err, G, G_lane
    uint64_t hs[4], ht[3];
    if (K > 0) {
        (void)table();
        LAUNCH(plan_kernel, grid_plan ? grid_plan : 1, 256, st, primes, n_dev, n_host, K, mode, g_sched, recs,
               nch, (unsigned long long *)(misc + M_FIRST64), (int *)(misc + M_ERR),
               (unsigned long long *)(misc + M_TERMS), lane ? gq : nullptr, segidx, L.segstride, LANE_SLICE,
               LANE_QMAX, (lane && lane2) ? (unsigned long long *)(misc + M_LANE_T) : nullptr);
        if (lane && lane2 && L.ngt > 0) {
            const uint64_t nbw = (L.ngt * 32 + 255) / 256;
            LAUNCH(lane_group_terms_kernel, (unsigned)(nbw < (uint64_t)c->sms * 16 ? nbw : c->sms * 16), 256, st,
                   primes, n_dev, n_host, mode, g_sched, L.ngt, gq, (unsigned long long *)(misc + M_LANE_T));
            const uint64_t nb = (L.ngt * 32 + 255) / 256;                 // a warp per group-test
            LAUNCH(lane_slices_kernel, (unsigned)(nb < (uint64_t)c->sms * 16 ? nb : c->sms * 16), 256, st, gq, L.ngt,
                   L.ntests, recs, K, nch, (const unsigned long long *)(misc + M_LANE_T), lane_items, 4096ull,
                   LANE_QMAX, (unsigned long long *)(misc + M_LANE_SLICED));
        }
    }
    TRY(scan_excl<uint64_t>(nch, K, start, start + K, tiles, st));
    if (lane) TRY(scan_excl<uint64_t>(gq, L.ngt, gstart, gstart + L.ngt, tiles, st));
    const bool stats = g_stats_on.load() != 0;
    const uint64_t budget = part_budget();
    // most lane groups sliced: every lane item runs the sliced chain code (WV_LANE_ALLSL=0/1 forces it;
    // otherwise the kernel decides from the slice counts on the device)
    const char *eas = getenv("WV_LANE_ALLSL");
    const uint32_t allsl_mode = eas ? (atoi(eas) ? 1u : 0u) : 2u;
    // partial slots of a lane-only window: 32 per group-test slice, sum_gt Q <= items wanted + ngt
    const double gbound = 32.0 * ((double)lane_items + (double)L.ngt);
    if (async_ok && sorted && lane && lane2 && !stats && L.hi <= WIDTH32_MAX && g_sched.w_force < 0 &&
        g_sched.v_force < 0 && gbound <= (double)budget && K > 0) {
        TRY(lane_chain_knob(st));
        CK(cudaMemsetAsync(misc + M_LANE_TERMS, 0, 8, st));
        CK(cudaMemsetAsync(misc + M_CNT, 0, 8, st));
        LAUNCH(kVariants[var0].lane, c->sms * c->occ[var0], RES_THREADS, st, recs, start, gstart, gq, L.ngt, 0ull,
               0ull, gstart + L.ngt, L.ntests, K, 0ull, part, (unsigned long long *)(misc + M_CNT),
               (unsigned long long *)(misc + M_LANE_TERMS), allsl_mode,
               (const unsigned long long *)(misc + M_LANE_SLICED));
        uint64_t fb = (K + 255) / 256;
        if (fb > (uint64_t)c->sms * 16) fb = (uint64_t)c->sms * 16;
        LAUNCH(finalize_kernel, (unsigned)fb, 256, st, recs, start, 0ull, K, 0ull, part, res_w, res_v);
        return WV_OK;
    }
    LAUNCH(split_kernel, 1, 32, st, start, K, (const unsigned long long *)(misc + M_FIRST64), misc + M_SPLIT);
    CK(cudaMemcpyAsync(ht, misc + M_TERMS, 24, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&h[0], misc + M_NPRIMES, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&h[2], start + K, 8, cudaMemcpyDeviceToHost, st));
    if (lane) CK(cudaMemcpyAsync(&h[3], gstart + L.ngt, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hs, misc + M_SPLIT, 32, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const uint64_t n = n_dev ? h[0] : n_host;
    if (n_primes_out) *n_primes_out = n;
    if ((int)h[1] != 0) return set_err(WV_EINVAL, "schedule chose a congruence not valid for some prime");
    const uint64_t G = h[2];
    std::vector<EvPair> evs;
    if (stats) {
        std::lock_guard<std::mutex> lk(g_stats_mu);
        g_stats.terms += ht[0] + ht[1] + ht[2];
        g_stats.terms32 += ht[0];
        g_stats.terms_fp += ht[1];
        g_stats.records += K;
        g_stats.chunks += G;
    }
    // class boundaries (sorted input): items [0,gb[1]) class 0, [gb[1],gb[2]) class 1, [gb[2],G) class 2
    const uint64_t gb[4] = {0, sorted ? hs[0] : 0, sorted ? hs[2] : 0, G};
    const uint64_t kbd[4] = {0, sorted ? hs[1] : 0, sorted ? hs[3] : 0, K};
    // batches of <= budget partial pairs, cut at record boundaries (lane mode: at group boundaries, so each
    // batch is whole lane items [hi_[b], hi_[b + 1]))
    std::vector<uint64_t> hk, hg, hi_;
    if (G <= budget) {
        hk = {0, K};
        hg = {0, G};
        hi_ = {0, h[3]};
    } else {
        // every record has <= CAP_CHUNKS chunks and every lane group <= 32 ntests LANE_QMAX slots, both << step
        const uint64_t step = budget / 2;
        const uint64_t nb = (G + step - 1) / step;
        LAUNCH(batch_bounds_kernel, (unsigned)((nb + 256) / 256), 256, st, start, K, step, nb, kb,
               lane ? 32ull * L.ntests : 1ull, lane ? gstart : nullptr, L.ntests);
        hk.resize(3 * (nb + 1));
        CK(cudaMemcpyAsync(hk.data(), kb, (lane ? 3 : 2) * (nb + 1) * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        hg.assign(hk.begin() + (nb + 1), hk.begin() + 2 * (nb + 1));   // partial-slot bounds start[kb[b]]
        if (lane) hi_.assign(hk.begin() + 2 * (nb + 1), hk.end());    // lane-item bounds
        hk.resize(nb + 1);
    }
    if (lane) CK(cudaMemsetAsync(misc + M_LANE_TERMS, 0, 8, st));   // the lane kernels' term counts, all batches
    for (size_t b = 0; b + 1 < hk.size(); b++) {
        const uint64_t klo = hk[b], khi = hk[b + 1], glo = hg[b], ghi = hg[b + 1];
        if (khi <= klo) continue;
        // 32-bit records: items [glo, min(ghi, g32)); 64-bit: [max(glo, g32), ghi)
        // per class: items [max(glo, gb[c]), min(ghi, gb[c+1])) of records [max(klo,kbd[c]), min(khi,kbd[c+1]));
        // unsorted input: every class kernel scans the whole batch and skips the other classes' records
        const uint64_t ia = lane ? hi_[b] : 0, ib = lane ? hi_[b + 1] : 0;
        if (lane && ib > ia) {     // lane mode for class 0: this batch's lane items
            TRY(lane_chain_knob(st));
            CK(cudaMemsetAsync(misc + M_CNT, 0, 8, st));
            EvPair ev{nullptr, nullptr, 0};
            if (stats) { CK(cudaEventCreate(&ev.a)); CK(cudaEventCreate(&ev.b)); CK(cudaEventRecord(ev.a, st)); }
            LAUNCH(kVariants[var0].lane, c->sms * c->occ[var0], RES_THREADS, st, recs, start, gstart, gq, L.ngt, ia,
                   ib - ia, (const uint64_t *)nullptr, L.ntests, K, glo, part, (unsigned long long *)(misc + M_CNT),
                   lane2 ? (unsigned long long *)(misc + M_LANE_TERMS) : nullptr, lane2 ? allsl_mode : 0u,
                   (const unsigned long long *)(misc + M_LANE_SLICED));
            if (stats) { CK(cudaEventRecord(ev.b, st)); evs.push_back(ev); }
        }
        for (int cls = 0; cls < 3; cls++) {
            if (cls == 0 && lane) continue;
            uint64_t a_ = glo, b_ = ghi, ka = klo, kz = khi;
            if (sorted) {
                a_ = glo > gb[cls] ? glo : gb[cls];
                b_ = ghi < gb[cls + 1] ? ghi : gb[cls + 1];
                ka = klo > kbd[cls] ? klo : kbd[cls];
                kz = khi < kbd[cls + 1] ? khi : kbd[cls + 1];
            }
            if (b_ <= a_ || kz <= ka) continue;
            CK(cudaMemsetAsync(misc + M_CNT + cls, 0, 8, st));
            EvPair ev{nullptr, nullptr, cls};
            if (stats) { CK(cudaEventCreate(&ev.a)); CK(cudaEventCreate(&ev.b)); CK(cudaEventRecord(ev.a, st)); }
            unsigned long long *cnt = (unsigned long long *)(misc + M_CNT + cls);
            const int var = cls == 0 ? var0 : g_variant[cls];
            const unsigned grid = c->sms * c->occ[var];
            LAUNCH(kVariants[var].fn, grid, RES_THREADS, st, recs, start, ka, kz, a_, b_, glo, part, cnt, 1u << cls,
                   segidx, L.segstride);
            if (stats) { CK(cudaEventRecord(ev.b, st)); evs.push_back(ev); }
        }
        const uint64_t nrec = khi - klo;
        uint64_t fb = (nrec + 255) / 256;
        if (fb > (uint64_t)c->sms * 16) fb = (uint64_t)c->sms * 16;
        LAUNCH(finalize_kernel, (unsigned)fb, 256, st, recs, start, klo, khi, glo, part, res_w, res_v);
    }
    if (stats && !evs.empty()) {
        uint64_t lane_terms = 0;
        if (lane && lane2) CK(cudaMemcpyAsync(&lane_terms, misc + M_LANE_TERMS, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (lane_terms) {
            std::lock_guard<std::mutex> lk(g_stats_mu);
            g_stats.terms += lane_terms;
            g_stats.terms32 += lane_terms;
        }
        double ms = 0, ms32 = 0, msfp = 0;
        for (auto &e : evs) {
            float t = 0;
            CK(cudaEventElapsedTime(&t, e.a, e.b));
            ms += t;
            if (e.cls == 0) ms32 += t;
            if (e.cls == 1) msfp += t;
            cudaEventDestroy(e.a);
            cudaEventDestroy(e.b);
        }
        std::lock_guard<std::mutex> lk(g_stats_mu);
        g_stats.residue_ms += ms;
        g_stats.residue32_ms += ms32;
        g_stats.residue_fp_ms += msfp;
        g_stats.residue_launches += evs.size();
    }
    return WV_OK;
}

// ------------------------------------------------------------------ device API
extern "C" int wv_device_workspace_bytes(uint64_t lo, uint64_t hi, uint32_t mode, uint32_t shard, uint32_t nshards,
                                         uint64_t block, size_t *workspace_bytes, size_t *prime_cap) {
    Layout L;
    TRY(make_layout(lo, hi, mode, shard, nshards, block, L));
    if (workspace_bytes) *workspace_bytes = L.total;
    if (prime_cap) *prime_cap = L.prime_cap;
    return WV_OK;
}

static int search_device_impl(const Layout &L, uint64_t *d_primes, uint64_t *d_res_w, uint64_t *d_res_v,
                              wv_hit *d_hits, uint64_t *d_checksum, void *ws, cudaStream_t st, size_t *n_primes,
                              size_t *n_hits) {
    NvtxRange range("wv_search_device");
    DevCtx *c;
    TRY(ctx_get(&c));
    uint64_t *misc = (uint64_t *)WS(ws, L.o_misc);
    CK(cudaMemsetAsync(misc, 0, M_SLOTS * 8, st));
    CK(cudaMemsetAsync(misc + M_FIRST64, 0xff, 16, st));
    const uint32_t *base;
    uint32_t nbh;
    const uint64_t *nbd;
    {
        NvtxRange r1("a1 sieve");
        TRY(base_list(c, L, ws, st, &base, &nbh, &nbd));
        TRY(run_sieve<uint64_t>(L.map, L.nseg, base, nbh, nbd, d_primes, L.prime_cap, misc + M_NPRIMES, ws, L, st));
    }
    uint64_t n = 0;
    const bool async_ok = !n_primes && !n_hits;        // no count wanted on the host
    TRY(run_residues(c, d_primes, misc + M_NPRIMES, 0, L.K, L.mode, true, d_res_w, d_res_v, ws, L, st,
                     async_ok ? nullptr : &n, async_ok));
    NvtxRange r6("a6 flags, hits, checksum");
    if (!async_ok && n > L.prime_cap)   // cannot happen: prime_cap is the Montgomery-Vaughan bound (sieve writes <= cap)
        return set_err(WV_ENOSPC, "prime count %llu exceeds bound %llu", (unsigned long long)n,
                       (unsigned long long)L.prime_cap);
    // residues not requested -> WV_RES_NONE; hit flags; checksum
    uint32_t *flags = (uint32_t *)WS(ws, L.o_flags);
    uint64_t *pos = (uint64_t *)WS(ws, L.o_pos);
    uint64_t *tiles = (uint64_t *)WS(ws, L.o_tiles);
    const uint64_t kmax = L.prime_cap;
    if (kmax > 0) {
        unsigned g = (unsigned)((kmax + 255) / 256 < (uint64_t)c->sms * 16 ? (kmax + 255) / 256 : c->sms * 16);
        LAUNCH(flags_kernel, g, 256, st, d_primes, misc + M_NPRIMES, 0, kmax, d_res_w, d_res_v, L.mode, flags,
               (unsigned long long *)(misc + M_CHECKSUM));
        TRY(scan_excl<uint32_t>(flags, kmax, pos, misc + M_NHITS, tiles, st));
        if (d_hits)
            LAUNCH(hits_scatter_kernel, g, 256, st, d_primes, misc + M_NPRIMES, kmax, d_res_w, d_res_v, flags, pos,
                   (HitOut *)d_hits);
    }
    if (d_checksum) CK(cudaMemcpyAsync(d_checksum, misc + M_CHECKSUM, 8, cudaMemcpyDeviceToDevice, st));
    if (n_primes) *n_primes = n;
    if (n_hits) {                      // the hit count is wanted on the host: wait for it
        uint64_t nh = 0;
        CK(cudaMemcpyAsync(&nh, misc + M_NHITS, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        *n_hits = nh;
    }
    return WV_OK;
}

extern "C" int wv_search_device(uint64_t lo, uint64_t hi, uint32_t mode, uint32_t shard, uint32_t nshards,
                                uint64_t block, uint64_t *d_primes, uint64_t *d_res_w, uint64_t *d_res_v,
                                wv_hit *d_hits, uint64_t *d_checksum, size_t prime_cap, void *d_workspace,
                                size_t workspace_bytes, void *stream, size_t *n_primes, size_t *n_hits) {
    Layout L;
    TRY(make_layout(lo, hi, mode, shard, nshards, block, L));
    if (!d_primes || !d_res_w || !d_res_v) return set_err(WV_EINVAL, "null output pointer");
    if (prime_cap < L.prime_cap) {
        if (n_primes) *n_primes = L.prime_cap;
        return set_err(WV_ENOSPC, "prime_cap %zu < required %llu", prime_cap, (unsigned long long)L.prime_cap);
    }
    cudaStream_t st = (cudaStream_t)stream;
    void *ws = d_workspace;
    if (ws && workspace_bytes < L.total)
        return set_err(WV_ENOSPC, "workspace %zu < required %zu bytes", workspace_bytes, L.total);
    if (!ws) CK(cudaMallocAsync(&ws, L.total, st));
    int rc = search_device_impl(L, d_primes, d_res_w, d_res_v, d_hits, d_checksum, ws, st, n_primes, n_hits);
    if (!d_workspace) {
        cudaFreeAsync(ws, st);
        cudaStreamSynchronize(st);
    }
    return rc;
}

// residues-only layout; the coarse seg index is sized for primes <= max_p
static void residues_layout(size_t n, uint64_t max_p, uint32_t mode, Layout &L) {
    memset(&L, 0, sizeof L);
    L.mode = mode;
    L.ntests = mode == 3 ? 2 : 1;
    L.prime_cap = n;
    L.K = (uint64_t)n * L.ntests;
    L.hi = max_p < WV_HI_MAX ? max_p + 1 : WV_HI_MAX;
    L.o_misc = 0;
    L.total = al(M_SLOTS * 8);
    L.tiles_n = 1;
    L.segstride = seg_stride(L.hi);
    layout_tail(L);
}

extern "C" int wv_residues_workspace_bytes(size_t n, uint64_t max_p, uint32_t mode, size_t *workspace_bytes) {
    if (mode < 1 || mode > 3) return set_err(WV_EINVAL, "mode %u not in {1,2,3}", mode);
    Layout L;
    residues_layout(n, max_p, mode, L);
    if (workspace_bytes) *workspace_bytes = L.total;
    return WV_OK;
}

extern "C" int wv_residues_device(const uint64_t *d_primes, size_t n, uint32_t mode, uint64_t *d_res_w,
                                  uint64_t *d_res_v, void *d_workspace, size_t workspace_bytes, void *stream) {
    if (mode < 1 || mode > 3) return set_err(WV_EINVAL, "mode %u not in {1,2,3}", mode);
    if (n == 0) return WV_OK;
    if (!d_primes || !d_res_w || !d_res_v) return set_err(WV_EINVAL, "null pointer");
    // the largest coarse seg index that fits the caller's workspace (a smaller layout is a prefix)
    Layout L;
    residues_layout(n, WV_HI_MAX, mode, L);
    if (d_workspace && workspace_bytes < L.total) {
        for (uint64_t mp : {(uint64_t)1 << 40, (uint64_t)1 << 33, (uint64_t)1 << 29, (uint64_t)5}) {
            residues_layout(n, mp, mode, L);
            if (workspace_bytes >= L.total) break;
        }
    }
    cudaStream_t st = (cudaStream_t)stream;
    void *ws = d_workspace;
    if (ws && workspace_bytes < L.total) return set_err(WV_ENOSPC, "workspace %zu < %zu", workspace_bytes, L.total);
    DevCtx *c;
    TRY(ctx_get(&c));
    if (!ws) CK(cudaMallocAsync(&ws, L.total, st));
    uint64_t *misc = (uint64_t *)WS(ws, L.o_misc);
    int rc = WV_OK;
    do {
        if (cudaMemsetAsync(misc, 0, M_SLOTS * 8, st) != cudaSuccess ||
            cudaMemsetAsync(misc + M_FIRST64, 0xff, 16, st) != cudaSuccess) {
            rc = set_err(WV_ECUDA, "memset failed");
            break;
        }
        rc = run_residues(c, d_primes, nullptr, n, L.K, mode, false, d_res_w, d_res_v, ws, L, st, nullptr);
        if (rc != WV_OK) break;
        unsigned g = (unsigned)((n + 255) / 256 < (uint64_t)c->sms * 16 ? (n + 255) / 256 : c->sms * 16);
        flags_kernel<<<g, 256, 0, st>>>(d_primes, nullptr, n, n, d_res_w, d_res_v, mode, nullptr, nullptr);
        g_launches.fetch_add(1);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = set_err(WV_ECUDA, "flags_kernel: %s", cudaGetErrorString(e));
    } while (0);
    if (!d_workspace) cudaFreeAsync(ws, st);
    if (cudaStreamSynchronize(st) != cudaSuccess && rc == WV_OK) rc = set_err(WV_ECUDA, "stream sync failed");
    return rc;
}

extern "C" int wv_sieve_device(uint64_t lo, uint64_t hi, uint64_t *d_primes, size_t cap, size_t *n,
                               void *d_workspace, size_t workspace_bytes, void *stream) {
    Layout L;
    TRY(make_layout(lo, hi, 1, 0, 1, 0, L));
    cudaStream_t st = (cudaStream_t)stream;
    void *ws = d_workspace;
    if (ws && workspace_bytes < L.total) return set_err(WV_ENOSPC, "workspace %zu < %zu", workspace_bytes, L.total);
    DevCtx *c;
    TRY(ctx_get(&c));
    if (!ws) CK(cudaMallocAsync(&ws, L.total, st));
    uint64_t *misc = (uint64_t *)WS(ws, L.o_misc);
    int rc = WV_OK;
    uint64_t cnt = 0;
    do {
        if (cudaMemsetAsync(misc, 0, M_SLOTS * 8, st) != cudaSuccess) { rc = set_err(WV_ECUDA, "memset"); break; }
        const uint32_t *base;
        uint32_t nbh;
        const uint64_t *nbd;
        if ((rc = base_list(c, L, ws, st, &base, &nbh, &nbd)) != WV_OK) break;
        if ((rc = run_sieve<uint64_t>(L.map, L.nseg, base, nbh, nbd, d_primes, cap, misc + M_NPRIMES, ws, L, st)) !=
            WV_OK)
            break;
        if (cudaMemcpyAsync(&cnt, misc + M_NPRIMES, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess) {
            rc = set_err(WV_ECUDA, "copy");
            break;
        }
    } while (0);
    if (!d_workspace) cudaFreeAsync(ws, st);
    if (cudaStreamSynchronize(st) != cudaSuccess && rc == WV_OK) rc = set_err(WV_ECUDA, "sync");
    if (rc != WV_OK) return rc;
    if (n) *n = cnt;
    if (cnt > cap) return set_err(WV_ENOSPC, "cap %zu < %llu primes", cap, (unsigned long long)cnt);
    return WV_OK;
}

extern "C" int wv_near_misses_device(const uint64_t *d_primes, const uint64_t *d_res_w, const uint64_t *d_res_v,
                                     size_t n, uint64_t bound, wv_nearmiss *d_out, size_t cap, size_t *n_out,
                                     uint64_t *d_hist_w, uint64_t *d_hist_v, void *d_workspace, void *stream) {
    static_assert(sizeof(wv_nearmiss) == sizeof(NearOut), "wv_nearmiss layout");
    if (!d_primes || !d_res_w || !d_res_v) return set_err(WV_EINVAL, "null pointer");
    DevCtx *c;
    TRY(ctx_get(&c));
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long *cnt = (unsigned long long *)d_workspace;
    if (!cnt) CK(cudaMallocAsync((void **)&cnt, 8, st));
    int rc = WV_OK;
    unsigned long long h = 0;
    if (cudaMemsetAsync(cnt, 0, 8, st) != cudaSuccess) rc = set_err(WV_ECUDA, "memset");
    if (rc == WV_OK && n > 0) {
        unsigned g = (unsigned)((n + 255) / 256 < (uint64_t)c->sms * 16 ? (n + 255) / 256 : c->sms * 16);
        nearmiss_kernel<<<g, 256, 0, st>>>(d_primes, n, d_res_w, d_res_v, bound, (NearOut *)d_out,
                                           d_out ? cap : 0, cnt, (unsigned long long *)d_hist_w,
                                           (unsigned long long *)d_hist_v);
        g_launches.fetch_add(1);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = set_err(WV_ECUDA, "nearmiss_kernel: %s", cudaGetErrorString(e));
    }
    if (rc == WV_OK && cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        rc = set_err(WV_ECUDA, "copy");
    if (!d_workspace) cudaFreeAsync(cnt, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess && rc == WV_OK) rc = set_err(WV_ECUDA, "near misses: %s", cudaGetErrorString(e));
    if (rc != WV_OK) return rc;
    if (n_out) *n_out = h;
    if (h > cap) return set_err(WV_ENOSPC, "near-miss cap %zu < %llu", cap, (unsigned long long)h);
    return WV_OK;
}

extern "C" int wv_prime_count(uint64_t lo, uint64_t hi, uint64_t *count) {
    Layout L;
    TRY(make_layout(lo, hi, 1, 0, 1, 0, L, false));
    DevCtx *c;
    TRY(ctx_get(&c));
    cudaStream_t st = c->stream;
    // compact workspace: misc, level-1 bitmap only, counts, offsets, base list, tiles
    const uint64_t nsegmax = L.nseg > L.nseg1 ? L.nseg : L.nseg1;
    {
        size_t o = 0;
        L.o_misc = o;   o += al(M_SLOTS * 8);
        L.o_bitmap = o; o += al((L.nseg1 + 1) * SIEVE_WORDS * 4);
        L.o_segcnt = o; o += al(nsegmax * 8);
        L.o_segoff = o; o += al((nsegmax + 1) * 8);
        L.o_base1 = o;  o += al(L.nbase1_cap * 4 + 4);
        L.o_tiles = o;  o += al(ntiles(nsegmax + 1) * 8);
        L.total = o;
    }
    const size_t need = L.total;
    void *ws = nullptr;
    CK(cudaMallocAsync(&ws, need, st));
    uint64_t *misc = (uint64_t *)WS(ws, L.o_misc);
    int rc = WV_OK;
    uint64_t cnt = 0;
    do {
        if (cudaMemsetAsync(misc, 0, M_SLOTS * 8, st) != cudaSuccess) { rc = set_err(WV_ECUDA, "memset"); break; }
        const uint32_t *base;
        uint32_t nbh;
        const uint64_t *nbd;
        if ((rc = base_list(c, L, ws, st, &base, &nbh, &nbd)) != WV_OK) break;
        uint64_t *segcnt = (uint64_t *)WS(ws, L.o_segcnt);
        uint64_t *segoff = (uint64_t *)WS(ws, L.o_segoff);
        uint64_t *tiles = (uint64_t *)WS(ws, L.o_tiles);
        if (L.nseg > 0) {
            sieve_segments_kernel<<<(unsigned)L.nseg, SIEVE_THREADS, 0, st>>>(L.map, base, nbh, nbd, nullptr, segcnt);
            g_launches.fetch_add(1);
            if ((rc = scan_excl<uint64_t>(segcnt, L.nseg, segoff, misc + M_NPRIMES, tiles, st)) != WV_OK) break;
        }
        if (cudaMemcpyAsync(&cnt, misc + M_NPRIMES, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess) {
            rc = set_err(WV_ECUDA, "copy");
            break;
        }
    } while (0);
    (void)nsegmax;
    cudaFreeAsync(ws, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess && rc == WV_OK) rc = set_err(WV_ECUDA, "prime_count: %s", cudaGetErrorString(e));
    if (rc == WV_OK && count) *count = cnt;
    return rc;
}

// ------------------------------------------------------------------ host API
static int search_host(uint64_t lo, uint64_t hi, uint32_t mode, uint32_t shard, uint32_t nshards, uint64_t block,
                       wv_hit *out_hits, size_t hits_cap, size_t *n_hits, wv_residue *out_res, size_t res_cap,
                       size_t *n_primes, uint64_t *checksum) {
    Layout L;
    TRY(make_layout(lo, hi, mode, shard, nshards, block, L));
    DevCtx *c;
    TRY(ctx_get(&c));
    cudaStream_t st = c->stream;
    const uint64_t cap = L.prime_cap > 0 ? L.prime_cap : 1;
    const size_t bytes = L.total + al(cap * 8) * 3 + al(cap * sizeof(wv_hit)) + al(cap * sizeof(wv_residue)) + 256;
    char *buf = nullptr;
    CK(cudaMallocAsync((void **)&buf, bytes, st));
    size_t o = 0;
    void *ws = buf + o;           o += L.total;
    uint64_t *primes = (uint64_t *)(buf + o); o += al(cap * 8);
    uint64_t *rw = (uint64_t *)(buf + o);     o += al(cap * 8);
    uint64_t *rv = (uint64_t *)(buf + o);     o += al(cap * 8);
    wv_hit *hits = (wv_hit *)(buf + o);       o += al(cap * sizeof(wv_hit));
    ResOut *packed = (ResOut *)(buf + o);     o += al(cap * sizeof(wv_residue));
    uint64_t *dchk = (uint64_t *)(buf + o);
    size_t np = 0, nh = 0;
    int rc = search_device_impl(L, primes, rw, rv, hits, dchk, ws, st, &np, &nh);
    if (rc == WV_OK) {
        if (n_primes) *n_primes = np;
        if (n_hits) *n_hits = nh;
        if (nh > hits_cap || (out_res && np > res_cap)) {
            rc = set_err(WV_ENOSPC, "capacity: hits %zu/%zu, residues %zu/%zu", nh, hits_cap, np, res_cap);
        } else {
            if (out_res && np > 0) {
                unsigned g = (unsigned)((np + 255) / 256 < (uint64_t)c->sms * 16 ? (np + 255) / 256 : c->sms * 16);
                pack_residues_kernel<<<g, 256, 0, st>>>(primes, np, rw, rv, packed);
                g_launches.fetch_add(1);
                cudaMemcpyAsync(out_res, packed, np * sizeof(wv_residue), cudaMemcpyDeviceToHost, st);
            }
            if (nh > 0) cudaMemcpyAsync(out_hits, hits, nh * sizeof(wv_hit), cudaMemcpyDeviceToHost, st);
            if (checksum) cudaMemcpyAsync(checksum, dchk, 8, cudaMemcpyDeviceToHost, st);
            cudaError_t e = cudaStreamSynchronize(st);
            if (e == cudaSuccess) e = cudaGetLastError();
            if (e != cudaSuccess) rc = set_err(WV_ECUDA, "copy-out: %s", cudaGetErrorString(e));
        }
    }
    cudaFreeAsync(buf, st);
    cudaStreamSynchronize(st);
    return rc;
}

extern "C" int wv_search(uint64_t lo, uint64_t hi, uint32_t mode, wv_hit *out_hits, size_t hits_cap, size_t *n_hits,
                         wv_residue *out_residues, size_t res_cap, size_t *n_primes) {
    return search_host(lo, hi, mode, 0, 1, 0, out_hits, hits_cap, n_hits, out_residues, res_cap, n_primes, nullptr);
}

extern "C" int wv_search_shard(uint64_t lo, uint64_t hi, uint32_t mode, uint32_t shard, uint32_t nshards,
                               uint64_t block, wv_hit *out_hits, size_t hits_cap, size_t *n_hits,
                               wv_residue *out_residues, size_t res_cap, size_t *n_primes, uint64_t *checksum) {
    return search_host(lo, hi, mode, shard, nshards, block, out_hits, hits_cap, n_hits, out_residues, res_cap,
                       n_primes, checksum);
}

extern "C" int wv_shard_blocks(uint64_t lo, uint64_t hi, uint32_t shard, uint32_t nshards, uint64_t block,
                               uint64_t *out, size_t cap, size_t *n, uint64_t *block_used) {
    Layout L;
    TRY(make_layout(lo, hi, 1, shard, nshards, block, L));
    const uint64_t nblocks = (hi - lo + L.block - 1) / L.block;
    const uint64_t pad = shard_pad(nblocks, nshards);
    size_t k = 0;
    for (uint64_t j = 0; j < (nblocks + pad) / nshards; j++) {
        const uint64_t vb = shard_block(j, shard, nshards);
        if (vb < pad) continue;
        const uint64_t b = vb - pad;
        const uint64_t a_ = lo + b * L.block, z = a_ + L.block < hi ? a_ + L.block : hi;
        if (z <= a_) continue;
        if (out && k < cap) { out[2 * k] = a_; out[2 * k + 1] = z; }
        k++;
    }
    if (n) *n = k;
    if (block_used) *block_used = L.block;
    if (out && k > cap) return set_err(WV_ENOSPC, "cap %zu < %zu blocks", cap, k);
    return WV_OK;
}

// ------------------------------------------------------------------ utilities
extern "C" uint64_t wv_checksum_term(uint64_t p, uint64_t res_w, uint64_t res_v) { return checksum_term(p, res_w, res_v); }

extern "C" int wv_congruence_count(void) { return (int)table().hdr.size(); }

extern "C" int wv_congruence_get(int id, wv_congruence *out) {
    const Table &T = table();
    if (id < 0 || id >= (int)T.hdr.size() || !out) return set_err(WV_EINVAL, "congruence id %d", id);
    const Cong &c = T.hdr[id];
    if (c.m > 33 || c.L_hi || c.L_lo >> 63) return set_err(WV_EINVAL, "congruence %d does not fit wv_congruence", id);
    memset(out, 0, sizeof *out);
    memcpy(out->name, c.name, 8);
    out->L = c.L_neg ? -(int64_t)c.L_lo : (int64_t)c.L_lo;
    out->e = c.e; out->m = c.m; out->min_p = c.min_p; out->excluded_p = c.excluded_p;
    for (uint32_t j = 0; j < c.m; j++) {
        const Term &t = T.terms[c.off + j];
        if (t.a_hi || t.a_lo >> 63) return set_err(WV_EINVAL, "coefficient too large");
        out->t[j] = wv_term{t.neg ? -(int64_t)t.a_lo : (int64_t)t.a_lo, t.xn, t.xd, t.yn, t.yd};
    }
    return WV_OK;
}

extern "C" int wv_congruence_header(int id, wv_cong_header *out) {
    const Table &T = table();
    if (id < 0 || id >= (int)T.hdr.size() || !out) return set_err(WV_EINVAL, "congruence id %d", id);
    const Cong &c = T.hdr[id];
    memcpy(out->name, c.name, 8);
    out->L_lo = c.L_lo; out->L_hi = c.L_hi; out->L_neg = c.L_neg;
    out->e = c.e; out->m = c.m; out->min_p = c.min_p; out->excluded_p = c.excluded_p; out->seg = c.seg;
    return WV_OK;
}

extern "C" int wv_congruence_term(int id, uint32_t j, wv_term128 *out) {
    const Table &T = table();
    if (id < 0 || id >= (int)T.hdr.size() || !out || j >= T.hdr[id].m) return set_err(WV_EINVAL, "term %d/%u", id, j);
    const Term &t = T.terms[T.hdr[id].off + j];
    out->a_lo = t.a_lo; out->a_hi = t.a_hi; out->neg = t.neg;
    out->xn = t.xn; out->xd = t.xd; out->yn = t.yn; out->yd = t.yd;
    return WV_OK;
}

extern "C" int wv_set_schedule_override(int w_id, int v_id) {
    const Table &T = table();
    const int n = (int)T.hdr.size();
    if (w_id >= n || v_id >= n) return set_err(WV_EINVAL, "congruence id out of range");
    if (w_id >= 0 && T.hdr[w_id].e != 3) return set_err(WV_EINVAL, "%s is not a Bernoulli congruence", T.hdr[w_id].name);
    if (v_id >= 0 && T.hdr[v_id].e != 2) return set_err(WV_EINVAL, "%s is not an Euler congruence", T.hdr[v_id].name);
    g_sched.w_force = w_id < 0 ? -1 : w_id;
    g_sched.v_force = v_id < 0 ? -1 : v_id;
    return WV_OK;
}

extern "C" int wv_schedule(uint64_t p, uint32_t test) {
    if (test != WV_MODE_W && test != WV_MODE_V) return set_err(WV_EINVAL, "test must be W or V");
    (void)table();
    return schedule(g_sched, p, test == WV_MODE_W ? 0 : 1);
}

extern "C" uint64_t wv_launch_count(void) { return g_launches.load(); }

extern "C" int wv_kernel_variant_info(int id, char *name, size_t name_cap, int *cls) {
    if (id < 0 || id >= NVAR) return set_err(WV_EINVAL, "variant %d out of range", id);
    if (name && name_cap) snprintf(name, name_cap, "%s", kVariants[id].name);
    if (cls) *cls = kVariants[id].cls;
    return WV_OK;
}

extern "C" int wv_set_kernel_variant(int cls, int id) {
    if (cls < 0 || cls > 2) return set_err(WV_EINVAL, "class %d", cls);
    read_variant_env();
    if (id < 0) { g_variant[cls] = kDefaultVariant[cls]; return WV_OK; }
    if (id >= NVAR || kVariants[id].cls != cls) return set_err(WV_EINVAL, "variant %d is not for class %d", id, cls);
    g_variant[cls] = id;
    return WV_OK;
}

extern "C" int wv_stats_enable(int on) {
    g_stats_on.store(on ? 1 : 0);
    return WV_OK;
}
extern "C" int wv_stats_get(wv_stats *out) {
    if (!out) return set_err(WV_EINVAL, "null");
    std::lock_guard<std::mutex> lk(g_stats_mu);
    *out = g_stats;
    return WV_OK;
}
extern "C" int wv_stats_reset(void) {
    std::lock_guard<std::mutex> lk(g_stats_mu);
    memset(&g_stats, 0, sizeof g_stats);
    return WV_OK;
}

extern "C" const char *wv_version(void) {
    return "libwv 0.2 (sm_100a; Mont32 p<2^30 | FP64 EFT p<2^44 | Mont64 p<2^62; sieve+plan+residue+finalize)";
}

extern "C" const char *wv_last_error(void) { return g_err; }

// ------------------------------------------------------------------ NEXT-3: index census
// Sieve -> per-prime plan (primitive root, exponent and item counts) -> scans -> batches of
// <= CEN_BUDGET index residues: walk, finalize, fix-up.  See wv_census.cuh and include/wv.h.
static const uint64_t CEN_BUDGET = 1ull << 25;     // index residues per batch (acc: 256 MB)

namespace {
struct DevBufs {                                   // cudaFreeAsync on scope exit
    cudaStream_t st;
    std::vector<void *> v;
    explicit DevBufs(cudaStream_t s) : st(s) {}
    ~DevBufs() { for (void *p : v) cudaFreeAsync(p, st); cudaStreamSynchronize(st); }
    template <typename T> int get(T **out, size_t n) {
        void *p = nullptr;
        if (cudaMallocAsync(&p, n ? n * sizeof(T) : 1, st) != cudaSuccess)
            return set_err(WV_ENOMEM, "cudaMallocAsync(%zu) failed", n * sizeof(T));
        v.push_back(p);
        *out = (T *)p;
        return WV_OK;
    }
};
}  // namespace

static int census_impl(uint64_t lo, uint64_t hi, uint32_t mode, wv_pair *out, size_t cap, size_t *n_pairs,
                       size_t *n_primes, uint64_t *checksum, wv_index_residue *out_res, size_t res_cap, size_t *n_res,
                       bool want_res) {
    static_assert(sizeof(wv_pair) == sizeof(CenPair), "wv_pair layout");
    if (hi <= lo) return set_err(WV_EINVAL, "empty or inverted range [%llu, %llu)", (unsigned long long)lo,
                                 (unsigned long long)hi);
    if (hi > CEN_HI_MAX) return set_err(WV_EINVAL, "census needs hi <= 2^26");
    if (mode < 1 || mode > 3) return set_err(WV_EINVAL, "mode %u not in {1,2,3}", mode);
    DevCtx *c;
    TRY(ctx_get(&c));
    cudaStream_t st = c->stream;
    const uint64_t lo5 = lo < 5 ? 5 : lo;
    uint64_t n = 0;
    DevBufs B(st);
    uint64_t *d_primes = nullptr;
    if (hi > lo5) {
        const uint64_t pc = prime_bound(hi - lo5) + 1;
        TRY(B.get(&d_primes, pc));
        size_t nn = 0;
        TRY(wv_sieve_device(lo5, hi, d_primes, pc, &nn, nullptr, 0, st));
        n = nn;
    }
    if (n_primes) *n_primes = n;
    std::vector<uint64_t> hp(n), heb(n + 1, 0), his(n + 1, 0);
    if (n) CK(cudaMemcpy(hp.data(), d_primes, n * 8, cudaMemcpyDeviceToHost));
    uint64_t nrec = 0;
    for (uint64_t i = 0; i < n; i++) nrec += (hp[i] - 3) / 2;
    if (n_res) *n_res = nrec;
    if (want_res && nrec > 0 && (!out_res || res_cap < nrec))
        return set_err(WV_ENOSPC, "cap %zu < %llu index residues", res_cap, (unsigned long long)nrec);
    uint64_t chk = 0, npairs = 0;
    std::vector<CenPair> hpairs;
    if (n) {
        uint32_t *d_g;
        uint64_t *d_ne, *d_ni, *d_eb, *d_is, *d_tiles;
        unsigned long long *d_misc;
        TRY(B.get(&d_g, n));
        TRY(B.get(&d_ne, n));
        TRY(B.get(&d_ni, n));
        TRY(B.get(&d_eb, n + 1));
        TRY(B.get(&d_is, n + 1));
        TRY(B.get(&d_tiles, ntiles(n + 1)));
        TRY(B.get(&d_misc, 8));
        CK(cudaMemsetAsync(d_misc, 0, 64, st));
        const unsigned gp = (unsigned)((n + 127) / 128 < (uint64_t)c->sms * 8 ? (n + 127) / 128 : c->sms * 8);
        LAUNCH(census_plan_kernel, gp, 128, st, d_primes, n, mode, d_g, d_ne, d_ni);
        TRY(scan_excl<uint64_t>(d_ne, n, d_eb, d_eb + n, d_tiles, st));
        TRY(scan_excl<uint64_t>(d_ni, n, d_is, d_is + n, d_tiles, st));
        CK(cudaMemcpyAsync(heb.data(), d_eb, (n + 1) * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(his.data(), d_is, (n + 1) * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        // batches [i0, i1) of <= CEN_BUDGET index residues (at least one prime)
        std::vector<uint64_t> cut{0};
        uint64_t amax = 0;
        while (cut.back() < n) {
            const uint64_t i0 = cut.back();
            uint64_t i1 = i0 + 1;
            while (i1 < n && heb[i1 + 1] - heb[i0] <= CEN_BUDGET) i1++;
            cut.push_back(i1);
            if (heb[i1] - heb[i0] > amax) amax = heb[i1] - heb[i0];
        }
        unsigned long long *d_acc;
        uint64_t *d_res = nullptr;
        CenFix *d_fix;
        CenPair *d_pairs;
        const uint64_t fcap = amax / 8 + 1024, pcap = cap > 65536 ? cap : 65536;
        TRY(B.get(&d_acc, amax));
        if (want_res) TRY(B.get(&d_res, amax));
        TRY(B.get(&d_fix, fcap));
        TRY(B.get(&d_pairs, pcap));
        std::vector<uint64_t> hres;
        const uint64_t per = mode == 3 ? 2 : 1;          // walked exponents per index record
        for (size_t b = 0; b + 1 < cut.size(); b++) {
            const uint64_t i0 = cut[b], i1 = cut[b + 1], nE = heb[i1] - heb[i0];
            CK(cudaMemsetAsync(d_acc, 0, nE * 8, st));
            CK(cudaMemsetAsync(d_misc + 2, 0, 24, st));  // fix count, unresolved, walk counter
            LAUNCH(census_walk_kernel, c->sms * c->occ_census, CEN_THREADS, st, d_primes, d_g, d_is, d_eb, i0, i1,
                   mode, d_acc, d_misc + 4);
            const unsigned gf = (unsigned)((i1 - i0) < (uint64_t)c->sms * 8 ? (i1 - i0) : c->sms * 8);
            LAUNCH(census_finalize_kernel, gf, CEN_FIN_T, st, d_primes, d_eb, i0, i1, mode, d_acc, d_res, d_pairs, pcap,
                   d_fix, fcap, d_misc);
            uint64_t hm[2] = {0, 0};
            CK(cudaMemcpyAsync(hm, d_misc + 2, 16, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (hm[0] > fcap) return set_err(WV_ECUDA, "census fix-up queue overflow (%llu > %llu)",
                                             (unsigned long long)hm[0], (unsigned long long)fcap);
            if (hm[0]) {
                const unsigned gx = (unsigned)((hm[0] * 32 + 255) / 256 < (uint64_t)c->sms * 8 ? (hm[0] * 32 + 255) / 256
                                                                                                : c->sms * 8);
                LAUNCH(census_fixup_kernel, gx, 256, st, d_primes, d_eb, i0, mode, d_fix, hm[0], d_res, d_pairs, pcap,
                       d_misc);
                CK(cudaMemcpyAsync(hm, d_misc + 3, 8, cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                if (hm[0]) return set_err(WV_ECUDA, "census: %llu B indices with no unit C_k among the congruences",
                                          (unsigned long long)hm[0]);
            }
            if (want_res) {
                hres.resize(nE);
                CK(cudaMemcpy(hres.data(), d_res, nE * 8, cudaMemcpyDeviceToHost));
                uint64_t r = 0;
                for (uint64_t i = 0; i < i0; i++) r += (hp[i] - 3) / 2;
                for (uint64_t i = i0; i < i1; i++) {
                    const uint64_t base = heb[i] - heb[i0], m = (hp[i] - 3) / 2;
                    for (uint64_t j = 0; j < m; j++, r++) {
                        wv_index_residue &o = out_res[r];
                        o.p = hp[i]; o.index = (uint32_t)(2 * j + 2); o.reserved = 0;
                        o.res_b = mode == 2 ? UINT64_MAX : hres[base + per * j];
                        o.res_e = mode == 1 ? UINT64_MAX : hres[base + per * j + (mode == 3 ? 1 : 0)];
                    }
                }
            }
        }
        uint64_t hm[2];
        CK(cudaMemcpyAsync(hm, d_misc, 16, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        npairs = hm[0];
        chk = hm[1];
        const uint64_t got = npairs < pcap ? npairs : pcap;
        hpairs.resize(got);
        if (got) CK(cudaMemcpy(hpairs.data(), d_pairs, got * sizeof(CenPair), cudaMemcpyDeviceToHost));
    }
    if (checksum) *checksum = chk;
    if (n_pairs) *n_pairs = npairs;
    std::sort(hpairs.begin(), hpairs.end(), [](const CenPair &a, const CenPair &b) {
        return a.p != b.p ? a.p < b.p : (a.kind != b.kind ? a.kind < b.kind : a.index < b.index);
    });
    if (out) memcpy(out, hpairs.data(), (hpairs.size() < cap ? hpairs.size() : cap) * sizeof(wv_pair));
    if (npairs > cap && (out || cap)) return set_err(WV_ENOSPC, "cap %zu < %llu pairs", cap, (unsigned long long)npairs);
    return WV_OK;
}

extern "C" int wv_census(uint64_t lo, uint64_t hi, uint32_t mode, wv_pair *out, size_t cap, size_t *n_pairs,
                         size_t *n_primes, uint64_t *checksum) {
    return census_impl(lo, hi, mode, out, cap, n_pairs, n_primes, checksum, nullptr, 0, nullptr, false);
}

extern "C" int wv_census_residues(uint64_t lo, uint64_t hi, uint32_t mode, wv_index_residue *out, size_t cap,
                                  size_t *n) {
    return census_impl(lo, hi, mode, nullptr, 0, nullptr, nullptr, nullptr, out, cap, n, true);
}

extern "C" uint64_t wv_census_checksum_term(uint64_t p, uint32_t index, uint32_t kind, uint64_t res) {
    return cen_checksum_term(p, index, kind, res);
}
