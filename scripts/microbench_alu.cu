// microbench_alu.cu -- measured per-SM throughput of the instructions the residue
// loop is built from (sm_100a): IMAD (mad.lo.u32), IMAD.WIDE (mad.wide.u32),
// IMAD.HI (mad.hi.u32), IADD3, VIADDMNMX-style add+min, DFMA, and a full lazy
// Mont32 product.  8 independent dependency chains per thread, 64 warps/SM.
// Each CTA records its SM id and clock64() at start and end; per SM the span is
// max(end) - min(start) over the CTAs that ran there (clock64 is a per-SM
// counter), so waves and launch gaps are inside the span.  Output: per-lane
// ops/clk/SM, the median over SMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench_alu scripts/microbench_alu.cu
//   ./microbench_alu [out.json]      (JSON: per-lane ops/clk/SM of each probe, for bench.py's peaks)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <algorithm>
#include <vector>

constexpr int CH = 8;
constexpr int ITERS = 16384;

template <int OP>
__global__ void __launch_bounds__(256) bench(uint64_t *out, unsigned long long *cyc, uint32_t seed) {
    // cyc[3 * blockIdx.x + {0, 1, 2}] = sm id, start, end
    uint32_t a[CH];
    uint64_t w[CH];
    double d[CH];
    const uint32_t b = seed | 1, c = seed * 7 + 3;
    for (int j = 0; j < CH; j++) {
        a[j] = seed + threadIdx.x * 13 + j;
        w[j] = a[j];
        d[j] = 1.0 + 1e-9 * a[j];
    }
    __syncthreads();
    long long t0 = clock64();
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    for (int i = 0; i < ITERS; i++) {
        #pragma unroll
        for (int j = 0; j < CH; j++) {
            if (OP == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(b), "r"(c));
            if (OP == 1) {
                uint32_t lo = (uint32_t)w[j];
                asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[j]) : "r"(lo), "r"(b));
            }
            if (OP == 2) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(b), "r"(c));
            if (OP == 3) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[j]) : "d"(0.999999), "d"(1e-7));
            if (OP == 4) asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(a[j]) : "r"(b), "r"(c));
            if (OP == 5) {   // lazy modular add: s = a + b; a = min(s, s - 2p)
                uint32_t s = a[j] + b;
                asm volatile("min.u32 %0, %1, %2;" : "=r"(a[j]) : "r"(s), "r"(s - c));
            }
            if (OP == 6) {   // Mont32 product a <- a*b R^-1 (lazy)
                uint64_t T;
                asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(T) : "r"(a[j]), "r"(b));
                uint32_t m = (uint32_t)T * c;
                uint64_t r;
                asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(m), "r"(b | 1), "l"(T));
                a[j] = (uint32_t)(r >> 32);
            }
            if (OP == 7) asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(a[j]) : "r"(b));
            if (OP == 8) {   // Mont64 product w <- w*b R^-1 (R = 2^64, lazy; the class-2 engine's form)
                const uint64_t B = ((uint64_t)b << 31) | 1u, P = ((uint64_t)c << 33) | 1u, PI = B * 3u + 1u;
                uint64_t lo = w[j] * B, hi = __umul64hi(w[j], B);
                uint64_t m = lo * PI;
                w[j] = hi + __umul64hi(m, P) + (lo != 0);
            }
        }
    }
    long long t1 = clock64();
    uint64_t acc = 0;
    for (int j = 0; j < CH; j++) acc += a[j] + w[j] + (uint64_t)d[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        cyc[3 * blockIdx.x] = smid;
        cyc[3 * blockIdx.x + 1] = (unsigned long long)t0;
        cyc[3 * blockIdx.x + 2] = (unsigned long long)clock64();
    }
}

static FILE *g_json = nullptr;
static int g_first = 1;

template <int OP>
void run(const char *name, const char *key, int sms, int ops_per_iter_chain) {
    const int blocks = sms * 8, threads = 256;     // 64 warps/SM if resident; waves are inside the span
    uint64_t *out;
    unsigned long long *cyc;
    cudaMalloc(&out, (size_t)blocks * threads * 8);
    cudaMalloc(&cyc, (size_t)blocks * 3 * 8);
    std::vector<unsigned long long> h((size_t)blocks * 3);
    for (int rep = 0; rep < 3; rep++) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        bench<OP><<<blocks, threads>>>(out, cyc, 12345u + rep);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpy(h.data(), cyc, h.size() * 8, cudaMemcpyDeviceToHost);
        std::vector<unsigned long long> lo(sms, ~0ull), hi(sms, 0);
        std::vector<int> nb(sms, 0);
        for (int b = 0; b < blocks; b++) {
            const int s = (int)h[3 * b];
            if (s < 0 || s >= sms) continue;
            lo[s] = std::min(lo[s], h[3 * b + 1]);
            hi[s] = std::max(hi[s], h[3 * b + 2]);
            nb[s]++;
        }
        std::vector<double> rate, span;
        for (int s = 0; s < sms; s++)
            if (nb[s] > 0) {
                const double ops = (double)nb[s] * threads * ITERS * CH * ops_per_iter_chain;   // per-lane ops
                rate.push_back(ops / (double)(hi[s] - lo[s]));
                span.push_back((double)(hi[s] - lo[s]));
            }
        std::sort(rate.begin(), rate.end());
        std::sort(span.begin(), span.end());
        const double med = rate[rate.size() / 2];
        const double mhz = span.back() / (ms * 1e3);      // longest SM span over the event time
        if (rep == 2) {
            printf("%-22s %8.2f ops/clk/SM (median over %zu SMs, min %.2f max %.2f)   %8.3f ms   ~%.0f MHz\n", name,
                   med, rate.size(), rate.front(), rate.back(), ms, mhz);
            if (g_json) {
                fprintf(g_json, "%s \"%s\": %.4f, \"%s_mhz\": %.1f", g_first ? "" : ",\n", key, med, key, mhz);
                g_first = 0;
            }
        }
    }
    cudaFree(out);
    cudaFree(cyc);
}

int main(int argc, char **argv) {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    int sms = prop.multiProcessorCount;
    printf("device %s, %d SMs\n", prop.name, sms);
    if (argc > 1) {
        g_json = fopen(argv[1], "w");
        fprintf(g_json, "{\"device\": \"%s\", \"sms\": %d, \"unit\": \"per-lane ops per clock per SM\",\n", prop.name,
                sms);
        fprintf(g_json, " \"how\": \"scripts/microbench_alu.cu: 8 independent chains/thread, 64 warps/SM, clock64 per CTA\",\n");
    }
    run<0>("IMAD (mad.lo)", "imad_per_clk_sm", sms, 1);
    run<7>("IMUL (mul.lo)", "imul_per_clk_sm", sms, 1);
    run<1>("IMAD.WIDE", "imad_wide_per_clk_sm", sms, 1);
    run<2>("IMAD.HI (mad.hi)", "imad_hi_per_clk_sm", sms, 1);
    run<4>("IADD (2 adds)", "iadd_per_clk_sm", sms, 2);
    run<5>("lazy modadd (add+min)", "modadd_ops_per_clk_sm", sms, 2);
    run<3>("DFMA", "dfma_per_clk_sm", sms, 1);
    run<6>("Mont32 product", "mont32_product_per_clk_sm", sms, 1);
    run<8>("Mont64 product", "mont64_product_per_clk_sm", sms, 1);
    if (g_json) {
        fprintf(g_json, "\n}\n");
        fclose(g_json);
    }
    return 0;
}
