// microbench_alu.cu -- measured per-SM throughput of the instructions the residue
// loop is built from (sm_100a): IMAD (mad.lo.u32), IMAD.WIDE (mad.wide.u32),
// IMAD.HI (mad.hi.u32), IADD3, VIADDMNMX-style add+min, DFMA, and a full lazy
// Mont32 product.  8 independent dependency chains per thread, 32 warps/SM,
// cycles from clock64() per CTA.  Output: ops/clk/SM (per-lane ops).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench_alu scripts/microbench_alu.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int CH = 8;
constexpr int ITERS = 2048;

template <int OP>
__global__ void __launch_bounds__(256) bench(uint64_t *out, unsigned long long *cyc, uint32_t seed) {
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
        }
    }
    long long t1 = clock64();
    uint64_t acc = 0;
    for (int j = 0; j < CH; j++) acc += a[j] + w[j] + (uint64_t)d[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) atomicMax(cyc, (unsigned long long)(t1 - t0));
}

template <int OP>
void run(const char *name, int sms, int ops_per_iter_chain) {
    const int blocks = sms * 8, threads = 256;     // 64 warps/SM
    uint64_t *out;
    unsigned long long *cyc;
    cudaMalloc(&out, (size_t)blocks * threads * 8);
    cudaMalloc(&cyc, 8);
    for (int rep = 0; rep < 2; rep++) {
        cudaMemset(cyc, 0, 8);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        bench<OP><<<blocks, threads>>>(out, cyc, 12345u + rep);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        double ops = (double)blocks * threads * ITERS * CH * ops_per_iter_chain;   // per-lane instructions
        double per_sm_clk = ops / sms / (double)c;
        if (rep == 1)
            printf("%-22s %8.2f ops/clk/SM   %8.3f ms   %.3e ops/s   (%.0f MHz effective)\n", name, per_sm_clk, ms,
                   ops / (ms * 1e-3), (double)c / (ms * 1e3));
    }
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    int sms = prop.multiProcessorCount;
    printf("device %s, %d SMs\n", prop.name, sms);
    run<0>("IMAD (mad.lo)", sms, 1);
    run<7>("IMUL (mul.lo)", sms, 1);
    run<1>("IMAD.WIDE", sms, 1);
    run<2>("IMAD.HI (mad.hi)", sms, 1);
    run<4>("IADD (2 adds)", sms, 2);
    run<5>("lazy modadd (add+min)", sms, 2);
    run<3>("DFMA", sms, 1);
    run<6>("Mont32 product", sms, 1);
    return 0;
}
