// microbench_term.cu -- terms/s of candidate hot loops (one term = one step of
// eqnComputeS with u = s^e advanced by finite differences), Mont32 variants.
// Each thread runs N terms for a fixed p; occupancy like the residue kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench_term scripts/microbench_term.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct M32 {
    uint32_t p, pinv, p2;
    __device__ __forceinline__ uint32_t mul(uint32_t a, uint32_t b) const {
        uint64_t T = (uint64_t)a * b;
        uint32_t m = (uint32_t)T * pinv;
        return (uint32_t)((T + (uint64_t)m * p) >> 32);
    }
    __device__ __forceinline__ uint32_t muladd(uint32_t a, uint32_t b, uint32_t c) const {
        uint64_t T = (uint64_t)a * b + ((uint64_t)c << 32);
        uint32_t m = (uint32_t)T * pinv;
        uint32_t t = (uint32_t)((T + (uint64_t)m * p) >> 32);
        return min(t, t - p2);
    }
    // variant B: lo/hi split, add c after the REDC
    __device__ __forceinline__ uint32_t mulB(uint32_t a, uint32_t b) const {
        uint32_t tl = a * b, th = __umulhi(a, b);
        uint32_t m = tl * pinv;
        uint32_t r;
        // r = hi(m p + (th:tl)) = hi(m p) + th + (tl != 0)
        asm("{\n\t.reg .u32 x;\n\t"
            "mad.lo.cc.u32 x, %1, %2, %3;\n\t"
            "madc.hi.u32 %0, %1, %2, %4;\n\t}"
            : "=r"(r) : "r"(m), "r"(p), "r"(tl), "r"(th));
        return r;
    }
    __device__ __forceinline__ uint32_t muladdB(uint32_t a, uint32_t b, uint32_t c) const {
        uint32_t tl = a * b, th = __umulhi(a, b) + c;
        uint32_t m = tl * pinv;
        uint32_t r;
        asm("{\n\t.reg .u32 x;\n\t"
            "mad.lo.cc.u32 x, %1, %2, %3;\n\t"
            "madc.hi.u32 %0, %1, %2, %4;\n\t}"
            : "=r"(r) : "r"(m), "r"(p), "r"(tl), "r"(th));
        return min(r, r - p2);
    }
    __device__ __forceinline__ uint32_t add(uint32_t a, uint32_t b) const {
        uint32_t s = a + b;
        return min(s, s - p2);
    }
};

template <int E, int V>
__global__ void __launch_bounds__(256) term_loop(uint32_t p, uint32_t pinv, uint32_t n, uint32_t *out) {
    M32 mo{p, pinv, 2 * p};
    uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t u = (tid * 2654435761u) % p, d1 = (tid * 40503u) % p, d2 = 12345 % p, d3 = 6;
    uint32_t a0 = 1, a1 = 0;
    #pragma unroll 1
    for (uint32_t i = 0; i < n; i += 8) {
        #pragma unroll
        for (int k = 0; k < 8; k++) {
            if (V == 0) {
                a1 = mo.muladd(a1, u, a0);
                a0 = mo.mul(a0, u);
            } else {
                a1 = mo.muladdB(a1, u, a0);
                a0 = mo.mulB(a0, u);
            }
            u = mo.add(u, d1);
            d1 = mo.add(d1, d2);
            if (E == 3) d2 = mo.add(d2, d3);
        }
    }
    out[tid] = a0 ^ a1;
}

template <int E, int V>
void run(const char *name, int sms) {
    const uint32_t p = 1000000007u;   // < 2^30
    uint32_t inv = p;
    for (int i = 0; i < 5; i++) inv *= 2u - p * inv;
    const uint32_t pinv = 0u - inv;
    uint32_t *out;
    const int blocks = sms * 5, threads = 256;    // 40 warps/SM like the residue kernel
    cudaMalloc(&out, blocks * threads * 4);
    const uint32_t n = 1 << 16;
    for (int rep = 0; rep < 3; rep++) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        term_loop<E, V><<<blocks, threads>>>(p, pinv, n, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double terms = (double)blocks * threads * n;
        if (rep == 2) printf("%-28s %8.3f ms  %.3e terms/s  %.2f terms/clk/SM @1.965GHz\n", name, ms,
                             terms / (ms * 1e-3), terms / (ms * 1e-3) / sms / 1.965e9);
    }
    cudaFree(out);
}

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    printf("%s %d SMs\n", prop.name, prop.multiProcessorCount);
    run<2, 0>("E=2 baseline (C REDC)", prop.multiProcessorCount);
    run<2, 1>("E=2 lo/hi + madc", prop.multiProcessorCount);
    run<3, 0>("E=3 baseline (C REDC)", prop.multiProcessorCount);
    run<3, 1>("E=3 lo/hi + madc", prop.multiProcessorCount);
    return 0;
}
