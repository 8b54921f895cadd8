// microbench_dual.cu -- terms/s of hot-loop variants for p < 2^30 (E = 2, 3):
//   INT   : Montgomery (Mont32) term stream on the IMAD pipes
//   FP    : exact FP64 error-free-transform term stream on the DFMA pipe
//   DUAL  : one INT and one FP stream interleaved in the same thread (cross-pipe ILP)
//   DUAL21: two INT streams + one FP stream
// Long runs (~0.3-1 s) so clocks settle.
// CAVEAT (found later): the output only consumes some streams' a1 chains, so
// the compiler deletes the unused ones and INTx2/x3/x4, DUAL21 are inflated.
// Single-stream INT / FP / DUAL numbers are valid.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench_dual scripts/microbench_dual.cu
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
    __device__ __forceinline__ uint32_t add(uint32_t a, uint32_t b) const {
        uint32_t s = a + b;
        return min(s, s - p2);
    }
};
struct MD {
    double p, pinv;
    static constexpr double MAGIC = 6755399441055744.0;
    __device__ __forceinline__ double mul(double a, double b) const {
        const double h = __dmul_rn(a, b);
        const double l = __fma_rn(a, b, -h);
        const double q = __dadd_rn(__fma_rn(h, pinv, MAGIC), -MAGIC);
        return __dadd_rn(__fma_rn(-q, p, h), l);
    }
    __device__ __forceinline__ double reduce(double x) const {
        const double q = __dadd_rn(__fma_rn(x, pinv, MAGIC), -MAGIC);
        return __fma_rn(-q, p, x);
    }
};

template <int E>
struct IS {   // INT stream
    uint32_t u, d1, d2, a0, a1;
    __device__ __forceinline__ void init(uint32_t seed, uint32_t p) { u = seed % p; d1 = (seed * 7) % p; d2 = 12 % p; a0 = 1; a1 = 0; }
    __device__ __forceinline__ void step(const M32 &m) {
        a1 = m.muladd(a1, u, a0);
        a0 = m.mul(a0, u);
        u = m.add(u, d1);
        d1 = m.add(d1, d2);
        if (E == 3) d2 = m.add(d2, 6);
    }
};
template <int E>
struct FS {   // FP64 stream
    double u, d1, d2, a0, a1;
    __device__ __forceinline__ void init(uint32_t seed, uint32_t p) { u = seed % p; d1 = (seed * 7) % (p / 2); d2 = 2; a0 = 1; a1 = 0; }
    __device__ __forceinline__ void step(const MD &m) {
        a1 = __dadd_rn(m.mul(a1, u), a0);
        a0 = m.mul(a0, u);
        u = __dadd_rn(u, d1);
        d1 = __dadd_rn(d1, d2);
        if (E == 3) d2 = __dadd_rn(d2, 6.0);
    }
    __device__ __forceinline__ void red(const MD &m) { u = m.reduce(u); d1 = m.reduce(d1); }
};

// V: 0 INT, 1 FP, 2 DUAL (1 INT + 1 FP), 3 DUAL21 (2 INT + 1 FP), 4 INT x2, 5 INT x3, 6 INT x4, 7 FP x2
template <int E, int V>
__global__ void __launch_bounds__(256) loop(uint32_t p, uint32_t pinv, double pd, double pinvd, uint32_t n, uint32_t *out) {
    M32 mi{p, pinv, 2 * p};
    MD mf{pd, pinvd};
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    IS<E> i1, i2, i3, i4;
    FS<E> f1, f2;
    i1.init(tid * 2654435761u + 1, p);
    i2.init(tid * 40503u + 7, p);
    i3.init(tid * 7u + 11, p);
    i4.init(tid * 13u + 17, p);
    f1.init(tid * 97u + 3, p);
    f2.init(tid * 101u + 5, p);
    #pragma unroll 1
    for (uint32_t it = 0; it < n; it += 16) {
        #pragma unroll
        for (int k = 0; k < 16; k++) {
            if (V == 0 || V == 2 || V == 3 || V == 4 || V == 5 || V == 6) i1.step(mi);
            if (V == 3 || V == 4 || V == 5 || V == 6) i2.step(mi);
            if (V == 5 || V == 6) i3.step(mi);
            if (V == 6) i4.step(mi);
            if (V == 1 || V == 2 || V == 3 || V == 7) f1.step(mf);
            if (V == 7) f2.step(mf);
        }
        if (V == 1 || V == 2 || V == 3 || V == 7) f1.red(mf);
        if (V == 7) f2.red(mf);
    }
    out[tid] = i1.a0 ^ i1.a1 ^ i2.a0 ^ i3.a0 ^ i4.a1 ^ (uint32_t)f1.a0 ^ (uint32_t)f1.a1 ^ (uint32_t)f2.a1;
}

template <int E, int V>
void run(const char *name, int sms, int bps, int streams) {
    const uint32_t p = 1000000007u;
    uint32_t inv = p;
    for (int i = 0; i < 5; i++) inv *= 2u - p * inv;
    const uint32_t pinv = 0u - inv;
    uint32_t *out;
    const int blocks = sms * bps, threads = 256;
    cudaMalloc(&out, blocks * threads * 4);
    const uint32_t n = 1 << 16;
    float best = 1e30f;
    for (int rep = 0; rep < 4; rep++) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        loop<E, V><<<blocks, threads>>>(p, pinv, (double)p, 1.0 / (double)p, n, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, loop<E, V>);
    double terms = (double)blocks * threads * n * streams;
    printf("E=%d %-8s regs %3d blocks/SM %d: %8.2f ms  %.3e terms/s\n", E, name, fa.numRegs, bps, best,
           terms / (best * 1e-3));
    cudaFree(out);
}

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    int sms = prop.multiProcessorCount;
    printf("%s %d SMs\n", prop.name, sms);
    for (int bps : {2, 4}) {
        run<2, 0>("INT", sms, bps, 1);
        run<2, 4>("INTx2", sms, bps, 2);
        run<2, 5>("INTx3", sms, bps, 3);
        run<2, 6>("INTx4", sms, bps, 4);
        run<2, 1>("FP", sms, bps, 1);
        run<2, 7>("FPx2", sms, bps, 2);
        run<3, 0>("INT", sms, bps, 1);
        run<3, 4>("INTx2", sms, bps, 2);
        run<3, 6>("INTx4", sms, bps, 4);
        run<3, 7>("FPx2", sms, bps, 2);
    }
    return 0;
}
