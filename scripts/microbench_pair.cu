// microbench_pair.cu -- terms/s of the class-0 pair step (two terms of eqnComputeS per step)
// in two forms, each with two spellings of the Montgomery product:
//   LOOP 0: the kernel's step2: u = s^e by finite differences, D = u1 u2 (one product),
//           N = u1 + u2, a1 <- REDC(a1 D + a0 N), a0 <- REDC(a0 D)          (3 products / pair)
//   LOOP 1: "polynomial pairs": D(s) = (s(s+1))^e and N(s) = s^e + (s+1)^e are polynomials in s
//           of degree 2e and e, advanced by step-2 finite differences -- no product for D
//                                                                               (2 products / pair)
//   MUL 0:  C spelling (as wv_mont.cuh);  MUL 1: inline PTX (mad.wide + explicit high word);
//   MUL 2:  subtractive REDC: m = T_lo p^{-1}, r = T_hi - hi(m p) + p  (no carry: the low words cancel).
//   MUL 3:  as 2, lazy adds forced onto the ALU pipe: x = a + b - 2p (one 3-input IADD3), r = min(x + 2p, x)
//           (VIADDMNMX) -- a 2-input add may be issued as IMAD.IADD on the busy FMA-heavy pipe.
//   MUL 4:  as 3 with -2p laundered through a shuffle, so ptxas cannot rewrite x + 2p as a + b.
// Each thread runs NP pair steps for one p; thread 0 writes its c1/c0 pieces, the host checks
// every variant against a plain reference sum of s^-e (exact, __int128).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench_pair scripts/microbench_pair.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int MUL>
struct M32 {
    uint32_t p, pinv, pinvp, p2, np2, r1, r2;
    __host__ __device__ void init(uint32_t p_) {
        p = p_; p2 = 2 * p;
        uint32_t inv = p;
        for (int i = 0; i < 5; i++) inv *= 2u - p * inv;
        pinv = 0u - inv;
        pinvp = inv;
        np2 = 0u - p2;
#ifdef __CUDA_ARCH__
        if (MUL == 4) asm volatile("shfl.sync.idx.b32 %0, %0, 0, 31, -1;" : "+r"(np2));
#endif
        r1 = (uint32_t)((1ull << 32) % p);
        r2 = (uint32_t)(((uint64_t)r1 * r1) % p);
    }
    __device__ __forceinline__ uint32_t redc(uint64_t T) const {
        if (MUL == 0) {
            uint32_t m = (uint32_t)T * pinv;
            return (uint32_t)((T + (uint64_t)m * p) >> 32);
        } else if (MUL >= 2) {
            // T < p 2^32 (true for T < 8 p^2 when p < 2^29, T < 4 p^2 when p < 2^30): result in (0, p + T/2^32)
            const uint32_t m = (uint32_t)T * pinvp;
            return (uint32_t)(T >> 32) - __umulhi(m, p) + p;
        } else {
            uint32_t m = (uint32_t)T * pinv, lo, hi;
            uint64_t r;
            asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(m), "r"(p), "l"(T));
            asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(r));
            return hi;
        }
    }
    __device__ __forceinline__ uint64_t wide(uint32_t a, uint32_t b) const {
        if (MUL != 1) return (uint64_t)a * b;
        uint64_t r;
        asm("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(b));
        return r;
    }
    __device__ __forceinline__ uint64_t wadd(uint32_t a, uint32_t b, uint64_t c) const {
        if (MUL != 1) return (uint64_t)a * b + c;
        uint64_t r;
        asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(c));
        return r;
    }
    __device__ __forceinline__ uint32_t mul(uint32_t a, uint32_t b) const { return redc(wide(a, b)); }
    __device__ __forceinline__ uint32_t add(uint32_t a, uint32_t b) const {
        if (MUL >= 3) {
            uint32_t x, r;
            asm("add.u32 %0, %1, %2;\n\tadd.u32 %0, %0, %3;" : "=r"(x) : "r"(a), "r"(b), "r"(np2));
            asm("{\n\t.reg .u32 t;\n\tadd.u32 t, %1, %2;\n\tmin.u32 %0, t, %1;\n\t}" : "=r"(r) : "r"(x), "r"(p2));
            return r;
        }
        uint32_t s = a + b; return min(s, s - p2);
    }
    __device__ __forceinline__ uint32_t mul2add(uint32_t a, uint32_t b, uint32_t c, uint32_t d) const {
        uint32_t t = redc(wadd(c, d, wide(a, b)));
        return min(t, t - p2);
    }
};

// (x (x+1))^E mod p and x^E + (x+1)^E mod p, host/device, plain residues in [0, p)
template <int E>
__host__ __device__ __forceinline__ uint32_t polyD(uint64_t x, uint32_t p) {
    uint64_t t = (x % p) * ((x + 1) % p) % p, r = t;
    for (int i = 1; i < E; i++) r = r * t % p;
    return (uint32_t)r;
}
template <int E>
__host__ __device__ __forceinline__ uint32_t polyN(uint64_t x, uint32_t p) {
    uint64_t a = x % p, b = (x + 1) % p, ra = a, rb = b;
    for (int i = 1; i < E; i++) { ra = ra * a % p; rb = rb * b % p; }
    return (uint32_t)((ra + rb) % p);
}

template <int LOOP, int MUL, int E, int S>
__global__ void __launch_bounds__(256) pair_loop(uint32_t p, uint32_t np, uint32_t s0base, uint32_t *out) {
    M32<MUL> mo;
    mo.init(p);
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t a0[S], a1[S];
    // LOOP 0 state
    uint32_t u[S], d1[S], d2[S];
    // LOOP 1 state: D and its 2E differences, N and its E differences (N in R-scaled form)
    uint32_t D[S][2 * E], N[S][E];
    uint32_t Dc = 0, Nc = 0;
    for (int st = 0; st < S; st++) {
        const uint64_t s = (tid == 0 && st == 0) ? s0base : (s0base + 977u * tid + 131071u * st) % (p - 4 * np - 8) + 1;
        a0[st] = mo.r1; a1[st] = 0;
        if (LOOP == 0) {
            u[st] = E == 3 ? (uint32_t)((s * s % p) * s % p) : (uint32_t)(s * s % p);
            if (E == 3) { d1[st] = (uint32_t)((3 * s * s + 3 * s + 1) % p); d2[st] = (uint32_t)((6 * s + 6) % p); }
            else { d1[st] = (uint32_t)(2 * s + 1); d2[st] = 2; }
        } else {
            uint32_t v[2 * E + 1], w[E + 1];
            for (int i = 0; i <= 2 * E; i++) v[i] = polyD<E>(s + 2 * i, p);
            for (int i = 0; i <= E; i++) w[i] = polyN<E>(s + 2 * i, p);
            for (int k = 1; k <= 2 * E; k++)
                for (int i = 2 * E; i >= k; i--) v[i] = (v[i] + p - v[i - 1]) % p;
            for (int k = 1; k <= E; k++)
                for (int i = E; i >= k; i--) w[i] = (w[i] + p - w[i - 1]) % p;
            for (int i = 0; i < 2 * E; i++) D[st][i] = v[i];
            for (int i = 0; i < E; i++) N[st][i] = mo.mul(w[i], mo.r2);   // x R
            Dc = v[2 * E]; Nc = mo.mul(w[E], mo.r2);
        }
    }
    #pragma unroll 1
    for (uint32_t i = 0; i < np; i += 4) {
        #pragma unroll
        for (int k = 0; k < 4; k++) {
            #pragma unroll
            for (int st = 0; st < S; st++) {
                if (LOOP == 0) {
                    const uint32_t u2 = mo.add(u[st], d1[st]);
                    if (E == 3) { d1[st] = mo.add(d1[st], d2[st]); d2[st] = mo.add(d2[st], 6); } else d1[st] += d2[st];
                    const uint32_t Nn = u[st] + u2;
                    const uint32_t Dd = mo.mul(u[st], u2);
                    u[st] = mo.add(u2, d1[st]);
                    if (E == 3) { d1[st] = mo.add(d1[st], d2[st]); d2[st] = mo.add(d2[st], 6); } else d1[st] += d2[st];
                    a1[st] = mo.mul2add(a1[st], Dd, a0[st], Nn);
                    a0[st] = mo.mul(a0[st], Dd);
                } else {
                    const uint32_t Dd = D[st][0], Nn = N[st][0];
                    a1[st] = mo.mul2add(a1[st], Dd, a0[st], Nn);
                    a0[st] = mo.mul(a0[st], Dd);
                    #pragma unroll
                    for (int q = 0; q < 2 * E - 1; q++) D[st][q] = mo.add(D[st][q], D[st][q + 1]);
                    D[st][2 * E - 1] = mo.add(D[st][2 * E - 1], Dc);
                    #pragma unroll
                    for (int q = 0; q < E - 1; q++) N[st][q] = mo.add(N[st][q], N[st][q + 1]);
                    N[st][E - 1] = mo.add(N[st][E - 1], Nc);
                }
            }
        }
    }
    uint32_t x = 0;
    for (int st = 0; st < S; st++) x ^= a0[st] ^ a1[st];
    out[tid] = x;
    if (tid == 0) { out[0] = a0[0]; out[1] = mo.mul(a1[0], 1); }   // c0 (R-form), c1 (R-form): S = c1 / c0
}

static uint64_t powm(uint64_t a, uint64_t e, uint64_t p) {
    unsigned __int128 r = 1, b = a % p;
    while (e) { if (e & 1) r = r * b % p; b = b * b % p; e >>= 1; }
    return (uint64_t)r;
}

template <int LOOP, int MUL, int E, int S>
void run(const char *name, int sms, int bps) {
    const uint32_t p = 2999999u;      // C2-size prime (< 2^22)
    const uint32_t np = 1 << 14, s0 = 12345;
    const int blocks = sms * bps, threads = 256;
    uint32_t *out;
    cudaMalloc(&out, (size_t)blocks * threads * 4);
    float best = 1e30f;
    for (int rep = 0; rep < 4; rep++) {
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        pair_loop<LOOP, MUL, E, S><<<blocks, threads>>>(p, np, s0, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep && ms < best) best = ms;
    }
    uint32_t h[2];
    cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
    // reference: sum_{s0 <= s < s0 + 2 np} s^-E mod p
    uint64_t ref = 0;
    for (uint64_t s = s0; s < s0 + 2ull * np; s++) ref = (ref + powm(powm(s, E, p), p - 2, p)) % p;
    const uint64_t got = (uint64_t)h[1] % p * powm(h[0] % p, p - 2, p) % p;
    const double terms = 2.0 * S * blocks * threads * np;
    printf("%-34s %7.3f ms  %.3e terms/s  %5.2f terms/clk/SM @1.965GHz  %s\n", name, best, terms / (best * 1e-3),
           terms / (best * 1e-3) / sms / 1.965e9, got == ref ? "ok" : "MISMATCH");
    cudaFree(out);
}


// LOOP 2: K-tuples: D = prod_{i<K} (s+i)^E, N = sum_i prod_{j!=i} (s+j)^E (degrees K E and (K-1) E), step K.
template <int E, int K>
__host__ __device__ __forceinline__ void polyDN(uint64_t x, uint32_t p, uint32_t &D, uint32_t &N) {
    uint64_t u[K];
    for (int i = 0; i < K; i++) { uint64_t a = (x + i) % p, r = a; for (int k = 1; k < E; k++) r = r * a % p; u[i] = r; }
    uint64_t d = 1; for (int i = 0; i < K; i++) d = d * u[i] % p;
    uint64_t n = 0;
    for (int i = 0; i < K; i++) { uint64_t t = 1; for (int j = 0; j < K; j++) if (j != i) t = t * u[j] % p; n = (n + t) % p; }
    D = (uint32_t)d; N = (uint32_t)n;
}

template <int MUL, int E, int K>
__global__ void __launch_bounds__(256) tuple_loop(uint32_t p, uint32_t nt, uint32_t s0base, uint32_t *out) {
    constexpr int DD = K * E, DN = (K - 1) * E;
    M32<MUL> mo;
    mo.init(p);
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t s = tid == 0 ? s0base : (s0base + 977u * tid) % (p - K * nt - 8) + 1;
    uint32_t D[DD + 1], N[DN + 1];
    {
        uint32_t v[DD + 1], w[DD + 1];
        for (int i = 0; i <= DD; i++) polyDN<E, K>(s + (uint64_t)K * i, p, v[i], w[i]);
        for (int k = 1; k <= DD; k++) for (int i = DD; i >= k; i--) v[i] = (v[i] + p - v[i - 1]) % p;
        for (int k = 1; k <= DN; k++) for (int i = DN; i >= k; i--) w[i] = (w[i] + p - w[i - 1]) % p;
        for (int i = 0; i <= DD; i++) D[i] = v[i];
        for (int i = 0; i <= DN; i++) N[i] = mo.mul(w[i], mo.r2);
    }
    uint32_t a0 = mo.r1, a1 = 0;
    #pragma unroll 1
    for (uint32_t i = 0; i < nt; i += 4) {
        #pragma unroll
        for (int k = 0; k < 4; k++) {
            a1 = mo.mul2add(a1, D[0], a0, N[0]);
            a0 = mo.mul(a0, D[0]);
            #pragma unroll
            for (int q = 0; q < DD; q++) D[q] = mo.add(D[q], D[q + 1]);
            #pragma unroll
            for (int q = 0; q < DN; q++) N[q] = mo.add(N[q], N[q + 1]);
        }
    }
    out[tid] = a0 ^ a1;
    if (tid == 0) { out[0] = a0; out[1] = mo.mul(a1, 1); }
}

template <int MUL, int E, int K>
void run_tuple(const char *name, int sms, int bps) {
    const uint32_t p = 2999999u;
    const uint32_t nt = 1 << 13, s0 = 12345;
    const int blocks = sms * bps, threads = 256;
    uint32_t *out;
    cudaMalloc(&out, (size_t)blocks * threads * 4);
    float best = 1e30f;
    for (int rep = 0; rep < 4; rep++) {
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        tuple_loop<MUL, E, K><<<blocks, threads>>>(p, nt, s0, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep && ms < best) best = ms;
    }
    uint32_t h[2];
    cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
    uint64_t ref = 0;
    for (uint64_t x = s0; x < s0 + (uint64_t)K * nt; x++) ref = (ref + powm(powm(x, E, p), p - 2, p)) % p;
    const uint64_t got = (uint64_t)h[1] % p * powm(h[0] % p, p - 2, p) % p;
    const double terms = (double)K * blocks * threads * nt;
    printf("%-34s %7.3f ms  %.3e terms/s  %5.2f terms/clk/SM @1.965GHz  %s\n", name, best, terms / (best * 1e-3),
           terms / (best * 1e-3) / sms / 1.965e9, got == ref ? "ok" : "MISMATCH");
    cudaFree(out);
}

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    const int sms = prop.multiProcessorCount;
    printf("%s, %d SMs\n", prop.name, sms);
    for (int bps = 4; bps <= 4; bps += 2) {
        run_tuple<2, 2, 2>("tuple K=2 sub E=2", sms, bps);
        run_tuple<2, 2, 3>("tuple K=3 sub E=2", sms, bps);
        run_tuple<2, 2, 4>("tuple K=4 sub E=2", sms, bps);
        run_tuple<2, 3, 2>("tuple K=2 sub E=3", sms, bps);
        run_tuple<2, 3, 3>("tuple K=3 sub E=3", sms, bps);
        run_tuple<2, 3, 4>("tuple K=4 sub E=3", sms, bps);
    }
    for (int bps = 2; bps <= 4; bps += 2) {
        printf("-- %d blocks of 256 per SM\n", bps);
        run<0, 0, 2, 1>("step2    C   E=2 S=1", sms, bps);
        run<0, 2, 2, 1>("step2    sub E=2 S=1", sms, bps);
        run<1, 0, 2, 1>("polypair C   E=2 S=1", sms, bps);
        run<1, 1, 2, 1>("polypair PTX E=2 S=1", sms, bps);
        run<1, 2, 2, 1>("polypair sub E=2 S=1", sms, bps);
        run<1, 2, 2, 2>("polypair sub E=2 S=2", sms, bps);
        run<0, 0, 3, 1>("step2    C   E=3 S=1", sms, bps);
        run<0, 2, 3, 1>("step2    sub E=3 S=1", sms, bps);
        run<1, 0, 3, 1>("polypair C   E=3 S=1", sms, bps);
        run<1, 2, 3, 1>("polypair sub E=3 S=1", sms, bps);
        run<1, 2, 3, 2>("polypair sub E=3 S=2", sms, bps);
        run<0, 3, 2, 1>("step2    alu E=2 S=1", sms, bps);
        run<1, 3, 2, 1>("polypair alu E=2 S=1", sms, bps);
        run<0, 3, 3, 1>("step2    alu E=3 S=1", sms, bps);
        run<1, 3, 3, 1>("polypair alu E=3 S=1", sms, bps);
        run<0, 4, 2, 1>("step2    alu4 E=2 S=1", sms, bps);
        run<1, 4, 2, 1>("polypair alu4 E=2 S=1", sms, bps);
        run<0, 4, 3, 1>("step2    alu4 E=3 S=1", sms, bps);
        run<1, 4, 3, 1>("polypair alu4 E=3 S=1", sms, bps);
    }
    return 0;
}
