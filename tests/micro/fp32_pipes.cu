// Microbenchmark: FMA-pipe issue cost of the FP32 instruction forms the
// moment kernel mixes (3-register FFMA / FMUL / FADD vs their packed FP32x2
// forms). Not part of the product; informs k_moments' instruction mix.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp32_pipes fp32_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int IT = 4096;
constexpr int CH = 8;  // independent chains per thread

__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float sum2(unsigned long long r) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
    return a + b;
}

// per-thread distinct registers for every operand (no immediates / constants)
#define SETUP                                                      \
    float b[CH], c[CH], a[CH];                                     \
    for (int i = 0; i < CH; ++i) {                                 \
        a[i] = threadIdx.x * 1e-7f + i;                            \
        b[i] = s + threadIdx.x * 1e-9f * i;                        \
        c[i] = 1e-7f * (i + 1) + threadIdx.x * 1e-12f;             \
    }
#define FINISH                                  \
    float t = 0.f;                              \
    for (int i = 0; i < CH; ++i) t += a[i];     \
    if (t == 1234.5f) out[0] = t;

__global__ void k_ffma(float* out, float s) {
    SETUP
    for (int it = 0; it < IT; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) a[i] = fmaf(a[i], b[i], c[i]);
    FINISH
}
__global__ void k_fmul(float* out, float s) {
    SETUP
    for (int it = 0; it < IT; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) a[i] = __fmul_rn(a[i], b[i]);
    FINISH
}
__global__ void k_fadd(float* out, float s) {
    SETUP
    for (int it = 0; it < IT; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) a[i] = __fadd_rn(a[i], b[i]);
    FINISH
}
__global__ void k_ffma2(float* out, float s) {
    SETUP
    unsigned long long A[CH], B[CH], C[CH];
    for (int i = 0; i < CH; ++i) { A[i] = pk(a[i], a[i] + 1.f); B[i] = pk(b[i], b[i]); C[i] = pk(c[i], c[i] * 2.f); }
    for (int it = 0; it < IT; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(A[i]) : "l"(B[i]), "l"(C[i]));
    for (int i = 0; i < CH; ++i) a[i] = sum2(A[i]);
    FINISH
}
__global__ void k_fadd2(float* out, float s) {
    SETUP
    unsigned long long A[CH], B[CH];
    for (int i = 0; i < CH; ++i) { A[i] = pk(a[i], a[i] + 1.f); B[i] = pk(b[i], b[i]); }
    for (int it = 0; it < IT; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(A[i]) : "l"(B[i]));
    for (int i = 0; i < CH; ++i) a[i] = sum2(A[i]);
    FINISH
}
__global__ void k_fmul2(float* out, float s) {
    SETUP
    unsigned long long A[CH], B[CH];
    for (int i = 0; i < CH; ++i) { A[i] = pk(a[i], a[i] + 1.f); B[i] = pk(b[i], b[i]); }
    for (int it = 0; it < IT; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(A[i]) : "l"(B[i]));
    for (int i = 0; i < CH; ++i) a[i] = sum2(A[i]);
    FINISH
}
// 1 FFMA2 + 1 scalar FFMA interleaved
__global__ void k_mix(float* out, float s) {
    SETUP
    unsigned long long A[CH], B[CH], C[CH];
    for (int i = 0; i < CH; ++i) { A[i] = pk(a[i], a[i] + 1.f); B[i] = pk(b[i], b[i]); C[i] = pk(c[i], c[i] * 2.f); }
    for (int it = 0; it < IT; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(A[i]) : "l"(B[i]), "l"(C[i]));
            a[i] = fmaf(a[i], b[i], c[i]);
        }
    for (int i = 0; i < CH; ++i) a[i] += sum2(A[i]);
    FINISH
}
// FFMA2 + integer/ALU op interleaved (does ALU co-issue for free?)
__global__ void k_ffma_alu(float* out, float s) {
    SETUP
    int x[CH];
    for (int i = 0; i < CH; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < IT; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            a[i] = fmaf(a[i], b[i], c[i]);
            x[i] = (x[i] ^ (x[i] >> 3)) + i;
        }
    for (int i = 0; i < CH; ++i) a[i] += (float)x[i];
    FINISH
}

template <class K>
float run(K k, float* out, int blocks, int threads) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k<<<blocks, threads>>>(out, 0.999f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r && ms < best) best = ms;
    }
    return best;
}

int main() {
    float* out;
    cudaMalloc(&out, 4);
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = sms * 8, threads = 256;
    const double warp_instr = (double)IT * CH * blocks * threads / 32;
    struct {
        const char* name;
        void (*k)(float*, float);
        double instr_per_chain;  // warp instructions per (it, chain)
    } tests[] = {{"FFMA 3-reg", k_ffma, 1},   {"FMUL 2-reg", k_fmul, 1}, {"FADD 2-reg", k_fadd, 1},
                 {"FFMA2", k_ffma2, 1},        {"FADD2", k_fadd2, 1},     {"FMUL2", k_fmul2, 1},     {"FFMA2+FFMA", k_mix, 2},
                 {"FFMA+ALU(3)", k_ffma_alu, 4}};
    for (auto& t : tests) {
        const float ms = run(t.k, out, blocks, threads);
        const double cyc = ms * 1e-3 * clk * 1e3;  // SM clock cycles (nominal)
        const double per_smsp = warp_instr * t.instr_per_chain / (sms * 4);
        printf("%-14s %8.3f ms  %.2f warp-instr/clk/SMSP  (cycles per warp-instr %.2f)\n", t.name, ms,
               per_smsp / cyc, cyc / per_smsp);
    }
    return 0;
}
