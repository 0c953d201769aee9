// Microbenchmark: FFMA2 throughput vs register-operand pattern (register-file
// bandwidth hypothesis for the correlator's MAC). Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 f2(float2 a, float b, float2 c) {
    float2 d;
    asm volatile("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %4};\n\t"
        "mov.b64 rc, {%5, %6};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b), "f"(c.x), "f"(c.y));
    return d;
}

constexpr int IT = 2048;

// P1: 8 z pairs, each used by 1 FFMA2 (z, E and acc all fresh reads)
__global__ void p1(float* out, float s) {
    float2 z[8], A[8]; float e[8];
    for (int i = 0; i < 8; ++i) { z[i] = make_float2(threadIdx.x * 1e-3f + i, s + i); A[i] = make_float2(0, 0); e[i] = s * i + threadIdx.x * 1e-6f; }
    for (int it = 0; it < IT; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) A[i] = f2(z[i], e[i], A[i]);
    }
    float t = 0; for (int i = 0; i < 8; ++i) t += A[i].x + A[i].y;
    if (t == 1234.5f) out[0] = t;
}
// P2: 4 z pairs, each used by 2 consecutive FFMA2 (A/B: the current correlator)
__global__ void p2(float* out, float s) {
    float2 z[4], A[4], B[4]; float er[4], ei[4];
    for (int i = 0; i < 4; ++i) { z[i] = make_float2(threadIdx.x * 1e-3f + i, s + i); A[i] = B[i] = make_float2(0, 0); er[i] = s * i + threadIdx.x * 1e-6f; ei[i] = s + i + threadIdx.x * 2e-6f; }
    for (int it = 0; it < IT; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i) { A[i] = f2(z[i], er[i], A[i]); B[i] = f2(z[i], ei[i], B[i]); }
    }
    float t = 0; for (int i = 0; i < 4; ++i) t += A[i].x + A[i].y + B[i].x + B[i].y;
    if (t == 1234.5f) out[0] = t;
}
// P3: 2 z pairs, each used by 4 consecutive FFMA2 (two candidates per lane)
__global__ void p3(float* out, float s) {
    float2 z[2], A[4], B[4]; float er[4], ei[4];
    for (int i = 0; i < 2; ++i) z[i] = make_float2(threadIdx.x * 1e-3f + i, s + i);
    for (int i = 0; i < 4; ++i) { A[i] = B[i] = make_float2(0, 0); er[i] = s * i + threadIdx.x * 1e-6f; ei[i] = s + i + threadIdx.x * 2e-6f; }
    for (int it = 0; it < IT; ++it) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            A[2*i] = f2(z[i], er[2*i], A[2*i]); B[2*i] = f2(z[i], ei[2*i], B[2*i]);
            A[2*i+1] = f2(z[i], er[2*i+1], A[2*i+1]); B[2*i+1] = f2(z[i], ei[2*i+1], B[2*i+1]);
        }
    }
    float t = 0; for (int i = 0; i < 4; ++i) t += A[i].x + A[i].y + B[i].x + B[i].y;
    if (t == 1234.5f) out[0] = t;
}

template <class K>
float run(K k, float* out, int blocks, int threads) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a); k<<<blocks, threads>>>(out, 0.999f); cudaEventRecord(b);
        cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (r && ms < best) best = ms;
    }
    return best;
}

int main() {
    float* out; cudaMalloc(&out, 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int occ : {4, 8, 16}) {
        const int blocks = sms * occ, threads = 128;  // occ x 4 warps per SM
        const double ffma2 = 8.0 * IT * blocks * threads;  // FFMA2 per kernel (8 per iteration)
        for (auto [name, k] : {std::pair{"P1 fresh z per FFMA2 ", p1}, std::pair{"P2 z shared by 2     ", p2},
                               std::pair{"P3 z shared by 4     ", p3}}) {
            float ms = run(k, out, blocks, threads);
            printf("warps/SM %3d  %s  %.1f TFLOP/s (FP32, 4 FLOP per FFMA2)\n", occ * 4, name,
                   4.0 * ffma2 / (ms * 1e-3) / 1e12);
        }
    }
    return 0;
}
