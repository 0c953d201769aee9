// FP32 CUDA-core peak probe: the roofline denominator for the correlator
// (MEASURED_PEAKS.json carries HBM and bf16 tensor peaks only). Independent
// FFMA chains with register operands at full occupancy, timed with events.
#include <cuda_runtime.h>

#include "b200geo.h"

namespace {

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void __launch_bounds__(256) k_ffma_peak(float* out, float b, float c) {
    float a[kChains];
#pragma unroll
    for (int i = 0; i < kChains; ++i) a[i] = threadIdx.x * 1e-7f + i;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) a[i] = fmaf(a[i], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < kChains; ++i) s += a[i];
    if (s == 12345.678f) out[0] = s;  // keep the chains alive
}

__global__ void __launch_bounds__(256) k_ffma2_peak(float* out, float b, float c) {
    unsigned long long a[kChains];
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
        const float lo = threadIdx.x * 1e-7f + i, hi = lo + 0.5f;
        asm("mov.b64 %0, {%1, %2};" : "=l"(a[i]) : "f"(lo), "f"(hi));
    }
    unsigned long long bb, cc;
    asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
    asm("mov.b64 %0, {%1, %1};" : "=l"(cc) : "f"(c));
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i)
            asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(bb), "l"(cc));
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[i]));
        s += lo + hi;
    }
    if (s == 12345.678f) out[0] = s;
}

__global__ void __launch_bounds__(256) k_dfma_peak(float* out, float bf, float cf) {
    const double b = bf, c = cf;
    double a[kChains];
#pragma unroll
    for (int i = 0; i < kChains; ++i) a[i] = threadIdx.x * 1e-7 + i;
    for (int it = 0; it < kIters / 8; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) a[i] = fma(a[i], b, c);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kChains; ++i) s += a[i];
    if (s == 12345.678) out[0] = (float)s;
}

template <class K>
double time_probe(K kernel, int blocks, int threads, float* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(e0);
        kernel<<<blocks, threads>>>(out, 0.999999f, 1e-7f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return best;
}

}  // namespace

/* FP32 TFLOP/s issued as packed FFMA2 (fma.rn.f32x2): tells whether the paired
 * form raises the FP32 ceiling or only saves issue slots. */
extern "C" int dg_fp32x2_peak_tflops(int device, double* tflops) {
    if (!tflops) return DG_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return DG_ERUNTIME;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    float* out = nullptr;
    if (cudaMalloc(&out, sizeof(float)) != cudaSuccess) return DG_ENOMEM;
    const int blocks = sms * 8, threads = 256;
    const double ms = time_probe(k_ffma2_peak, blocks, threads, out);
    const cudaError_t err = cudaGetLastError();
    cudaFree(out);
    if (err != cudaSuccess) return DG_ERUNTIME;
    *tflops = 4.0 * kChains * (double)kIters * blocks * threads / (ms * 1e-3) / 1e12;
    return DG_OK;
}

extern "C" int dg_fp32_peak_tflops(int device, double* tflops) {
    if (!tflops) return DG_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return DG_ERUNTIME;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    float* out = nullptr;
    if (cudaMalloc(&out, sizeof(float)) != cudaSuccess) return DG_ENOMEM;
    const int blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(e0);
        k_ffma_peak<<<blocks, threads>>>(out, 0.999999f, 1e-7f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
    }
    const cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (err != cudaSuccess) return DG_ERUNTIME;
    const double flops = 2.0 * kChains * (double)kIters * blocks * threads;
    *tflops = flops / (best * 1e-3) / 1e12;
    return DG_OK;
}

/* FP64 TFLOP/s of independent DFMA chains: the ceiling of the exact geometry,
 * refinement and re-rank kernels. */
extern "C" int dg_fp64_peak_tflops(int device, double* tflops) {
    if (!tflops) return DG_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return DG_ERUNTIME;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    float* out = nullptr;
    if (cudaMalloc(&out, sizeof(float)) != cudaSuccess) return DG_ENOMEM;
    const int blocks = sms * 8, threads = 256;
    const double ms = time_probe(k_dfma_peak, blocks, threads, out);
    const cudaError_t err = cudaGetLastError();
    cudaFree(out);
    if (err != cudaSuccess) return DG_ERUNTIME;
    *tflops = 2.0 * kChains * (double)(kIters / 8) * blocks * threads / (ms * 1e-3) / 1e12;
    return DG_OK;
}
