// Check of the warp-level 1024-point FFT (csrc/dg_fft.cuh) against an FP64 DFT on
// the host: forward and inverse, max |error| relative to the vector's RMS.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2508_06672_b200/csrc \
//        -o /tmp/fft_check fft_check.cu
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "dg_fft.cuh"

template <bool INV>
__global__ void k_fft(const float2* in, float2* out, int nvec) {
    __shared__ float2 tw[1024];
    __shared__ float2 xb[4][32 * 33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    dg::fft1024_twiddles(tw, threadIdx.x, blockDim.x);
    __syncthreads();
    const int vec = blockIdx.x * 4 + warp;
    if (vec >= nvec) return;
    float2 v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = in[vec * 1024 + lane + 32 * i];
    dg::fft1024_warp<INV>(v, tw, xb[warp], lane);
#pragma unroll
    for (int i = 0; i < 32; ++i) out[vec * 1024 + lane + 32 * i] = v[i];
}

int main() {
    const int nvec = 8;
    std::vector<float2> h(nvec * 1024), o(nvec * 1024);
    srand(1);
    for (auto& x : h) x = make_float2(rand() / (float)RAND_MAX - 0.5f, rand() / (float)RAND_MAX - 0.5f);
    float2 *di, *dout;
    cudaMalloc(&di, h.size() * 8);
    cudaMalloc(&dout, h.size() * 8);
    cudaMemcpy(di, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    for (int inv = 0; inv < 2; ++inv) {
        if (inv)
            k_fft<true><<<(nvec + 3) / 4, 128>>>(di, dout, nvec);
        else
            k_fft<false><<<(nvec + 3) / 4, 128>>>(di, dout, nvec);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(o.data(), dout, o.size() * 8, cudaMemcpyDeviceToHost);
        double worst = 0;
        for (int v = 0; v < nvec; ++v) {
            double rms = 0, emax = 0;
            std::vector<std::complex<double>> X(1024);
            for (int k = 0; k < 1024; ++k) {
                std::complex<double> acc = 0;
                for (int n = 0; n < 1024; ++n) {
                    const double ang = (inv ? 2.0 : -2.0) * M_PI * (double)((long)n * k % 1024) / 1024.0;
                    acc += std::complex<double>(h[v * 1024 + n].x, h[v * 1024 + n].y) *
                           std::complex<double>(cos(ang), sin(ang));
                }
                X[k] = acc;
                rms += std::norm(acc);
            }
            rms = sqrt(rms / 1024);
            for (int k = 0; k < 1024; ++k)
                emax = fmax(emax, std::abs(X[k] - std::complex<double>(o[v * 1024 + k].x, o[v * 1024 + k].y)));
            worst = fmax(worst, emax / rms);
        }
        printf("%s: max |err| / rms = %.3e\n", inv ? "inverse" : "forward", worst);
    }
    return 0;
}
