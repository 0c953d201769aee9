// K3 block moments as FFT cross-correlations (the k_moments alternative for
// B >= 256).
//
// For block b (y1 samples [bB, bB + B)) and moment m the moments of every TDOA
// value d are one cross-correlation:
//     M_m[b](d) = sum_{j<B} a_m[j] conj(y2[bB + j + d]),   a_m[j] = y1c[bB + j] T_m(t_j)
// (y1c zero past N and y2 zero outside [0, N) realise the overlap masks). For a
// window of G = L - B consecutive lags d0 .. d0 + G - 1 with s[n] = y2[bB + d0 + n],
// n < L = 1024, no circular wrap reaches the used lags, so
//     M_m[b](d0 + t) = conj( IFFT_L( conj(FFT_L(a_m)) . FFT_L(s) )[t] ) / L.
// Per (block, window) that is one forward FFT of s and R inverse FFTs, against
// the direct sums' G * B / 2 * R FP32x2 MACs: ~9x fewer operations at B = 512.
//   k_mfft     one persistent kernel, one warp per work unit from one queue:
//              first the (block, m) spectra conj(FFT(a_m)) / L (R * nblk warp
//              FFTs, published per block), then the (window, block) items: FFT of
//              s into the warp's shared buffer, then per m the pointwise product
//              and the inverse FFT, outputs written straight to the buckets' moment
//              rows (the layout k_evaluate_tc reads: [bucket][block][m], odd m x i)
//              It also records each (window, block, m) correlation's mean square:
//              FFT rounding spreads ~5e-7 of a window's RMS over all its lags, the
//              scale the refinement test needs.
//   k_fft_bucket_energy  one warp per bucket: those energies summed over the
//              bucket's blocks for k_evaluate_tc.
// FFTs: dg_fft.cuh (warp-level, FP32, ~5e-7 of the vector's RMS).
#include <cuda_runtime.h>
#include <stdint.h>

#include "dg_device.cuh"
#include "dg_fft.cuh"
#include "dg_internal.cuh"

namespace dg {

namespace {

constexpr int kFftL = kFftLen;
constexpr int kFftWarps = 8;  // warps per CTA (one CTA per SM: 8 x 24.4 KB of buffers)
constexpr int kXbuf = 32 * 33;
constexpr int kMaxLagsPerLane = 24;  // G / 32 for B >= 256

struct FftWarpSmem {
    float2 xbuf[kXbuf];   // transpose
    float2 sbuf[kFftL];   // FFT of the y2 window
    float2 abuf[kFftL];   // conj(FFT(a_m)) / L of the current moment (TMA-staged)
};
struct FftSmem {
    float2 tw[kFftL];
    FftWarpSmem w[kFftWarps];
    uint64_t bar[kFftWarps];
};

// one (block, moment) spectrum: conj(FFT(a_m)) / L, a_m[j] = y1c[bB + j] T_m(t_j)
// (tchebT: the Chebyshev table moment-major, one coalesced row per moment)
__device__ __forceinline__ void afft_unit(int b, int m, int lane, const float2* __restrict__ y1c,
                                          int N, int B, int R, const float* __restrict__ tchebT,
                                          const float2* tw, float2* xbuf, float2* __restrict__ af) {
    float2 v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const int j = lane + 32 * i;
        const int k = b * B + j;
        float2 a = make_float2(0.f, 0.f);
        if (j < B && k < N) {
            const float2 y = y1c[k];
            const float t = tchebT[m * B + j];
            a = make_float2(y.x * t, y.y * t);
        }
        v[i] = a;
    }
    fft1024_warp<false>(v, tw, xbuf, lane);
    float2* dst = af + ((size_t)b * R + m) * kFftL;
    constexpr float inv = 1.0f / kFftL;
#pragma unroll
    for (int i = 0; i < 32; ++i) dst[lane + 32 * i] = make_float2(v[i].x * inv, -v[i].y * inv);
}

__global__ void __launch_bounds__(32 * kFftWarps, 1)
k_mfft(const int* __restrict__ ubin, int bin0, int nbins, int ngroups, int G, int N, int B,
       int R, int nblk, const float2* __restrict__ y1c, const float* __restrict__ tchebT,
       float2* __restrict__ af, int* __restrict__ ready, const float2* __restrict__ y2p,
       int padf, float2* __restrict__ mom, int nbmax, float* __restrict__ fe,
       int* __restrict__ queue) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    FftSmem& sm = *reinterpret_cast<FftSmem*>(smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    fft1024_twiddles(sm.tw, threadIdx.x, blockDim.x);
    if (threadIdx.x < kFftWarps) mbar_init(&sm.bar[threadIdx.x], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    FftWarpSmem& ws = sm.w[warp];
    uint64_t* bar = &sm.bar[warp];
    uint32_t phase = 0;  // completed TMA copies of this warp
    // one queue: first the (block, moment) spectra (block-major), then the (window,
    // block) items; an item waits until its block's R spectra are published. Every
    // spectrum is claimed before any item, by a warp that never waits: no deadlock.
    const int nA = nblk * R;
    const int total = nA + ngroups * nblk;
    for (;;) {
        int it = 0;
        if (lane == 0) it = atomicAdd(queue, 1);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= total) break;
        if (it < nA) {
            const int b = it / R, m = it - b * R;
            afft_unit(b, m, lane, y1c, N, B, R, tchebT, sm.tw, ws.xbuf, af);
            __threadfence();  // the spectrum, then its publication
            __syncwarp();
            if (lane == 0) atomicAdd(&ready[b], 1);
            continue;
        }
        const int j = it - nA;
        const int g = j / nblk, b = j - g * nblk;
        if (lane == 0) {
            while (*reinterpret_cast<volatile int*>(&ready[b]) < R) __nanosleep(64);
            __threadfence();
            asm volatile("fence.proxy.async.global;" ::: "memory");  // read by TMA below
        }
        __syncwarp();
        // windows at absolute multiples of G, so any bin-range part of a step (the
        // multi-GPU work units) computes every moment with the same FFTs
        const int bin_a = (bin0 / G + g) * G;  // first bin of the window
        const int d0 = bin_a - (N - 1);
        const float2* afb = af + (size_t)b * R * kFftL;
        if (lane == 0) {  // moment 0's spectrum, in flight during the window's FFT
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bar, kFftL * sizeof(float2));
            tma_load_1d(ws.abuf, afb, kFftL * sizeof(float2), bar);
        }
        // s[n] = y2[bB + d0 + n], n < L (zero outside [0, N): the padded copy)
        float2 v[32];
        const float2* src = y2p + padf + (ptrdiff_t)b * B + d0;
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = src[lane + 32 * i];
        // this lane's lags t = lane + 32 k: moment-row offset of (bucket, block b)
        // or -1 (once per window, not per moment). No padding rows: k_evaluate_tc,
        // the only reader of FFT moments, stops at each bucket's nb
        int roff[kMaxLagsPerLane];
#pragma unroll
        for (int k = 0; k < kMaxLagsPerLane; ++k) {
            roff[k] = -1;
            const int t = lane + 32 * k;
            const int bin = bin_a + t;
            if (t < G && bin >= bin0 && bin < bin0 + nbins) {
                const int u = ubin[bin - bin0];
                if (u >= 0) {
                    const int d = bin - (N - 1);
                    const int kb = d < 0 ? -d : 0, ke = d > 0 ? N - d : N;
                    const int bf = kb / B, bl = (ke - 1) / B;
                    if (b >= bf && b <= bl) roff[k] = (u * nbmax + (b - bf)) * R;
                }
            }
        }
        fft1024_warp<false>(v, sm.tw, ws.xbuf, lane);
#pragma unroll
        for (int i = 0; i < 32; ++i) ws.sbuf[lane + 32 * i] = v[i];
        __syncwarp();
        // moments in pairs (R even): m's outputs wait in registers for m + 1's, then
        // one 16-byte store per lag and pair
        float2 keep[kMaxLagsPerLane];
        for (int m = 0; m < R; ++m) {
            mbar_wait(bar, phase & 1);
            ++phase;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const float2 p = ws.abuf[lane + 32 * i], q = ws.sbuf[lane + 32 * i];
                v[i] = make_float2(fmaf(p.x, q.x, -p.y * q.y), fmaf(p.x, q.y, p.y * q.x));
            }
            __syncwarp();
            if (lane == 0 && m + 1 < R) {  // the next moment's spectrum during this IFFT
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(bar, kFftL * sizeof(float2));
                tma_load_1d(ws.abuf, afb + (size_t)(m + 1) * kFftL, kFftL * sizeof(float2), bar);
            }
            fft1024_warp<true>(v, sm.tw, ws.xbuf, lane);
            {  // the window's mean square (all L outputs): the FFT rounding's scale
                float e = 0.f;
#pragma unroll
                for (int i = 0; i < 32; ++i) e = fmaf(v[i].x, v[i].x, fmaf(v[i].y, v[i].y, e));
#pragma unroll
                for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
                if (lane == 0) fe[((size_t)g * R + m) * nblk + b] = e * (1.0f / kFftL);
            }
            // M = conj(c); odd moments stored times i: i conj(c) = (c.y, c.x)
            if ((m & 1) == 0) {
#pragma unroll
                for (int k = 0; k < kMaxLagsPerLane; ++k) keep[k] = make_float2(v[k].x, -v[k].y);
            } else {
#pragma unroll
                for (int k = 0; k < kMaxLagsPerLane; ++k) {
                    if (roff[k] < 0) continue;
                    *reinterpret_cast<float4*>(mom + (size_t)roff[k] + m - 1) =
                        make_float4(keep[k].x, keep[k].y, v[k].y, v[k].x);
                }
            }
        }
    }
}

// one warp per bucket: qf[u][m] = sum_{b in the bucket's blocks} fe[window][m][b]
// (contiguous in b: coalesced; every moment's loads in flight together)
template <int R>
__global__ void k_fft_bucket_energy(const Bucket* __restrict__ buckets,
                                    const int* __restrict__ n_buckets, const float* __restrict__ fe,
                                    int bin0, int G, int nblk, int N, int B,
                                    float* __restrict__ qf) {
    const int lane = threadIdx.x & 31;
    const int nbk = *n_buckets;
    for (int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < nbk;
         u += (gridDim.x * blockDim.x) >> 5) {
        const Bucket bk = buckets[u];
        const int win = (bk.d + N - 1) / G - bin0 / G;
        const int bf = (bk.d < 0 ? -bk.d : 0) / B;
        const float* f = fe + (size_t)win * R * nblk + bf;
        float e[R];
#pragma unroll
        for (int m = 0; m < R; ++m) e[m] = 0.f;
        for (int b = lane; b < bk.nb; b += 32) {
#pragma unroll
            for (int m = 0; m < R; ++m) e[m] += f[(size_t)m * nblk + b];
        }
#pragma unroll
        for (int m = 0; m < R; ++m) {
#pragma unroll
            for (int o = 16; o; o >>= 1) e[m] += __shfl_xor_sync(0xffffffffu, e[m], o);
        }
        if (lane < R) {
            float v = 0.f;
#pragma unroll
            for (int m = 0; m < R; ++m) v = lane == m ? e[m] : v;
            qf[(size_t)u * kMaxMoments + lane] = v;
        }
    }
}

}  // namespace

void launch_fft_bucket_energy(const Bucket* buckets, const int* n_buckets, int max_buckets,
                              const float* fe, int bin0, int G, int nblk, int N, int B, int R,
                              float* qf, cudaStream_t st) {
    const int blocks = (max_buckets + 7) / 8;
    const int grid = blocks < 148 * 16 ? blocks : 148 * 16;
#define DG_FBE(RR)                                                                             \
    k_fft_bucket_energy<RR><<<grid, 256, 0, st>>>(buckets, n_buckets, fe, bin0, G, nblk, N, B, qf)
    switch (R) {
        case 8: DG_FBE(8); break;
        case 10: DG_FBE(10); break;
        case 12: DG_FBE(12); break;
        case 14: DG_FBE(14); break;
        default: DG_FBE(16); break;
    }
#undef DG_FBE
}

bool moments_fft_supported(int B) { return B >= 256 && B <= 768; }

size_t moments_fft_af_bytes(int N, int B, int R) {
    const int nblk = (N + B - 1) / B;
    return (size_t)nblk * R * kFftL * sizeof(float2);
}

size_t moments_fft_fe_floats(int N, int B, int R) {
    const int nblk = (N + B - 1) / B, G = kFftL - B;
    const int ngroups = (2 * N - 1 + G - 1) / G + 1;
    return (size_t)ngroups * nblk * R;
}

void launch_moments_fft(int B, int R, const int* ubin, int bin0, int nbins, int N,
                        const float* tchebT, const float2* y1c, const float2* y2p, int padf,
                        float2* mom, int nbmax, float2* af, float* fe, int* queue, int sm_count,
                        cudaStream_t st) {
    const int nblk = (N + B - 1) / B;
    const int G = kFftL - B;
    const int ngroups = (bin0 + nbins - 1) / G - bin0 / G + 1;  // absolute windows
    const size_t smem = sizeof(FftSmem);
    static size_t attr_m[64] = {};
    ensure_smem(k_mfft, smem, attr_m);
    // queue[0]: the work queue; queue[1 .. nblk]: published spectra per block
    cudaMemsetAsync(queue, 0, (size_t)(nblk + 1) * sizeof(int), st);
    k_mfft<<<sm_count, 32 * kFftWarps, smem, st>>>(ubin, bin0, nbins, ngroups, G, N, B, R, nblk,
                                                   y1c, tchebT, af, queue + 1, y2p, padf, mom,
                                                   nbmax, fe, queue);
}

}  // namespace dg
