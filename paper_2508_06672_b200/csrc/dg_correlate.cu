// K3: the correlator — Eq. 11 (reference correlate.hpp:44-71) on CUDA cores.
//
// One warp = one task = up to 32 candidates sharing one integer TDOA d (the
// d-bucketing in dg_kernels.cu), so the product stream
//     z[k] = y1[k] conj(y2[k+d]),   k in [max(0,-d), min(N, N-d))
// and the overlap range are common to all 32 lanes; each lane is one
// candidate with its own FDOA f (cycles/sample) and evaluates
//     S = | sum_k z[k] e^{j 2 pi f k} |.
//
// Per 256-sample chunk:
//   1. TMA: one lane issues two 1-D bulk copies (cp.async.bulk + mbarrier
//      complete_tx) of y1[c0..] and y2[c0+d..] for the NEXT chunk into the
//      warp's other shared-memory buffer (double buffering, no registers).
//   2. The warp forms z for this chunk from shared memory once (8 samples
//      per lane) and stores it to the warp's z buffer.
//   3. Every lane accumulates  A += z * Er[j],  B += z * Ei[j]  with packed
//      FP32x2 FMAs (FFMA2: z pair from one broadcast LDS.128 covering two
//      samples, the phasor-table entry as a broadcast scalar operand), so
//      per block of 16 samples  C = sum_j z E[j] = (A.x - B.y, A.y + B.x).
//      C is rotated by W_b = e^{j 2 pi f (c0 + 16 b)} (one complex multiply
//      per 16 samples, re-anchored every chunk from an FP64-reduced phase)
//      and summed; chunk sums are accumulated in FP64.
// Cost per sample per candidate: 2 FFMA2 + 1/2 LDS.128 + ~0.6 scalar FP32 for
// the block rotation + ~0.2 shared (z production, anchor) instructions.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "dg_internal.cuh"

namespace dg {

namespace {

constexpr int kYPad = 8;  // extra samples per y2 staging buffer (parity shift + slack)

__device__ __forceinline__ float2 ffma2(float2 a, float b, float2 c) {
    float2 d;
    asm("{.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\t"
        "mov.b64 rb, {%4, %4};\n\t"
        "mov.b64 rc, {%5, %6};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\t"
        "mov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b), "f"(c.x), "f"(c.y));
    return d;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// 1-D bulk copy global -> shared (TMA engine), completion on `bar`
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <int kCh>
struct alignas(16) WarpSmemT {
    float2 y1[2][kCh];          // staged y1[c0 .. c0+kCh); z overwrites it in place
    float2 y2[2][kCh + kYPad];  // staged y2[(c0+d)&~1 ..)
    uint64_t bar[2];
    uint64_t pad;
};

}  // namespace

// LB: phasor-table length (samples per block); CH: samples per staged chunk.
template <int LB, int CH>
__global__ void __launch_bounds__(32 * kWarpsPerCta, 2)
k_correlate(const Task* __restrict__ tasks, const int* __restrict__ n_tasks,
            const int* __restrict__ sorted, const double* __restrict__ fdoa,
            const float2* __restrict__ y1, const float2* __restrict__ y2, int N, double fs,
            double* __restrict__ s_out, uint32_t* __restrict__ flag_bits, int64_t flag_base) {
    using WarpSmem = WarpSmemT<CH>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpSmem& ws = reinterpret_cast<WarpSmem*>(smem_raw)[warp];
    const int t = blockIdx.x * kWarpsPerCta + warp;
    if (t >= *n_tasks) return;
    const Task tk = tasks[t];
    const int d = tk.d;
    const int p = lane < tk.count ? sorted[tk.start + lane] : -1;
    const double f = p >= 0 ? fdoa[p] / fs : 0.0;  // cycles per sample

    const int kb = d < 0 ? -d : 0;
    const int ke = (N - d) < N ? (N - d) : N;
    const int kb0 = kb & ~1;  // even chunk origin: 16-byte aligned y1
    const int n_chunks = (ke - kb0 + CH - 1) / CH;
    const int shift = (kb0 + d) & 1;  // y2 staging starts at the even index below c0+d
    constexpr uint32_t kY1Bytes = CH * sizeof(float2);
    constexpr uint32_t kY2Bytes = (CH + 2) * sizeof(float2);

    if (lane == 0) {
        mbar_init(&ws.bar[0], 1);
        mbar_init(&ws.bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto issue = [&](int c, int buf) {
        const int c0 = kb0 + c * CH;
        mbar_expect_tx(&ws.bar[buf], kY1Bytes + kY2Bytes);
        tma_load_1d(ws.y1[buf], y1 + c0, kY1Bytes, &ws.bar[buf]);
        tma_load_1d(ws.y2[buf], y2 + (c0 + d - shift), kY2Bytes, &ws.bar[buf]);
    };
    if (lane == 0) issue(0, 0);

    // phasor table E[j] = e^{j 2 pi f j} and the block step W1 = e^{j 2 pi f LB},
    // FP64 range reduction, then single-precision sincospi of the fraction
    float er[LB], ei[LB];
#pragma unroll
    for (int j = 0; j < LB; ++j) {
        const double x = f * (double)j;
        sincospif((float)(2.0 * (x - rint(x))), &ei[j], &er[j]);
    }
    float w1r, w1i;
    {
        const double x = f * (double)LB;
        sincospif((float)(2.0 * (x - rint(x))), &w1i, &w1r);
    }

    double acc_re = 0.0, acc_im = 0.0;
    float z2 = 0.f;
    for (int c = 0; c < n_chunks; ++c) {
        const int buf = c & 1;
        const int c0 = kb0 + c * CH;
        if (lane == 0 && c + 1 < n_chunks) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(c + 1, buf ^ 1);
        }
        mbar_wait(&ws.bar[buf], (c >> 1) & 1);

        // ---- z = y1 conj(y2), zero outside [kb, ke); written over y1 in place ----
        float4* zq = reinterpret_cast<float4*>(ws.y1[buf]);
        const float2* s2 = ws.y2[buf] + shift;
#pragma unroll
        for (int i = 0; i < CH / 64; ++i) {
            const int q = lane + 32 * i;
            const int k = c0 + 2 * q;
            const float4 a = zq[q];
            const float2 b0 = s2[2 * q], b1 = s2[2 * q + 1];
            const bool v0 = k >= kb && k < ke, v1 = k + 1 >= kb && k + 1 < ke;
            float4 zz;
            zz.x = v0 ? fmaf(a.x, b0.x, a.y * b0.y) : 0.f;
            zz.y = v0 ? fmaf(a.y, b0.x, -(a.x * b0.y)) : 0.f;
            zz.z = v1 ? fmaf(a.z, b1.x, a.w * b1.y) : 0.f;
            zz.w = v1 ? fmaf(a.w, b1.x, -(a.z * b1.y)) : 0.f;
            z2 = fmaf(zz.x, zz.x, fmaf(zz.y, zz.y, fmaf(zz.z, zz.z, fmaf(zz.w, zz.w, z2))));
            zq[q] = zz;
        }
        __syncwarp();

        // ---- blocks in reverse, Horner: H = (((C_last) W1 + C_last-1) W1 + ...) ----
        //      chunk sum = W(c0) * H,  C_b = sum_j z[c0 + LB b + j] E[j]
        float hr = 0.f, hi = 0.f;
#pragma unroll
        for (int b = CH / LB - 1; b >= 0; --b) {
            float2 A0 = make_float2(0.f, 0.f), B0 = A0, A1 = A0, B1 = A0;
#pragma unroll
            for (int j = 0; j < LB; j += 4) {
                const float4 za = zq[(b * LB + j) >> 1];
                const float4 zb = zq[(b * LB + j + 2) >> 1];
                A0 = ffma2(make_float2(za.x, za.y), er[j], A0);
                B0 = ffma2(make_float2(za.x, za.y), ei[j], B0);
                A1 = ffma2(make_float2(za.z, za.w), er[j + 1], A1);
                B1 = ffma2(make_float2(za.z, za.w), ei[j + 1], B1);
                A0 = ffma2(make_float2(zb.x, zb.y), er[j + 2], A0);
                B0 = ffma2(make_float2(zb.x, zb.y), ei[j + 2], B0);
                A1 = ffma2(make_float2(zb.z, zb.w), er[j + 3], A1);
                B1 = ffma2(make_float2(zb.z, zb.w), ei[j + 3], B1);
            }
            // C = A + jB with A = A0 + A1, B = B0 + B1
            const float cr = (A0.x + A1.x) - (B0.y + B1.y);
            const float ci = (A0.y + A1.y) + (B0.x + B1.x);
            const float nr = fmaf(hr, w1r, fmaf(-hi, w1i, cr));
            hi = fmaf(hr, w1i, fmaf(hi, w1r, ci));
            hr = nr;
        }
        // anchor W = e^{j 2 pi f c0} from the FP64-reduced phase
        float wr, wi;
        {
            const double x = f * (double)c0;
            sincospif((float)(2.0 * (x - rint(x))), &wi, &wr);
        }
        acc_re += (double)fmaf(wr, hr, -(wi * hi));
        acc_im += (double)fmaf(wr, hi, wi * hr);
        __syncwarp();  // this stage's buffers are free for the next bulk copy
    }

#pragma unroll
    for (int o = 16; o; o >>= 1) z2 += __shfl_xor_sync(0xffffffffu, z2, o);
    if (p >= 0) {
        const double s = sqrt(acc_re * acc_re + acc_im * acc_im);
        s_out[p] = s;
        if (s < (double)kRefineTau * sqrt((double)z2)) {
            const int64_t e = flag_base + p;
            atomicOr(&flag_bits[e >> 5], 1u << (e & 31));
        }
    }
}

namespace {

template <int LB, int CH>
void launch_variant(int blocks, cudaStream_t st, const Task* tasks, const int* n_tasks,
                    const int* sorted, const double* fdoa, const float2* y1, const float2* y2,
                    int N, double fs, double* s_out, uint32_t* flag_bits, int64_t flag_base) {
    const size_t smem = sizeof(WarpSmemT<CH>) * kWarpsPerCta;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_correlate<LB, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attr_set = true;
    }
    k_correlate<LB, CH><<<blocks, 32 * kWarpsPerCta, smem, st>>>(
        tasks, n_tasks, sorted, fdoa, y1, y2, N, fs, s_out, flag_bits, flag_base);
}

int variant_from_env() {
    const char* v = getenv("DG_CORRELATE_VARIANT");
    return v ? atoi(v) : 0;
}

}  // namespace

void launch_correlate(const Task* tasks, const int* n_tasks, int max_tasks, const int* sorted,
                      const double* fdoa, const float2* y1, const float2* y2, int N, double fs,
                      double* s_out, uint32_t* flag_bits, int64_t flag_base, cudaStream_t st) {
    const int blocks = (max_tasks + kWarpsPerCta - 1) / kWarpsPerCta;
    if (blocks <= 0) return;
    static const int variant = variant_from_env();
    switch (variant) {
        case 1:
            launch_variant<32, 256>(blocks, st, tasks, n_tasks, sorted, fdoa, y1, y2, N, fs, s_out,
                                    flag_bits, flag_base);
            break;
        case 2:
            launch_variant<16, 512>(blocks, st, tasks, n_tasks, sorted, fdoa, y1, y2, N, fs, s_out,
                                    flag_bits, flag_base);
            break;
        default:
            launch_variant<16, 256>(blocks, st, tasks, n_tasks, sorted, fdoa, y1, y2, N, fs, s_out,
                                    flag_bits, flag_base);
    }
}

}  // namespace dg
