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

#include "dg_device.cuh"
#include "dg_internal.cuh"

namespace dg {

namespace {

constexpr int kYPad = 8;  // extra samples per y2 staging buffer (parity shift + slack)

// e^{i 2 pi x} for an FP64 cycle count: FP64 range reduction and sincospi,
// one rounding to FP32 (<= 0.5 ulp): the phasor tables, block steps and chunk
// anchors carry no FP32 argument rounding, whose systematic phase error
// aliased into the block sums of strong off-TDOA chirp products
__device__ __forceinline__ void cis_f64(double x, float* c, float* s) {
    double sd, cd;
    sincospi(2.0 * (x - rint(x)), &sd, &cd);
    *c = (float)cd;
    *s = (float)sd;
}

template <int kCh>
struct alignas(16) WarpSmemT {
    float2 y1[2][kCh];          // staged y1[c0 .. c0+kCh); z overwrites it in place
    float2 y2[2][kCh + kYPad];  // staged y2[(c0+d)&~1 ..)
    uint64_t bar[2];
    uint64_t pad;
};

}  // namespace

// NC: candidates per lane (a warp task holds up to 32*NC candidates of one d);
// LB: phasor-table length (samples per block); CH: samples per staged chunk;
// WPC: warps per CTA; MINB: CTAs per SM the register budget is sized for.
template <int NC, int LB, int CH, int WPC, int MINB>
__global__ void __launch_bounds__(32 * WPC, MINB)
k_correlate(const Task* __restrict__ tasks, const int* __restrict__ n_tasks,
            const int* __restrict__ sorted, const double* __restrict__ fdoa,
            const float2* __restrict__ y1, const float2* __restrict__ y2, int N, double fs,
            double* __restrict__ s_out, uint32_t* __restrict__ flag_bits, int64_t flag_base,
            float tau) {
    using WarpSmem = WarpSmemT<CH>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpSmem& ws = reinterpret_cast<WarpSmem*>(smem_raw)[warp];
    const int t = blockIdx.x * WPC + warp;
    if (t >= *n_tasks) return;
    const Task tk = tasks[t];
    const int d = tk.d;
    int p[NC];
    double f[NC];  // cycles per sample
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const int slot = lane + 32 * c;
        p[c] = slot < tk.count ? sorted[tk.start + slot] : -1;
        f[c] = p[c] >= 0 ? fdoa[p[c]] / fs : 0.0;
    }

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

    // phasor tables E[j] = e^{j 2 pi f j} and block steps W1 = e^{j 2 pi f LB},
    // FP64 range reduction, then single-precision sincospi of the fraction
    float er[NC][LB], ei[NC][LB], w1r[NC], w1i[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
#pragma unroll
        for (int j = 0; j < LB; ++j) {
            const double x = f[c] * (double)j;
            cis_f64(x, &er[c][j], &ei[c][j]);
        }
        const double x = f[c] * (double)LB;
        cis_f64(x, &w1r[c], &w1i[c]);
    }

    // this candidate's FP32 error scale: the block sums round relative to the
    // blocks (eb = sum_b |C_b|^2), the Horner chunk sums relative to the chunks
    // (e2 = sum_c |chunk sum|^2), the phasor tables' rounding relative to the
    // samples (z2 = ||z||_2^2, shared by the warp). For noise all three are
    // ||z||_2^2; a tone at the candidate's frequency makes the chunk term CH/LB x
    // larger, a chirp off its TDOA (coherent within blocks, not within chunks)
    // the block term, and a product tone that aliases onto the block length
    // (block sums cancel, the tables' systematic errors add up) needs the floor.
    double acc_re[NC], acc_im[NC], e2[NC], eb[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc_re[c] = acc_im[c] = e2[c] = eb[c] = 0.0;
    float z2 = 0.f;
    for (int ch = 0; ch < n_chunks; ++ch) {
        const int buf = ch & 1;
        const int c0 = kb0 + ch * CH;
        if (lane == 0 && ch + 1 < n_chunks) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(ch + 1, buf ^ 1);
        }
        mbar_wait(&ws.bar[buf], (ch >> 1) & 1);

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
        float hr[NC], hi[NC], bq[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) hr[c] = hi[c] = bq[c] = 0.f;
        constexpr int QB = LB / 2;        // z quads (2 samples each) per block
        constexpr int NB = CH / LB;       // blocks per chunk
        float4 znext = zq[(NB - 1) * QB];  // rolling one-quad-ahead prefetch
#pragma unroll
        for (int b = NB - 1; b >= 0; --b) {
            float2 A[NC], B[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) A[c] = B[c] = make_float2(0.f, 0.f);
#pragma unroll
            for (int jj = 0; jj < QB; ++jj) {
                const float4 zz = znext;
                if (jj + 1 < QB)
                    znext = zq[b * QB + jj + 1];
                else if (b > 0)
                    znext = zq[(b - 1) * QB];
                const int j = 2 * jj;
                const float2 z0 = make_float2(zz.x, zz.y), z1 = make_float2(zz.z, zz.w);
                // each z pair feeds 2*NC consecutive FFMA2 (operand reuse)
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    A[c] = ffma2(z0, er[c][j], A[c]);
                    B[c] = ffma2(z0, ei[c][j], B[c]);
                }
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    A[c] = ffma2(z1, er[c][j + 1], A[c]);
                    B[c] = ffma2(z1, ei[c][j + 1], B[c]);
                }
            }
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const float cr = A[c].x - B[c].y, ci = A[c].y + B[c].x;  // C = A + jB
                bq[c] = fmaf(cr, cr, fmaf(ci, ci, bq[c]));
                const float nr = fmaf(hr[c], w1r[c], fmaf(-hi[c], w1i[c], cr));
                hi[c] = fmaf(hr[c], w1i[c], fmaf(hi[c], w1r[c], ci));
                hr[c] = nr;
            }
        }
        // anchor W = e^{j 2 pi f c0} from the FP64-reduced phase
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            float wr, wi;
            const double x = f[c] * (double)c0;
            cis_f64(x, &wr, &wi);
            acc_re[c] += (double)fmaf(wr, hr[c], -(wi * hi[c]));
            acc_im[c] += (double)fmaf(wr, hi[c], wi * hr[c]);
            e2[c] += (double)fmaf(hr[c], hr[c], hi[c] * hi[c]);
            eb[c] += (double)bq[c];
        }
        __syncwarp();  // this stage's buffers are free for the next bulk copy
    }

#pragma unroll
    for (int o = 16; o; o >>= 1) z2 += __shfl_xor_sync(0xffffffffu, z2, o);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        if (p[c] < 0) continue;
        const double s = sqrt(acc_re[c] * acc_re[c] + acc_im[c] * acc_im[c]);
        s_out[p[c]] = s;
        if (s < (double)tau * sqrt(fmax(fmax(e2[c], eb[c]), (double)z2))) {
            const int64_t e = flag_base + p[c];
            atomicOr(&flag_bits[e >> 5], 1u << (e & 31));
        }
    }
}

namespace {

template <int NC, int LB, int CH, int WPC, int MINB>
void launch_variant(int n_tasks_max, cudaStream_t st, const Task* tasks, const int* n_tasks,
                    const int* sorted, const double* fdoa, const float2* y1, const float2* y2,
                    int N, double fs, double* s_out, uint32_t* flag_bits, int64_t flag_base,
                    float tau) {
    auto kern = k_correlate<NC, LB, CH, WPC, MINB>;
    const size_t smem = sizeof(WarpSmemT<CH>) * WPC;
    static size_t attr[64] = {};
    ensure_smem(kern, smem, attr);
    const int blocks = (n_tasks_max + WPC - 1) / WPC;
    kern<<<blocks, 32 * WPC, smem, st>>>(tasks, n_tasks, sorted, fdoa, y1, y2, N, fs, s_out,
                                         flag_bits, flag_base, tau);
}

}  // namespace

// two candidates per lane (a 64-candidate warp task), 3 CTAs x 4 warps per SM
// (148 registers): the variant kept from the r01 sweep of (NC, LB, CH, WPC, MINB)
int correlate_task_size() { return 64; }

void launch_correlate(const Task* tasks, const int* n_tasks, int max_tasks, const int* sorted,
                      const double* fdoa, const float2* y1, const float2* y2, int N, double fs,
                      double* s_out, uint32_t* flag_bits, int64_t flag_base, float tau,
                      cudaStream_t st) {
    if (max_tasks <= 0) return;
    launch_variant<2, 16, 256, 4, 3>(max_tasks, st, tasks, n_tasks, sorted, fdoa, y1, y2, N, fs,
                                     s_out, flag_bits, flag_base, tau);
}

}  // namespace dg
