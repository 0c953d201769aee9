// K3c: candidate evaluation of the block-moment correlator with the block sums on
// the 5th-generation tensor cores (tcgen05, TMEM accumulators).
//
// For a TDOA bucket with moments M'_m[b] (b < nb, m < R; odd m stored times i) each
// candidate needs C_b = sum_m c_m M'_m[b] for every block (k_evaluate: R FFMA2 per
// candidate-block) and then S = |sum_b W^b C_b|. The first step is a real GEMM:
//   D[i][2b + ri] = sum_k A[i][k] B[2b + ri][k],  A[i][k] = c_k(candidate i),
//   B[2b][k] = Re M'_k[b],  B[2b+1][k] = Im M'_k[b],  K = R padded to 16,
// one 128-candidate tile x 2 nb columns per bucket tile, i.e. tcgen05.mma
// kind::f16 (BF16 operands, FP32 accumulation in TMEM) with M = 128, N = 2 nb
// (<= 256 per instruction) and K = 16 in one instruction. BF16 keeps 8
// significand bits, so both operands are split into three BF16 parts
// x = h + m + l (exact for an FP32 moment; 24 bits of the FP64 coefficient) and
// D = hl + mm + lh + hm + mh + hh (every product term down to 2^-16 relative;
// the dropped ones are <= 2^-24): FP32-class C_b, checked by the same error
// model as the FFMA2 path.
//
// One CTA (4 warps, 128 threads = the 128 TMEM lanes = one candidate each) per
// bucket from a dynamic queue; the bucket's moments arrive by TMA bulk copy into
// a 2-stage ring; all threads split them into the B operand (no-swizzle K-major
// core-matrix layout); per tile each thread computes its candidate's J_m(x)
// (FP64) into the A operand; thread 0 issues the six MMAs and commits to an
// mbarrier; each thread then reads its TMEM lane 32 columns (16 blocks) at a time
// (two tcgen05.ld.32x32b.x16) and runs the group sums as
// k_evaluate does: A, V, |C_b|^2 on FFMA2 with W_j = W_1^j (FP64 recurrence,
// rounded once), FP64 anchors across groups, refinement flag
// refine_moment (dg_device.cuh).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "dg_device.cuh"
#include "dg_internal.cuh"

namespace dg {

namespace {

constexpr int kTcThreads = 128;
constexpr int kTcStages = 1;
constexpr int kTcK = 16;          // K (moments) padded: one kind::f16 instruction
constexpr int kTcG = 16;          // blocks per epilogue group (32 TMEM columns)
constexpr uint32_t kLBO = 128;    // bytes between the two 16-byte K chunks of a core matrix pair
constexpr uint32_t kSBO = 256;    // bytes between 8-row groups (2 K chunks x 128 B)
constexpr int kParts = 3;         // BF16 parts per operand
constexpr int kChunkCols = 128;   // TMEM columns per MMA chunk (4 groups of 16 blocks)

// byte offset of the 16-byte chunk (row r, K chunk c: k = 8c .. 8c + 7) in the
// no-swizzle K-major core-matrix layout
__device__ __forceinline__ uint32_t cm_off(int r, int c) {
    return (uint32_t)(r >> 3) * kSBO + (uint32_t)c * kLBO + (uint32_t)(r & 7) * 16u;
}

// two FP32 values x = h + m + l exactly in BF16 parts (each residual is exact in
// FP32), packed in pairs: out[0] = h, out[1] = m, out[2] = l
__device__ __forceinline__ void split3x2(float x0, float x1, uint32_t (&out)[3]) {
    __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
    float2 f = __bfloat1622float2(h);
    const float r0 = x0 - f.x, r1 = x1 - f.y;
    __nv_bfloat162 m = __floats2bfloat162_rn(r0, r1);
    f = __bfloat1622float2(m);
    __nv_bfloat162 l = __floats2bfloat162_rn(r0 - f.x, r1 - f.y);
    out[0] = *reinterpret_cast<uint32_t*>(&h);
    out[1] = *reinterpret_cast<uint32_t*>(&m);
    out[2] = *reinterpret_cast<uint32_t*>(&l);
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((kLBO >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((kSBO >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    return d;                // base offset 0, legacy LBO mode, SWIZZLE_NONE
}

// kind::f16, D f32, A/B BF16 K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t instr_desc(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// two x16 loads, one wait (the group's 32 columns in one TMEM round trip)
__device__ __forceinline__ void tmem_ld16x2(uint32_t taddr, float (&v0)[16], float (&v1)[16]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
          "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr + 16u));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        v0[i] = __uint_as_float(r[i]);
        v1[i] = __uint_as_float(r[16 + i]);
    }
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

struct TcLayout {
    int NP;           // B rows: 2 blocks per group-column pair, 32 * ceil(nbmax / 16)
    int ncols;        // TMEM columns allocated: one column chunk (<= kChunkCols)
    size_t ring_f2;   // float2 per ring stage
    size_t part_b;    // bytes of one BF16 part of B (NP x 16)
    size_t off_b, off_a, bytes;
};

__host__ __device__ inline TcLayout tc_layout(int nbmax, int R) {
    TcLayout L{};
    L.NP = 2 * kTcG * ((nbmax + kTcG - 1) / kTcG);
    L.ncols = 32;
    while (L.ncols < L.NP && L.ncols < kChunkCols) L.ncols <<= 1;
    L.ring_f2 = (size_t)nbmax * R;
    L.part_b = (size_t)L.NP * kTcK * 2;
    const size_t ring = (kTcStages * L.ring_f2 * 8 + 1023) / 1024 * 1024;
    L.off_b = ring;                                  // B parts h | m | l
    L.off_a = L.off_b + kParts * L.part_b;           // A parts h | m | l, 128 x 16 each
    L.bytes = L.off_a + kParts * (size_t)128 * kTcK * 2;
    return L;
}

constexpr size_t kPartA = (size_t)128 * kTcK * 2;

template <int R>
__global__ void __launch_bounds__(kTcThreads, 4)
k_evaluate_tc(const FftErr fx, const Bucket* __restrict__ buckets, const int* __restrict__ n_buckets,
              int* __restrict__ queue, const int* __restrict__ sorted,
              const double* __restrict__ fdoa, double fs, const double* __restrict__ nu_c_p,
              int B, const float2* __restrict__ mom, int nbmax, double* __restrict__ s_out,
              uint32_t* __restrict__ flag_bits, int64_t flag_base, float tau, float tau_noise,
              const double* __restrict__ e1, const double* __restrict__ e2, int N) {
    constexpr int G = kTcG;
    static_assert(R <= kTcK && R % 2 == 0, "moments");
    const TcLayout L = tc_layout(nbmax, R);
    extern __shared__ __align__(1024) float4 smem4[];
    char* base = reinterpret_cast<char*>(smem4);
    const float2* ring = reinterpret_cast<const float2*>(base);
    char* Bs = base + L.off_b;
    char* As = base + L.off_a;
    __shared__ uint64_t full[kTcStages], empty[kTcStages], mma_bar;
    __shared__ int slot_u[kTcStages];
    __shared__ uint32_t tmem_base_s;
    __shared__ float qm2[kTcK];  // Q_m^2 = sum_b |M_m[b]|^2 of the bucket
    __shared__ float qf2m[kTcK];  // FFT moments: sum_b of the window's mean square
    __shared__ double z2w[kTcThreads / 32];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nbk = *n_buckets;
    const double nu_c = *nu_c_p;
    const double inv_fs = 1.0 / fs;  // (the fast path's nu; refinement and re-rank keep fdoa / fs)

    auto produce = [&](int k, bool block) -> bool {  // thread 0 (as k_evaluate)
        const int sl = k % kTcStages;
        if (k >= kTcStages) {
            const uint32_t par = ((k / kTcStages) - 1) & 1;
            if (block)
                mbar_wait(&empty[sl], par);
            else if (!mbar_test(&empty[sl], par))
                return false;
        }
        const int u = atomicAdd(queue, 1);
        slot_u[sl] = u;
        if (u < nbk) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const uint32_t bytes = (uint32_t)buckets[u].nb * R * sizeof(float2);
            mbar_expect_tx(&full[sl], bytes);
            tma_load_1d(base + sl * L.ring_f2 * 8, mom + (size_t)u * nbmax * R, bytes, &full[sl]);
        } else {
            mbar_arrive(&full[sl]);
        }
        return true;
    };
    if (warp == 0) {  // TMEM for this CTA's lifetime (warp-wide alloc)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&tmem_base_s)),
                     "r"((uint32_t)L.ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < kTcStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(&mma_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
    int produced = 0;
    if (tid == 0)
        for (; produced < kTcStages; ++produced) produce(produced, false);

    const uint32_t sA = smem_u32(As), sB = smem_u32(Bs);
    uint32_t mma_phase = 0;
    for (int k = 0;; ++k) {
        if (tid == 0) {
            for (; produced <= k; ++produced) produce(produced, true);
            while (produced < k + kTcStages && produce(produced, false)) ++produced;
        }
        const int sl = k % kTcStages;
        mbar_wait(&full[sl], (k / kTcStages) & 1);
        const int u = slot_u[sl];
        if (u >= nbk) break;
        const Bucket bk = buckets[u];
        const int nb = bk.nb;
        // the first tile's candidate, loaded now so the latency hides under the B split
        int p = tid < bk.count ? sorted[bk.start + tid] : -1;
        double fd = p >= 0 ? fdoa[p] : 0.0;
        const float2* mb = ring + sl * L.ring_f2;
        const int ng = (nb + G - 1) / G;
        const int np = 2 * G * ng;  // B rows / TMEM columns used by this bucket
        for (int m = warp; m < R; m += kTcThreads / 32) {  // Q_m^2, fixed order
            float q2 = 0.f;
            for (int b = lane; b < nb; b += 32) {
                const float2 v = mb[b * R + m];
                q2 = fmaf(v.x, v.x, fmaf(v.y, v.y, q2));
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) q2 += __shfl_xor_sync(0xffffffffu, q2, o);
            if (lane == 0) qm2[m] = q2;
        }
        // FFT moments: the rounding's scale, the lag window's energy over the bucket's
        // blocks (k_fft_bucket_energy)
        if (fx.qf && tid < R) qf2m[tid] = fx.qf[(size_t)u * kMaxMoments + tid];
        {  // ||z||_2^2 of the bucket (the floor of the error scale), fixed order
            double z2 = bucket_z2_part(e1, e2, N, bk.d, B, tid, kTcThreads);
#pragma unroll
            for (int o = 16; o; o >>= 1) z2 += __shfl_xor_sync(0xffffffffu, z2, o);
            if (lane == 0) z2w[warp] = z2;
        }
        // B operand: per (block b, K chunk c) the rows 2b (Re) and 2b + 1 (Im),
        // columns 8c .. 8c + 7, three BF16 parts; zeros beyond nb / R
        for (int e = tid; e < (np / 2) * 2; e += kTcThreads) {
            const int b = e >> 1, c = e & 1;
            uint32_t re[kParts][4], im[kParts][4];
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                const int m = 8 * c + j;
                if (b < nb && m < R)  // R even: m + 1 < R; 16-byte aligned pair
                    v = *reinterpret_cast<const float4*>(mb + b * R + m);
                uint32_t t[3];
                split3x2(v.x, v.z, t);
                re[0][j / 2] = t[0];
                re[1][j / 2] = t[1];
                re[2][j / 2] = t[2];
                split3x2(v.y, v.w, t);
                im[0][j / 2] = t[0];
                im[1][j / 2] = t[1];
                im[2][j / 2] = t[2];
            }
#pragma unroll
            for (int q = 0; q < kParts; ++q) {
                *reinterpret_cast<uint4*>(Bs + q * L.part_b + cm_off(2 * b, c)) =
                    make_uint4(re[q][0], re[q][1], re[q][2], re[q][3]);
                *reinterpret_cast<uint4*>(Bs + q * L.part_b + cm_off(2 * b + 1, c)) =
                    make_uint4(im[q][0], im[q][1], im[q][2], im[q][3]);
            }
        }
        __syncthreads();
        if (tid == 0) mbar_arrive(&empty[sl]);  // the ring slot is free again
        double zfloor = 0.0;
#pragma unroll
        for (int w = 0; w < kTcThreads / 32; ++w) zfloor += z2w[w];
        const RefineBucket rfb =
            refine_bucket(zfloor, bucket_coherence(qm2, R, zfloor), tau, tau_noise);

        for (int t0 = 0; t0 < bk.count; t0 += 128) {
            const double nu = p >= 0 ? fma(fd, inv_fs, -nu_c) : 0.0;
            const int pc = p;  // this tile's candidate; p / fd now prefetch the next tile's
            {
                const int nx = t0 + 128 + tid;
                p = nx < bk.count ? sorted[bk.start + nx] : -1;
                fd = p >= 0 ? fdoa[p] : 0.0;
            }
            // warps without a candidate in this tile skip the Bessel terms and the
            // epilogue (their A rows are zero); tcgen05.ld stays warp-uniform
            const bool warp_live = __any_sync(0xffffffffu, pc >= 0);
            // the moments' own FP32 rounding as this candidate's block sums inherit
            // it: sqrt(sum_m a_m^2 Q_m^2)
            double qe2 = 0.0;
            // ---- A operand: this thread's candidate, c_m rounded to FP32 (as the
            // FFMA2 path) and split exactly into three BF16 parts ----
            {
                float cf[kTcK];
#pragma unroll
                for (int m = 0; m < kTcK; ++m) cf[m] = 0.f;
                if (pc >= 0) {
                    double jv[R];
                    bessel_j<R>(3.141592653589793 * nu * (double)B, jv);
                    float qa = 0.f, qb = 0.f;  // a scale: FP32, two independent chains
#pragma unroll
                    for (int m = 0; m < R; ++m) {
                        cf[m] = (float)((m == 0 ? 1.0 : 2.0) * (((m >> 1) & 1) ? -1.0 : 1.0) * jv[m]);
                        if (m & 1)
                            qb = fmaf(cf[m] * cf[m], qm2[m], qb);
                        else
                            qa = fmaf(cf[m] * cf[m], qm2[m], qa);
                    }
                    qe2 = (double)qa + (double)qb;
                    if (fx.qf) {  // FFT moments: the window's excess energy, weighted
                        float fa = 0.f, fb = 0.f;
#pragma unroll
                        for (int m = 0; m < R; ++m) {
                            if (m & 1)
                                fb = fmaf(cf[m] * cf[m], qf2m[m], fb);
                            else
                                fa = fmaf(cf[m] * cf[m], qf2m[m], fa);
                        }
                        const double qf2 = (double)fa + (double)fb;
                        qe2 += (double)fx.kappa * fmax(qf2 - qe2, 0.0);
                    }
                }
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    uint32_t w[kParts][4];
#pragma unroll
                    for (int j = 0; j < 8; j += 2) {
                        uint32_t t[3];
                        split3x2(cf[8 * c + j], cf[8 * c + j + 1], t);
                        w[0][j / 2] = t[0];
                        w[1][j / 2] = t[1];
                        w[2][j / 2] = t[2];
                    }
#pragma unroll
                    for (int q = 0; q < kParts; ++q)
                        *reinterpret_cast<uint4*>(As + q * kPartA + cm_off(tid, c)) =
                            make_uint4(w[q][0], w[q][1], w[q][2], w[q][3]);
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic -> async proxy
            tc_fence_before();
            __syncthreads();
            // the bucket's columns in chunks of kChunkCols TMEM columns: MMA a chunk,
            // then every thread reads its lane of it (4 groups of 16 blocks)
            float wtr[G], wti[G];
            double sr = 1.0, si = 0.0;
            double acc_re = 0.0, acc_im = 0.0, ar = 1.0, ai = 0.0;
            float en = 0.f;  // sum_b |C_b|^2: an error scale, FP32
            float w16r = 1.f, w16i = 0.f, pnd_r = 0.f, pnd_i = 0.f;
            bool pend = false;
            for (int c0 = 0; c0 < np; c0 += kChunkCols) {
                const int nn = np - c0 < kChunkCols ? np - c0 : kChunkCols;
                if (tid == 0) {
                    tc_fence_after();
                    const uint32_t idesc = instr_desc(nn);
                    const uint32_t boff = (uint32_t)(c0 >> 3) * kSBO;
                    // smallest terms first: hl, mm, lh, hm, mh, hh
                    constexpr int pa[6] = {0, 1, 2, 0, 1, 0};
                    constexpr int pb[6] = {2, 1, 0, 1, 0, 0};
#pragma unroll
                    for (int t = 0; t < 6; ++t)
                        mma_bf16(tmem, smem_desc(sA + pa[t] * (uint32_t)kPartA),
                                 smem_desc(sB + pb[t] * (uint32_t)L.part_b + boff), idesc,
                                 t ? 1u : 0u);
                    mma_commit(&mma_bar);
                }
                if (c0 == 0 && warp_live) {
                    // W_j = W_1^j while the MMAs run: W_0..W_4 by an FP64 recurrence,
                    // W_8 = W_4^2, W_12 = W_8 W_4, W_16 = W_8^2 in FP64, each rounded
                    // once to FP32; W_{4a+b} = W_{4a} W_b as one FP32 complex product
                    const double x1 = nu * (double)B;
                    double w1r, w1i;
                    sincospi(2.0 * (x1 - rint(x1)), &w1i, &w1r);
                    double br[5], bi[5];
                    br[0] = 1.0;
                    bi[0] = 0.0;
#pragma unroll
                    for (int j = 1; j <= 4; ++j) {
                        br[j] = fma(br[j - 1], w1r, -bi[j - 1] * w1i);
                        bi[j] = fma(br[j - 1], w1i, bi[j - 1] * w1r);
                    }
                    const double w8r = fma(br[4], br[4], -bi[4] * bi[4]), w8i = 2.0 * br[4] * bi[4];
                    const double w12r = fma(w8r, br[4], -w8i * bi[4]);
                    const double w12i = fma(w8r, bi[4], w8i * br[4]);
                    const double s16r = fma(w8r, w8r, -w8i * w8i), s16i = 2.0 * w8r * w8i;
                    w16r = (float)s16r;
                    w16i = (float)s16i;
                    sr = fma(s16r, s16r, -s16i * s16i);  // W_32: the anchor step of a group pair
                    si = 2.0 * s16r * s16i;
                    const float hr[4] = {1.f, (float)br[4], (float)w8r, (float)w12r};
                    const float hi4[4] = {0.f, (float)bi[4], (float)w8i, (float)w12i};
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const float lr = (float)br[b], li = (float)bi[b];
#pragma unroll
                        for (int a = 0; a < 4; ++a) {
                            wtr[4 * a + b] = fmaf(hr[a], lr, -hi4[a] * li);
                            wti[4 * a + b] = fmaf(hr[a], li, hi4[a] * lr);
                        }
                    }
                }
                mbar_wait(&mma_bar, mma_phase);
                mma_phase ^= 1;
                tc_fence_after();
                for (int gc = 0; warp_live && gc < nn; gc += 2 * G) {
                    float v[2][16];
                    tmem_ld16x2(lane_addr + (uint32_t)gc, v[0], v[1]);
                    // two interleaved chains per sum (blocks 0-7 / 8-15 of the group)
                    float2 A0 = make_float2(0.f, 0.f), V0 = A0, E0 = A0, A1 = A0, V1 = A0, E1 = A0;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float2 C0 = make_float2(v[0][2 * j], v[0][2 * j + 1]);
                        const float2 C1 = make_float2(v[1][2 * j], v[1][2 * j + 1]);
                        A0 = ffma2(C0, wtr[j], A0);
                        A1 = ffma2(C1, wtr[j + 8], A1);
                        V0 = ffma2(C0, wti[j], V0);
                        V1 = ffma2(C1, wti[j + 8], V1);
                        E0 = ffma2v(C0, C0, E0);
                        E1 = ffma2v(C1, C1, E1);
                    }
                    const float2 A = add2(A0, A1), V = add2(V0, V1), E2 = add2(E0, E1);
                    const float hr = A.x - V.y, hi = A.y + V.x;
                    en += E2.x + E2.y;
                    if (!pend) {  // groups in pairs: the first one waits in FP32
                        pnd_r = hr;
                        pnd_i = hi;
                        pend = true;
                    } else {  // pair sum h_g + W_16 h_{g+1} (FP32), then one FP64 anchor
                        pnd_r = fmaf(w16r, hr, fmaf(-w16i, hi, pnd_r));
                        pnd_i = fmaf(w16r, hi, fmaf(w16i, hr, pnd_i));
                        acc_re = fma(ar, (double)pnd_r, fma(-ai, (double)pnd_i, acc_re));
                        acc_im = fma(ar, (double)pnd_i, fma(ai, (double)pnd_r, acc_im));
                        const double nr = fma(ar, sr, -ai * si);  // advance by W_32
                        ai = fma(ar, si, ai * sr);
                        ar = nr;
                        pend = false;
                    }
                }
                tc_fence_before();  // this chunk's TMEM reads done before the next MMAs
                __syncthreads();
            }
            if (pend) {  // a last unpaired group
                acc_re = fma(ar, (double)pnd_r, fma(-ai, (double)pnd_i, acc_re));
                acc_im = fma(ar, (double)pnd_i, fma(ai, (double)pnd_r, acc_im));
            }
            if (pc >= 0) {
                const double s2 = acc_re * acc_re + acc_im * acc_im;
                s_out[pc] = sqrt(s2);
                if (refine_moment(s2, (double)en, qe2, rfb)) {
                    const int64_t e = flag_base + pc;
                    atomicOr(&flag_bits[e >> 5], 1u << (e & 31));
                }
            }
        }
        __syncthreads();  // B / A / q2s reuse by the next bucket
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"((uint32_t)L.ncols));
}

template <int R>
void evaluate_tc_variant(FftErr fx, const Bucket* buckets, const int* n_buckets, int* queue, int max_buckets,
                         const int* sorted, const double* fdoa, double fs, const double* nu_c,
                         int B, const float2* mom, int nbmax, double* s_out, uint32_t* flag_bits,
                         int64_t flag_base, float tau, float tau_noise, const double* e1,
                         const double* e2, int N, int sm_count, cudaStream_t st) {
    auto kern = k_evaluate_tc<R>;
    const TcLayout L = tc_layout(nbmax, R);
    // CTAs per SM bounded by TMEM (512 columns per SM): request enough shared
    // memory that no more CTAs than fit in TMEM are resident on one SM
    const int per_sm = 512 / L.ncols;
    size_t smem = L.bytes;
    const size_t floor_bytes = (size_t)(228 * 1024) / (per_sm + 1) + 1024;
    if (smem < floor_bytes) smem = floor_bytes;
    static size_t attr[64] = {};
    ensure_smem(kern, smem, attr);
    // resident CTAs: TMEM-bound, or shared-memory-bound (228 KB per SM, 1 KB
    // reserved per CTA, ~1 KB of static shared memory)
    int resident = (int)((228 * 1024) / (smem + 2048));
    if (resident > per_sm) resident = per_sm;
    if (resident < 1) resident = 1;
    int grid = sm_count * resident;
    if (grid > max_buckets) grid = max_buckets > 0 ? max_buckets : 1;
    kern<<<grid, kTcThreads, smem, st>>>(fx, buckets, n_buckets, queue, sorted, fdoa, fs, nu_c, B, mom,
                                         nbmax, s_out, flag_bits, flag_base, tau, tau_noise, e1,
                                         e2, N);
}

}  // namespace

bool evaluate_tc_supported(int nbmax, int R) {
    const TcLayout L = tc_layout(nbmax, R);
    return L.ncols <= 512 && L.bytes <= 200 * 1024 && R <= kTcK;
}

void launch_evaluate_tc(FftErr fx, int R, const Bucket* buckets, const int* n_buckets, int* queue,
                        int max_buckets, const int* sorted, const double* fdoa, double fs,
                        const double* nu_c, int B, const float2* mom, int nbmax, double* s_out,
                        uint32_t* flag_bits, int64_t flag_base, float tau, float tau_noise,
                        const double* e1, const double* e2, int N, int sm_count,
                        cudaStream_t st) {
#define DG_TC_CASE(RR)                                                                          \
    evaluate_tc_variant<RR>(fx, buckets, n_buckets, queue, max_buckets, sorted, fdoa, fs, nu_c, B, \
                            mom, nbmax, s_out, flag_bits, flag_base, tau, tau_noise, e1, e2, N, \
                            sm_count, st)
    switch (R) {
        case 8: DG_TC_CASE(8); break;
        case 10: DG_TC_CASE(10); break;
        case 12: DG_TC_CASE(12); break;
        case 14: DG_TC_CASE(14); break;
        default: DG_TC_CASE(16); break;
    }
#undef DG_TC_CASE
}

}  // namespace dg
