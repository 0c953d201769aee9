// K3 (block-moment form): Eq. 11 (reference correlate.hpp:44-71) factored so
// that the work shared by all candidates of one integer TDOA d is done once.
//
// For a d-bucket the product stream z[k] = y1[k] conj(y2[k+d]) over the
// overlap [kb, ke) is cut into blocks of B samples starting at kb. With the
// block-centred coordinate t_j = (2j - (B-1)) / B in (-1, 1) and x = pi nu B
// (nu = fdoa/fs in cycles/sample), the Jacobi-Anger expansion
//     e^{i x t} = sum_m (2 - delta_m0) i^m J_m(x) T_m(t)
// gives, for block b,
//     sum_j z[kb+bB+j] e^{i 2 pi nu j} = e^{i x (B-1)/B} sum_m a_m(x) M_m[b],
//     M_m[b] = sum_j z[kb+bB+j] T_m(t_j)            (shared by the bucket)
// so each candidate needs R real-by-complex MACs per block instead of B
// complex MACs, plus one Horner step e^{i 2 pi nu B} across blocks:
//     S = | sum_b e^{i 2 pi nu B b} sum_m a_m M_m[b] |.
// The truncation after R terms is bounded by 2 (x/2)^R / R! of the block's
// L1 norm; the host picks (B, R) per step from the step's FDOA range so that
// bound is <= 1e-8. y1 is pre-rotated by the
// step's centre frequency nu_c (k_center, FP64 phase) so |x| is set by the
// half-width of the FDOA range, not its offset.
//
//   k_center    y1c[k] = fp32(y1[k] e^{i 2 pi nu_c k})           (FP64 math)
//   k_moments   per (bucket, 32-block chunk): z into shared memory, then
//               M_m[b] on FFMA2 with the Chebyshev table broadcast from smem
//   k_evaluate  one warp = up to 64 candidates of one bucket (2 per lane):
//               J_m(x) by series + backward recurrence (FP64), block loop on
//               FFMA2 with the bucket's moments as broadcast loads, Horner in
//               FP32 within groups of G blocks, FP64-reduced anchors, FP64 sum.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "dg_internal.cuh"

namespace dg {

namespace {

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

// e^{i 2 pi x} for an FP64 cycle count: exact FP64 range reduction, FP32 sincospi
__device__ __forceinline__ void cis_cycles(double x, float* c, float* s) {
    sincospif((float)(2.0 * (x - rint(x))), s, c);
}

constexpr int kChunkBlocks = 32;  // blocks per k_moments work item (one per lane)

// two staging buffers of one bucket's moments
inline size_t evaluate_smem(int nbmax, int R) { return 2 * (size_t)nbmax * R * sizeof(float2); }
constexpr int kMomThreads = 256;

// table + max(z chunk, per-warp partial moments)
constexpr size_t moments_smem(int B) {
    return (size_t)B * kMaxMoments * sizeof(float) +
           sizeof(float2) * ((size_t)kChunkBlocks * (B + 1) > (size_t)8 * 32 * (kMaxMoments + 1)
                                 ? (size_t)kChunkBlocks * (B + 1)
                                 : (size_t)8 * 32 * (kMaxMoments + 1));
}

__global__ void k_center(const double2* __restrict__ y, int N, const double* __restrict__ nu_c,
                         float2* __restrict__ out) {
    const double nc = *nu_c;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
        const double ph = nc * (double)k;
        double s, c;
        sincospi(2.0 * (ph - rint(ph)), &s, &c);
        const double2 v = y[k];
        out[k] = make_float2((float)(v.x * c - v.y * s), (float)(v.x * s + v.y * c));
    }
}

template <int B, int R>
__global__ void __launch_bounds__(kMomThreads, 2)
k_moments(const Bucket* __restrict__ buckets, const int* __restrict__ n_buckets, int cpb,
          const float* __restrict__ tcheb, const float2* __restrict__ y1c,
          const float2* __restrict__ y2, int N, float2* __restrict__ mom, int nbmax) {
    static_assert(B % 64 == 0 && B <= 256, "block length");
    static_assert(R % 2 == 0 && R <= kMaxMoments, "moment count");
    constexpr int RQ = (R + 3) / 4;          // float4 rows of the table actually read
    constexpr int ZS = B + 1;                // padded z row (conflict-free column reads)
    constexpr int JW = B / 8;                // samples per warp in the moment pass
    extern __shared__ float4 smem4[];
    float* ts = reinterpret_cast<float*>(smem4);                    // [B][kMaxMoments]
    float2* zs = reinterpret_cast<float2*>(ts + B * kMaxMoments);   // [32][ZS]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < B * kMaxMoments; i += kMomThreads) ts[i] = tcheb[i];

    const int nitems = *n_buckets * cpb;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
        const int u = item / cpb, c = item - u * cpb;
        const Bucket bk = buckets[u];
        const int b0 = c * kChunkBlocks;
        if (b0 >= bk.nb) continue;  // uniform: this chunk is past the overlap
        const int d = bk.d;
        const int kb = d < 0 ? -d : 0;
        const int ke = d > 0 ? N - d : N;
        const int k0 = kb + b0 * B;
        __syncthreads();  // table loaded / previous item's reduction consumed

        // ---- z = y1c conj(y2[k+d]) for the chunk, zero past the overlap ----
#pragma unroll 4
        for (int i = tid; i < kChunkBlocks * B; i += kMomThreads) {
            const int k = k0 + i;
            float2 zz = make_float2(0.f, 0.f);
            if (k < ke) {
                const float2 a = y1c[k], b = y2[k + d];
                zz.x = fmaf(a.x, b.x, a.y * b.y);
                zz.y = fmaf(a.y, b.x, -(a.x * b.y));
            }
            zs[(i / B) * ZS + (i % B)] = zz;
        }
        __syncthreads();

        // ---- lane = block, warp = slice of j: partial moments on FFMA2 ----
        float2 acc[R];
#pragma unroll
        for (int m = 0; m < R; ++m) acc[m] = make_float2(0.f, 0.f);
        const float2* zrow = zs + lane * ZS + warp * JW;
        const float4* trow = reinterpret_cast<const float4*>(ts + warp * JW * kMaxMoments);
#pragma unroll 4
        for (int j = 0; j < JW; ++j) {
            const float2 zv = zrow[j];
#pragma unroll
            for (int q = 0; q < RQ; ++q) {
                const float4 t = trow[j * (kMaxMoments / 4) + q];
                if (4 * q + 0 < R) acc[4 * q + 0] = ffma2(zv, t.x, acc[4 * q + 0]);
                if (4 * q + 1 < R) acc[4 * q + 1] = ffma2(zv, t.y, acc[4 * q + 1]);
                if (4 * q + 2 < R) acc[4 * q + 2] = ffma2(zv, t.z, acc[4 * q + 2]);
                if (4 * q + 3 < R) acc[4 * q + 3] = ffma2(zv, t.w, acc[4 * q + 3]);
            }
        }
        __syncthreads();  // every warp is done reading zs
        // partials -> smem [warp][block][R+1] (reuses the z buffer), fixed-order sum
        float2* red = zs;
#pragma unroll
        for (int m = 0; m < R; ++m) red[(warp * 32 + lane) * (R + 1) + m] = acc[m];
        __syncthreads();
        const int nbc = min(kChunkBlocks, bk.nb - b0);
        float2* dst = mom + ((size_t)u * nbmax + b0) * R;
        for (int o = tid; o < nbc * R; o += kMomThreads) {
            const int b = o / R, m = o - b * R;
            float2 s = red[b * (R + 1) + m];
#pragma unroll
            for (int w = 1; w < 8; ++w) {
                const float2 v = red[(w * 32 + b) * (R + 1) + m];
                s.x += v.x;
                s.y += v.y;
            }
            // odd moments are stored times i, so a candidate's block value is
            // one real-weighted sum  C_b = sum_m c_m M'_m  (k_evaluate)
            dst[o] = (m & 1) ? make_float2(-s.y, s.x) : s;
        }
    }
}

// J_0..J_{R-1}(x) (first kind), FP64: series for J_{R-1}, J_R (fast: m >> x),
// then the stable backward recurrence J_{m-1} = (2m/x) J_m - J_{m+1}.
template <int R>
__device__ __forceinline__ void bessel_j(double x, double (&j)[R]) {
    const double ax = fabs(x);
    if (ax < 1e-6) {
#pragma unroll
        for (int m = 0; m < R; ++m) j[m] = 0.0;
        j[0] = 1.0 - 0.25 * x * x;
        if (R > 1) j[1] = 0.5 * x;
        return;
    }
    const double h = 0.5 * x, h2 = h * h;
    // (x/2)^(R-1) / (R-1)!
    double t = 1.0;
#pragma unroll
    for (int m = 1; m < R; ++m) t *= h * (1.0 / m);
    double jr1 = 0.0, jr = 0.0;  // J_{R-1}, J_R
    {
        double term = t, s = t;
#pragma unroll
        for (int k = 1; k <= 12; ++k) {
            term *= -h2 * (1.0 / (k * (R - 1 + k)));
            s += term;
        }
        jr1 = s;
        term = t * h * (1.0 / R);
        s = term;
#pragma unroll
        for (int k = 1; k <= 12; ++k) {
            term *= -h2 * (1.0 / (k * (R + k)));
            s += term;
        }
        jr = s;
    }
    const double inv = 2.0 / x;
    j[R - 1] = jr1;
    double jp = jr, jc = jr1;
#pragma unroll
    for (int m = R - 1; m >= 1; --m) {
        const double jm = fma((double)m * inv, jc, -jp);
        jp = jc;
        jc = jm;
        j[m - 1] = jm;
    }
}

// ---- TMA helpers (1-D bulk copy global -> shared, mbarrier completion) ----
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
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ float2 ffma2v(float2 a, float2 b, float2 c) {  // elementwise
    float2 d;
    asm("{.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\t"
        "mov.b64 rb, {%4, %5};\n\t"
        "mov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\t"
        "mov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}

constexpr int kEvalWarps = 4;
constexpr int kEvalNC = 2;                              // candidates per lane
constexpr int kEvalPass = 32 * kEvalWarps * kEvalNC;   // candidates per CTA pass

// One CTA per d-bucket (dynamic queue), the bucket's moments staged in shared
// memory by one TMA bulk copy (double-buffered: the next bucket's copy runs
// under this bucket's evaluation); each lane evaluates kEvalNC candidates:
//   C_b = sum_m c_m M'_m[b]                       (R FFMA2, broadcast LDS.128)
//   group g of G blocks:  A += Re(W_j) C_b, V += Im(W_j) C_b, e += C_b o C_b
//   H_g = A + iV;  acc += e^{i 2 pi nu B G g} H_g   (anchor from an FP64 phase)
// W_j = e^{i 2 pi nu B j} (j < G) are rounded once from FP64 phases.
template <int R, int G>
__global__ void __launch_bounds__(32 * kEvalWarps, 4)
k_evaluate(const Bucket* __restrict__ buckets, const int* __restrict__ n_buckets,
           int* __restrict__ queue, const int* __restrict__ sorted,
           const double* __restrict__ fdoa, double fs, const double* __restrict__ nu_c_p, int B,
           const float2* __restrict__ mom, int nbmax, double* __restrict__ s_out,
           uint32_t* __restrict__ flag_bits, int64_t flag_base, float tau) {
    extern __shared__ float4 smem4[];
    float4* mbuf[2] = {smem4, smem4 + (size_t)nbmax * R / 2};
    __shared__ uint64_t bar[2];
    __shared__ int next_u[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nbk = *n_buckets;
    const double nu_c = *nu_c_p;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const int u0 = atomicAdd(queue, 1);
        next_u[0] = u0;
        if (u0 < nbk) {
            const uint32_t bytes = (uint32_t)buckets[u0].nb * R * sizeof(float2);
            mbar_expect_tx(&bar[0], bytes);
            tma_load_1d(mbuf[0], mom + (size_t)u0 * nbmax * R, bytes, &bar[0]);
        }
    }
    __syncthreads();
    uint32_t phase[2] = {0u, 0u};
    for (int it = 0;; ++it) {
        const int buf = it & 1;
        const int u = next_u[buf];
        if (u >= nbk) break;
        if (tid == 0) {  // claim and prefetch the next bucket into the other buffer
            const int un = atomicAdd(queue, 1);
            next_u[buf ^ 1] = un;
            if (un < nbk) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const uint32_t bytes = (uint32_t)buckets[un].nb * R * sizeof(float2);
                mbar_expect_tx(&bar[buf ^ 1], bytes);
                tma_load_1d(mbuf[buf ^ 1], mom + (size_t)un * nbmax * R, bytes, &bar[buf ^ 1]);
            }
        }
        const Bucket bk = buckets[u];
        const int nb = bk.nb;
        mbar_wait(&bar[buf], phase[buf]);
        phase[buf] ^= 1u;
        const float4* mb = mbuf[buf];

        for (int base = warp * 32 * kEvalNC; base < bk.count; base += kEvalPass) {
            int p[kEvalNC];
            double nu[kEvalNC];
            float cf[kEvalNC][R];
            float wtr[kEvalNC][G], wti[kEvalNC][G];
#pragma unroll
            for (int c = 0; c < kEvalNC; ++c) {
                const int slot = base + 32 * c + lane;
                p[c] = slot < bk.count ? sorted[bk.start + slot] : -1;
                nu[c] = p[c] >= 0 ? fdoa[p[c]] / fs - nu_c : 0.0;
                double jv[R];
                bessel_j<R>(3.141592653589793 * nu[c] * (double)B, jv);
                // a_m M_m = (2 - delta_m0) (-1)^(m/2) J_m M'_m  (M' = i^(m mod 2) M)
#pragma unroll
                for (int m = 0; m < R; ++m)
                    cf[c][m] = (float)((m == 0 ? 1.0 : 2.0) * (((m >> 1) & 1) ? -1.0 : 1.0) * jv[m]);
#pragma unroll
                for (int j = 0; j < G; ++j)
                    cis_cycles(nu[c] * (double)B * (double)j, &wtr[c][j], &wti[c][j]);
            }
            double acc_re[kEvalNC], acc_im[kEvalNC], en[kEvalNC];
#pragma unroll
            for (int c = 0; c < kEvalNC; ++c) acc_re[c] = acc_im[c] = en[c] = 0.0;
            const int ng = (nb + G - 1) / G;
            for (int g = 0; g < ng; ++g) {
                float2 A[kEvalNC], V[kEvalNC], E2[kEvalNC];
#pragma unroll
                for (int c = 0; c < kEvalNC; ++c)
                    A[c] = V[c] = E2[c] = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    const int b = g * G + j;
                    if (b < nb) {
                        float4 mv[R / 2];
#pragma unroll
                        for (int q = 0; q < R / 2; ++q) mv[q] = mb[b * (R / 2) + q];
#pragma unroll
                        for (int c = 0; c < kEvalNC; ++c) {
                            // smallest terms first (the c_m decay with m)
                            float2 C = make_float2(0.f, 0.f);
#pragma unroll
                            for (int q = R / 2 - 1; q >= 0; --q) {
                                C = ffma2(make_float2(mv[q].z, mv[q].w), cf[c][2 * q + 1], C);
                                C = ffma2(make_float2(mv[q].x, mv[q].y), cf[c][2 * q], C);
                            }
                            A[c] = ffma2(C, wtr[c][j], A[c]);
                            V[c] = ffma2(C, wti[c][j], V[c]);
                            E2[c] = ffma2v(C, C, E2[c]);
                        }
                    }
                }
#pragma unroll
                for (int c = 0; c < kEvalNC; ++c) {
                    const float hr = A[c].x - V[c].y, hi = A[c].y + V[c].x;
                    float ar, ai;
                    cis_cycles(nu[c] * (double)(g * G) * (double)B, &ar, &ai);
                    acc_re[c] += (double)fmaf(ar, hr, -(ai * hi));
                    acc_im[c] += (double)fmaf(ar, hi, ai * hr);
                    en[c] += (double)(E2[c].x + E2[c].y);
                }
            }
            // FP32 error scale of this candidate: sqrt(sum_b |C_b|^2) (DESIGN.md
            // section 5); below tau of it the value is re-evaluated in FP64
#pragma unroll
            for (int c = 0; c < kEvalNC; ++c) {
                if (p[c] < 0) continue;
                const double sv = sqrt(acc_re[c] * acc_re[c] + acc_im[c] * acc_im[c]);
                s_out[p[c]] = sv;
                if (sv < (double)tau * sqrt(en[c])) {
                    const int64_t e = flag_base + p[c];
                    atomicOr(&flag_bits[e >> 5], 1u << (e & 31));
                }
            }
        }
        __syncthreads();  // everyone is done with mbuf[buf] and has read next_u
    }
}

// algorithmic work of one step (FP32x2 MACs): moments sum nb*B*R, evaluation
// sum count*nb*R — the numerators of the roofline in bench.py
__global__ void k_work_count(const Bucket* __restrict__ buckets, const int* __restrict__ n_buckets,
                             int B, int R, unsigned long long* __restrict__ work) {
    unsigned long long a = 0, b = 0;
    for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < *n_buckets;
         u += gridDim.x * blockDim.x) {
        const Bucket bk = buckets[u];
        a += (unsigned long long)bk.nb * B * R;
        b += (unsigned long long)bk.count * bk.nb * R;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if ((threadIdx.x & 31) == 0 && (a || b)) {
        atomicAdd(&work[0], a);
        atomicAdd(&work[1], b);
    }
}

template <int B, int R>
void moments_variant(const Bucket* buckets, const int* n_buckets, int cpb, const float* tcheb,
                     const float2* y1c, const float2* y2, int N, float2* mom, int nbmax,
                     int grid, cudaStream_t st) {
    auto kern = k_moments<B, R>;
    const size_t smem = moments_smem(B);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    kern<<<grid, kMomThreads, smem, st>>>(buckets, n_buckets, cpb, tcheb, y1c, y2, N, mom, nbmax);
}

template <int B>
void moments_b(int R, const Bucket* buckets, const int* n_buckets, int cpb, const float* tcheb,
               const float2* y1c, const float2* y2, int N, float2* mom, int nbmax,
               int grid, cudaStream_t st) {
    switch (R) {
        case 8: moments_variant<B, 8>(buckets, n_buckets, cpb, tcheb, y1c, y2, N, mom, nbmax, grid, st); break;
        case 10: moments_variant<B, 10>(buckets, n_buckets, cpb, tcheb, y1c, y2, N, mom, nbmax, grid, st); break;
        case 12: moments_variant<B, 12>(buckets, n_buckets, cpb, tcheb, y1c, y2, N, mom, nbmax, grid, st); break;
        default: moments_variant<B, 16>(buckets, n_buckets, cpb, tcheb, y1c, y2, N, mom, nbmax, grid, st); break;
    }
}

template <int R>
void evaluate_variant(const Bucket* buckets, const int* n_buckets, int* queue, int max_buckets,
                      const int* sorted, const double* fdoa, double fs, const double* nu_c, int B,
                      const float2* mom, int nbmax, double* s_out, uint32_t* flag_bits,
                      int64_t flag_base, float tau, int sm_count, cudaStream_t st) {
    auto kern = k_evaluate<R, 8>;
    const size_t smem = evaluate_smem(nbmax, R);
    static size_t attr = 0;
    if (smem > attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = smem;
    }
    int grid = sm_count * 4;
    if (grid > max_buckets) grid = max_buckets > 0 ? max_buckets : 1;
    kern<<<grid, 32 * kEvalWarps, smem, st>>>(buckets, n_buckets, queue, sorted, fdoa, fs, nu_c,
                                              B, mom, nbmax, s_out, flag_bits, flag_base, tau);
}

}  // namespace

void launch_center(const double2* y, int N, const double* nu_c, float2* out, cudaStream_t st) {
    int blocks = (N + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    k_center<<<blocks, 256, 0, st>>>(y, N, nu_c, out);
}

void launch_work_count(const Bucket* buckets, const int* n_buckets, int B, int R,
                       unsigned long long* work, cudaStream_t st) {
    k_work_count<<<64, 256, 0, st>>>(buckets, n_buckets, B, R, work);
}

size_t moments_smem_bytes(int B) { return moments_smem(B); }

void launch_moments(int B, int R, const Bucket* buckets, const int* n_buckets, int cpb,
                    const float* tcheb, const float2* y1c, const float2* y2, int N, float2* mom,
                    int nbmax, int sm_count, cudaStream_t st) {
    const int grid = sm_count * 2;
    switch (B) {
        case 64: moments_b<64>(R, buckets, n_buckets, cpb, tcheb, y1c, y2, N, mom, nbmax, grid, st); break;
        case 128: moments_b<128>(R, buckets, n_buckets, cpb, tcheb, y1c, y2, N, mom, nbmax, grid, st); break;
        default: moments_b<256>(R, buckets, n_buckets, cpb, tcheb, y1c, y2, N, mom, nbmax, grid, st); break;
    }
}

size_t evaluate_smem_bytes(int nbmax, int R) { return evaluate_smem(nbmax, R); }

void launch_evaluate(int R, const Bucket* buckets, const int* n_buckets, int* queue,
                     int max_buckets, const int* sorted, const double* fdoa, double fs,
                     const double* nu_c, int B, const float2* mom, int nbmax, double* s_out,
                     uint32_t* flag_bits, int64_t flag_base, float tau, int sm_count,
                     cudaStream_t st) {
#define DG_EVAL_CASE(RR)                                                                    \
    evaluate_variant<RR>(buckets, n_buckets, queue, max_buckets, sorted, fdoa, fs, nu_c, B, \
                         mom, nbmax, s_out, flag_bits, flag_base, tau, sm_count, st)
    switch (R) {
        case 8: DG_EVAL_CASE(8); break;
        case 10: DG_EVAL_CASE(10); break;
        case 12: DG_EVAL_CASE(12); break;
        default: DG_EVAL_CASE(16); break;
    }
#undef DG_EVAL_CASE
}

}  // namespace dg
