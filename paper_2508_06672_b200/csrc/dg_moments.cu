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
            dst[o] = s;
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

template <int R, int G>
__global__ void __launch_bounds__(128, 4)
k_evaluate(const Task* __restrict__ tasks, const int* __restrict__ n_tasks,
           const Bucket* __restrict__ buckets, const int* __restrict__ sorted,
           const double* __restrict__ fdoa, double fs, const double* __restrict__ nu_c_p, int B,
           const float2* __restrict__ mom, int nbmax,
           double* __restrict__ s_out, uint32_t* __restrict__ flag_bits, int64_t flag_base,
           float tau) {
    constexpr int NC = 2;
    const int lane = threadIdx.x & 31;
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (t >= *n_tasks) return;
    const Task tk = tasks[t];
    const int u = tk.pad;
    const Bucket bk = buckets[u];
    const int nb = bk.nb;
    const double nu_c = *nu_c_p;

    int p[NC];
    double nu[NC];
    float cf[NC][R];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const int slot = lane + 32 * c;
        p[c] = slot < tk.count ? sorted[tk.start + slot] : -1;
        nu[c] = p[c] >= 0 ? fdoa[p[c]] / fs - nu_c : 0.0;
        double jv[R];
        bessel_j<R>(3.141592653589793 * nu[c] * (double)B, jv);
        // a_m = (2 - delta_m0) i^m J_m: even m -> real part sign (+,-,+,...),
        // odd m -> imaginary part sign (+,-,...)
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const double sg = ((m >> 1) & 1) ? -1.0 : 1.0;
            cf[c][m] = (float)((m == 0 ? 1.0 : 2.0) * sg * jv[m]);
        }
    }

    // W_j = e^{i 2 pi nu B j}, j < G: each rounded once from an FP64 phase, so
    // the group sum sum_j W_j C_{gG+j} has no recurrence error
    float wtr[NC][G], wti[NC][G];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int j = 0; j < G; ++j) cis_cycles(nu[c] * (double)B * (double)j, &wtr[c][j], &wti[c][j]);

    double acc_re[NC], acc_im[NC], en[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc_re[c] = acc_im[c] = en[c] = 0.0;
    const float4* mb = reinterpret_cast<const float4*>(mom + (size_t)u * nbmax * R);
    const int ng = (nb + G - 1) / G;
    for (int g = 0; g < ng; ++g) {
        float hr[NC], hi[NC], ge[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) hr[c] = hi[c] = ge[c] = 0.f;
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const int b = g * G + j;
            if (b < nb) {
                float4 mv[R / 2];
#pragma unroll
                for (int q = 0; q < R / 2; ++q) mv[q] = __ldg(mb + (size_t)b * (R / 2) + q);
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    // C_b = E + iO, smallest terms first (the c_m decay with m)
                    float2 E = make_float2(0.f, 0.f), O = make_float2(0.f, 0.f);
#pragma unroll
                    for (int q = R / 2 - 1; q >= 0; --q) {
                        E = ffma2(make_float2(mv[q].x, mv[q].y), cf[c][2 * q], E);
                        O = ffma2(make_float2(mv[q].z, mv[q].w), cf[c][2 * q + 1], O);
                    }
                    const float cr = E.x - O.y, ci = E.y + O.x;
                    hr[c] = fmaf(wtr[c][j], cr, fmaf(-wti[c][j], ci, hr[c]));
                    hi[c] = fmaf(wtr[c][j], ci, fmaf(wti[c][j], cr, hi[c]));
                    ge[c] = fmaf(cr, cr, fmaf(ci, ci, ge[c]));
                }
            }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            float ar, ai;
            cis_cycles(nu[c] * (double)(g * G) * (double)B, &ar, &ai);
            acc_re[c] += (double)fmaf(ar, hr[c], -(ai * hi[c]));
            acc_im[c] += (double)fmaf(ar, hi[c], ai * hr[c]);
            en[c] += (double)ge[c];
        }
    }

    // FP32 error scale of this candidate: sqrt(sum_b |C_b|^2) (DESIGN.md
    // section 5); below tau of it the value is re-evaluated in FP64
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        if (p[c] < 0) continue;
        const double s = sqrt(acc_re[c] * acc_re[c] + acc_im[c] * acc_im[c]);
        s_out[p[c]] = s;
        if (s < (double)tau * sqrt(en[c])) {
            const int64_t e = flag_base + p[c];
            atomicOr(&flag_bits[e >> 5], 1u << (e & 31));
        }
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
void evaluate_variant(int max_tasks, const Task* tasks, const int* n_tasks, const Bucket* buckets,
                      const int* sorted, const double* fdoa, double fs, const double* nu_c, int B,
                      const float2* mom, int nbmax, double* s_out,
                      uint32_t* flag_bits, int64_t flag_base, float tau, cudaStream_t st) {
    constexpr int kWarps = 4;
    const int blocks = (max_tasks + kWarps - 1) / kWarps;
    k_evaluate<R, 8><<<blocks, 32 * kWarps, 0, st>>>(tasks, n_tasks, buckets, sorted, fdoa, fs,
                                                     nu_c, B, mom, nbmax, s_out,
                                                     flag_bits, flag_base, tau);
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

void launch_evaluate(int R, int max_tasks, const Task* tasks, const int* n_tasks,
                     const Bucket* buckets, const int* sorted, const double* fdoa, double fs,
                     const double* nu_c, int B, const float2* mom, int nbmax, double* s_out, uint32_t* flag_bits, int64_t flag_base, float tau,
                     cudaStream_t st) {
    if (max_tasks <= 0) return;
    switch (R) {
        case 8: evaluate_variant<8>(max_tasks, tasks, n_tasks, buckets, sorted, fdoa, fs, nu_c, B, mom, nbmax, s_out, flag_bits, flag_base, tau, st); break;
        case 10: evaluate_variant<10>(max_tasks, tasks, n_tasks, buckets, sorted, fdoa, fs, nu_c, B, mom, nbmax, s_out, flag_bits, flag_base, tau, st); break;
        case 12: evaluate_variant<12>(max_tasks, tasks, n_tasks, buckets, sorted, fdoa, fs, nu_c, B, mom, nbmax, s_out, flag_bits, flag_base, tau, st); break;
        default: evaluate_variant<16>(max_tasks, tasks, n_tasks, buckets, sorted, fdoa, fs, nu_c, B, mom, nbmax, s_out, flag_bits, flag_base, tau, st); break;
    }
}

}  // namespace dg
