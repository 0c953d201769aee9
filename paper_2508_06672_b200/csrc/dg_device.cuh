// Device helpers shared by the correlator kernels (dg_moments.cu, dg_nufft.cu):
// packed FP32x2 FMAs, 1-D TMA bulk copies with mbarrier completion, Bessel
// functions for the Jacobi-Anger coefficients. Internal; not installed.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

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
[[maybe_unused]] __device__ __forceinline__ void cis_cycles(double x, float* c, float* s) {
    sincospif((float)(2.0 * (x - rint(x))), s, c);
}

// TMA helpers (1-D bulk copy global -> shared, mbarrier completion)
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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// J_0..J_{R-1}(x) (first kind), FP64: series for J_{R-1}, J_R (fast: m >> x),
// then the stable backward recurrence J_{m-1} = (2m/x) J_m - J_{m+1}. The series
// J_n = (h^n / n!) sum_k a_k (h^2)^k, a_k = prod_{i<=k} -1 / (i (n + i)), h = x/2,
// run as Horner polynomials in h^2 with compile-time coefficients (one DFMA per
// term), h^n by repeated squaring.
struct JSeries {
    double a[13];  // a_0 .. a_12
    double inv_fact;
};
__host__ __device__ constexpr JSeries jseries_coefs(int n) {
    JSeries c{};
    double a = 1.0;
    c.a[0] = 1.0;
    for (int k = 1; k <= 12; ++k) {
        a *= -1.0 / ((double)k * (double)(n + k));
        c.a[k] = a;
    }
    double f = 1.0;
    for (int i = 2; i <= n; ++i) f /= (double)i;
    c.inv_fact = f;
    return c;
}
template <int E>
__device__ __forceinline__ double ipow(double h) {  // h^E, E >= 0
    if constexpr (E == 0) {
        return 1.0;
    } else if constexpr (E == 1) {
        return h;
    } else {
        const double q = ipow<E / 2>(h);
        return (E & 1) ? q * q * h : q * q;
    }
}
template <int N>
__device__ __forceinline__ double jseries(double h, double h2) {  // J_N(2h), |h| <~ 2
    constexpr JSeries C = jseries_coefs(N);
    double p = C.a[12];
#pragma unroll
    for (int k = 11; k >= 0; --k) p = fma(p, h2, C.a[k]);
    return ipow<N>(h) * C.inv_fact * p;
}
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
    const double jr1 = jseries<R - 1>(h, h2);  // J_{R-1}
    const double jr = jseries<R>(h, h2);       // J_R
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

// a bucket's ||z||_2^2 estimate from the captures' |y|^2 prefix sums: sum over its
// blocks (absolute index, length B, clipped to the overlap [kb, ke)) of
// E1_b E2_b / len_b — exact when either capture has a constant envelope within
// a block; the moment path's refinement floor. Threads t < nt of a group each
// take blocks t, t + nt, ...; the caller reduces the partial sums in order.
__device__ __forceinline__ double bucket_z2_part(const double* __restrict__ e1,
                                                 const double* __restrict__ e2, int N, int d,
                                                 int B, int t, int nt) {
    const int kb = d < 0 ? -d : 0, ke = d > 0 ? N - d : N;
    double acc = 0.0;
    for (int b = kb / B + t; b * B < ke; b += nt) {
        const int lo = max(kb, b * B), hi = min(ke, (b + 1) * B);
        if (lo >= hi) continue;
        const double E1 = e1[hi] - e1[lo], E2 = e2[hi + d] - e2[lo + d];
        acc = fma(E1, E2 / (double)(hi - lo), acc);
    }
    return acc;
}

// The block-moment refinement test. coh in [0, 1] is the
// bucket's coherence: 0 when its moments carry only the energy an incoherent
// (noise) product stream gives them, rho = sum_m Q_m^2 / <T_m^2> / (R ||z||_2^2)
// ~ 1, and 1 from rho >= 1.5 on (a tone, or a chirp product aliasing onto the
// block length, makes some moments coherent). The FP32 value S is re-evaluated
// when it is small next to the noise floor ||z||_2 (tau_noise for incoherent
// buckets, whose rounding has a ~3x smaller constant, rising to tau) or next
// to the coherent part of its error scales, sqrt(max(en, qe2) - (1 - coh) zfloor)
// (tau); a fully coherent bucket gets S < tau sqrt(max(en, qe2, zfloor)).
__device__ __forceinline__ double bucket_coherence(const float* qm2, int R, double zfloor) {
    double q = 0.0;
    for (int m = 0; m < R; ++m) q += (m ? 2.0 : 1.0) * (double)qm2[m];  // <T_0^2> = 1, <T_m^2> ~ 1/2
    const double rho = zfloor > 0.0 ? q / ((double)R * zfloor) : 1.0;
    return fmin(fmax((rho - 1.0) * 2.0, 0.0), 1.0);
}

// per-bucket constants of the test, compared on S^2 (no square roots per candidate)
struct RefineBucket {
    double thr0;  // (tau_f)^2 zfloor
    double base;  // (1 - coh) zfloor
    double tau2;  // tau^2
};
__device__ __forceinline__ RefineBucket refine_bucket(double zfloor, double coh, float tau,
                                                      float tau_noise) {
    const double tf = (double)tau_noise + ((double)tau - (double)tau_noise) * coh;
    return RefineBucket{tf * tf * zfloor, (1.0 - coh) * zfloor, (double)tau * (double)tau};
}
// S < tau_f sqrt(zfloor)  or  S < tau sqrt(max(en, qe2) - (1 - coh) zfloor), on s2 = S^2
__device__ __forceinline__ bool refine_moment(double s2, double en, double qe2,
                                              const RefineBucket& r) {
    const double ex = fmax(fmax(en, qe2) - r.base, 0.0);
    return s2 < r.thr0 || s2 < r.tau2 * ex;
}

__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\t"
        "mov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\t"
        "mov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}

__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\t"
        "mov.b64 rb, {%4, %5};\n\t"
        "sub.rn.f32x2 rd, ra, rb;\n\t"
        "mov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}

__device__ __forceinline__ float2 fmul2(float2 a, float b) {  // a * {b, b}
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\t"
        "mov.b64 rb, {%4, %4};\n\t"
        "mul.rn.f32x2 rd, ra, rb;\n\t"
        "mov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b));
    return d;
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


}  // namespace
}  // namespace dg
