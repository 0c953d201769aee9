// Warp-level 1024-point complex FFT in FP32 (the block moments' cross-correlation
// form, dg_moments_fft.cu).
//
// Distribution: element n of the 1024-vector lives in lane (n mod 32), register
// v[n / 32] — on input and on output alike. 1024 = 32 x 32 (four-step):
//   pass 1  each lane a 32-point FFT over its own registers (n = lane + 32 n2):
//           Y_lane[k2]
//   twiddle Y_lane[k2] *= w^(lane k2)  (w = e^(-+2 pi i / 1024), a 32 x 32 table in
//           shared memory, FP64-evaluated then rounded once)
//   transpose through a 32 x 33 shared buffer (lane k2 now holds Y_n1[k2], n1 = 0..31)
//   pass 2  each lane a 32-point FFT over n1: X[lane + 32 k1] in v[k1].
// The 32-point FFTs are radix-2 DIT on registers with compile-time twiddles.
// Forward: X[k] = sum_n x[n] e^(-2 pi i n k / 1024); inverse: e^(+...), unscaled.
#pragma once
#include <cuda_runtime.h>

namespace dg {

// cos(2 pi j / 32), j = 0..15 (exact 0 / 1 where due); the forward twiddle e^(-2 pi i j / 32)
// is (tw32_c, -tw32_s)
__host__ __device__ constexpr float tw32_c(int j) {
    return j == 0   ? 1.0f
           : j == 1 ? (float)0.98078528040323043
           : j == 2 ? (float)0.92387953251128674
           : j == 3 ? (float)0.83146961230254524
           : j == 4 ? (float)0.70710678118654752
           : j == 5 ? (float)0.55557023301960218
           : j == 6 ? (float)0.38268343236508977
           : j == 7 ? (float)0.19509032201612826
           : j == 8 ? 0.0f
           : j == 9 ? (float)-0.19509032201612826
           : j == 10 ? (float)-0.38268343236508977
           : j == 11 ? (float)-0.55557023301960218
           : j == 12 ? (float)-0.70710678118654752
           : j == 13 ? (float)-0.83146961230254524
           : j == 14 ? (float)-0.92387953251128674
                     : (float)-0.98078528040323043;
}
// sin(2 pi j / 32) = cos(2 pi |j - 8| / 32)
__host__ __device__ constexpr float tw32_s(int j) { return tw32_c(j < 8 ? 8 - j : j - 8); }

// packed FP32x2 add / subtract (one FADD2 instead of two FADD)
__device__ __forceinline__ float2 fft_add2(float2 a, float2 b) {
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
__device__ __forceinline__ float2 fft_sub2(float2 a, float2 b) {
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

// one radix-2 DIT stage of span M (compile-time, so every index is a register)
template <bool INV, int M>
__device__ __forceinline__ void fft32_stage(float2 (&x)[32]) {
    constexpr int H = M / 2;
#pragma unroll
    for (int k = 0; k < 32; k += M) {
#pragma unroll
        for (int j = 0; j < H; ++j) {
            const int e = j * (32 / M);  // twiddle index of e^(-+2 pi i j / M)
            const float wc = tw32_c(e), ws = INV ? tw32_s(e) : -tw32_s(e);
            const float2 b = x[k + j + H];
            float2 t;
            if (e == 0) {
                t = b;
            } else if (e == 8) {  // multiply by -+i
                t = INV ? make_float2(-b.y, b.x) : make_float2(b.y, -b.x);
            } else {
                t = make_float2(fmaf(wc, b.x, -ws * b.y), fmaf(wc, b.y, ws * b.x));
            }
            const float2 a = x[k + j];
            x[k + j] = fft_add2(a, t);
            x[k + j + H] = fft_sub2(a, t);
        }
    }
}

// 32-point FFT on registers, natural order in and out. INV: e^(+...).
template <bool INV>
__device__ __forceinline__ void fft32(float2 (&x)[32]) {
    // bit-reversal permutation (register renaming after unrolling)
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const int r = ((i & 1) << 4) | ((i & 2) << 2) | (i & 4) | ((i & 8) >> 2) | ((i & 16) >> 4);
        if (r > i) {
            const float2 t = x[i];
            x[i] = x[r];
            x[r] = t;
        }
    }
    fft32_stage<INV, 2>(x);
    fft32_stage<INV, 4>(x);
    fft32_stage<INV, 8>(x);
    fft32_stage<INV, 16>(x);
    fft32_stage<INV, 32>(x);
}

// tw[k2 * 32 + n1] = e^(-2 pi i n1 k2 / 1024) (forward); conjugated for INV.
// xbuf: this warp's 32 x 33 float2 transpose buffer.
template <bool INV>
__device__ __forceinline__ void fft1024_warp(float2 (&v)[32], const float2* __restrict__ tw,
                                             float2* __restrict__ xbuf, int lane) {
    fft32<INV>(v);
#pragma unroll
    for (int k2 = 1; k2 < 32; ++k2) {
        const float2 w = tw[k2 * 32 + lane];
        const float ws = INV ? -w.y : w.y;
        const float2 a = v[k2];
        v[k2] = make_float2(fmaf(w.x, a.x, -ws * a.y), fmaf(w.x, a.y, ws * a.x));
    }
    __syncwarp();
#pragma unroll
    for (int k2 = 0; k2 < 32; ++k2) xbuf[k2 * 33 + lane] = v[k2];
    __syncwarp();
#pragma unroll
    for (int n1 = 0; n1 < 32; ++n1) v[n1] = xbuf[lane * 33 + n1];
    fft32<INV>(v);
}

// fill tw[k2 * 32 + n1] = e^(-2 pi i n1 k2 / 1024) (FP64 evaluation, one rounding)
__device__ __forceinline__ void fft1024_twiddles(float2* tw, int tid, int nthreads) {
    for (int i = tid; i < 1024; i += nthreads) {
        const int k2 = i >> 5, n1 = i & 31;
        double s, c;
        sincospi(-2.0 * (double)(n1 * k2) / 1024.0, &s, &c);
        tw[i] = make_float2((float)c, (float)s);
    }
}

}  // namespace dg
