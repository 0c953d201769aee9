// Output writers from device memory (reference io.hpp:171-280):
// byte-identical CSV surfaces ("%.17g,%.17g,%.17g\n" per cell, io.hpp:174-183)
// and P5 heatmaps (io.hpp:245-268) formatted on the GPU, so a 4M-cell surface
// never round-trips through host snprintf. The binary DGGR layout (io.hpp:187-202)
// needs no formatting and is written by the host side (dg_io.cpp) straight
// from a pinned copy of the device values.
//
// "%.17g" is reproduced exactly (glibc: correctly rounded, ties to even, "%g"
// style selection and trailing-zero removal) with exact big-integer arithmetic:
// for v = m 2^q, the 17 significant digits are floor(v 10^(16-E)) with
// E = floor(log10 v); the scaling is a multiply by 10^k and a right shift by
// -q (v < 1e17) or a division by 10^j (v >= 1e17, then v is an integer).
// HBM-bound formatting: one thread per number, 32-byte slots, then one thread
// per CSV row gathers its three slots at the row's scanned offset.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/cub.cuh>

#include "dg_internal.cuh"

namespace dg {

namespace {

constexpr int kLimbs = 40;  // 1280 bits: m 10^340 (subnormals) and m 2^971 fit

struct Big {
    uint32_t w[kLimbs];
    int n;
};

__device__ void big_mul_small(Big& b, uint32_t f) {
    uint64_t carry = 0;
    for (int i = 0; i < b.n; ++i) {
        const uint64_t t = (uint64_t)b.w[i] * f + carry;
        b.w[i] = (uint32_t)t;
        carry = t >> 32;
    }
    if (carry) b.w[b.n++] = (uint32_t)carry;
}

__device__ void big_shl(Big& b, int s) {
    const int words = s >> 5, bits = s & 31;
    if (bits) {
        uint32_t carry = 0;
        for (int i = 0; i < b.n; ++i) {
            const uint32_t v = b.w[i];
            b.w[i] = (v << bits) | carry;
            carry = v >> (32 - bits);
        }
        if (carry) b.w[b.n++] = carry;
    }
    if (words) {
        for (int i = b.n - 1; i >= 0; --i) b.w[i + words] = b.w[i];
        for (int i = 0; i < words; ++i) b.w[i] = 0;
        b.n += words;
    }
}

__device__ uint32_t big_div_small(Big& b, uint32_t d) {  // b /= d, returns b % d
    uint64_t r = 0;
    for (int i = b.n - 1; i >= 0; --i) {
        const uint64_t cur = (r << 32) | b.w[i];
        b.w[i] = (uint32_t)(cur / d);
        r = cur % d;
    }
    while (b.n > 0 && b.w[b.n - 1] == 0) --b.n;
    return (uint32_t)r;
}

__device__ uint32_t big_bit(const Big& b, int i) {
    const int w = i >> 5;
    return w < b.n ? (b.w[w] >> (i & 31)) & 1u : 0u;
}

__device__ bool big_any_below(const Big& b, int nbits) {  // any of bits [0, nbits) set
    const int full = nbits >> 5;
    for (int i = 0; i < full && i < b.n; ++i)
        if (b.w[i]) return true;
    const int rem = nbits & 31;
    if (rem && full < b.n && (b.w[full] & ((1u << rem) - 1u))) return true;
    return false;
}

__device__ uint64_t big_bits64(const Big& b, int s) {  // bits [s, s + 64)
    uint64_t r = 0;
    const int w = s >> 5, off = s & 31;
    for (int k = 0; k < 3; ++k) {
        const int i = w + k;
        if (i >= b.n) break;
        const int at = 32 * k - off;
        if (at >= 64) break;
        r |= at >= 0 ? (uint64_t)b.w[i] << at : (uint64_t)b.w[i] >> (-at);
    }
    return r;
}

__device__ const uint32_t kPow10[10] = {1u,      10u,      100u,      1000u,      10000u,
                                         100000u, 1000000u, 10000000u, 100000000u, 1000000000u};

// floor(|v| 10^(16-E)) for v = m 2^q, with the rounding decision for the
// discarded part (round to nearest, ties to even): returns the digits and
// sets *up when the 17-digit value must be incremented.
__device__ uint64_t scaled_digits(uint64_t m, int q, int E, bool* up) {
    Big b;
    b.w[0] = (uint32_t)m;
    b.w[1] = (uint32_t)(m >> 32);
    b.n = b.w[1] ? 2 : 1;
    const int k = 16 - E;
    if (k >= 0) {
        for (int t = k; t > 0; t -= 9) big_mul_small(b, kPow10[t >= 9 ? 9 : t]);
        if (q >= 0) {
            big_shl(b, q);
            *up = false;
            return big_bits64(b, 0);
        }
        const int s = -q;
        const uint64_t d = big_bits64(b, s);
        const bool half = big_bit(b, s - 1);
        const bool sticky = big_any_below(b, s - 1);
        *up = half && (sticky || (d & 1));
        return d;
    }
    // v >= 1e17: an integer (q >= 4); divide by 10^(j-1) keeping a sticky bit,
    // then the last digit decides the rounding
    big_shl(b, q);
    bool sticky = false;
    for (int t = -k - 1; t > 0; t -= 9) sticky |= big_div_small(b, kPow10[t >= 9 ? 9 : t]) != 0;
    const uint64_t qd = big_bits64(b, 0);
    const uint64_t d = qd / 10, last = qd % 10;
    *up = last > 5 || (last == 5 && (sticky || (d & 1)));
    return d;
}

}  // namespace

// "%.17g" of v into out (no terminator); returns the length (<= 24)
__device__ int format_g17(double v, char* out) {
    const uint64_t bits = (uint64_t)__double_as_longlong(v);
    const bool neg = bits >> 63;
    const int ex = (int)((bits >> 52) & 0x7ff);
    const uint64_t frac = bits & ((1ull << 52) - 1);
    int n = 0;
    if (neg) out[n++] = '-';
    if (ex == 0x7ff) {
        const char* t = frac ? "nan" : "inf";
        for (int i = 0; i < 3; ++i) out[n++] = t[i];
        return n;
    }
    if (ex == 0 && frac == 0) {
        out[n++] = '0';
        return n;
    }
    const uint64_t m = ex ? (frac | (1ull << 52)) : frac;
    const int q = ex ? ex - 1075 : -1074;
    int E = (int)floor(log10(fabs(v)));
    bool up = false;
    uint64_t d = 0;
    for (int it = 0; it < 4; ++it) {  // the log10 estimate may be one off
        d = scaled_digits(m, q, E, &up);
        if (d >= 100000000000000000ull) {
            ++E;
        } else if (d < 10000000000000000ull) {
            --E;
        } else {
            break;
        }
    }
    if (up && ++d == 100000000000000000ull) {
        d = 10000000000000000ull;
        ++E;
    }
    char dg[17];
    for (int i = 16; i >= 0; --i) {
        dg[i] = (char)('0' + d % 10);
        d /= 10;
    }
    int nd = 17;
    while (nd > 1 && dg[nd - 1] == '0') --nd;
    if (E < -4 || E >= 17) {  // %e style
        out[n++] = dg[0];
        if (nd > 1) {
            out[n++] = '.';
            for (int i = 1; i < nd; ++i) out[n++] = dg[i];
        }
        out[n++] = 'e';
        out[n++] = E < 0 ? '-' : '+';
        const int a = E < 0 ? -E : E;
        if (a >= 100) out[n++] = (char)('0' + a / 100);
        out[n++] = (char)('0' + (a / 10) % 10);
        out[n++] = (char)('0' + a % 10);
    } else if (E >= 0) {  // %f style, E + 1 integer digits
        for (int i = 0; i <= E; ++i) out[n++] = dg[i];
        if (nd > E + 1) {
            out[n++] = '.';
            for (int i = E + 1; i < nd; ++i) out[n++] = dg[i];
        }
    } else {  // 0.000ddd
        out[n++] = '0';
        out[n++] = '.';
        for (int i = 0; i < -E - 1; ++i) out[n++] = '0';
        for (int i = 0; i < nd; ++i) out[n++] = dg[i];
    }
    return n;
}

namespace {

// axis value i = start + i * step (GridAxis::value, geodesy.hpp:145), no contraction
__global__ void k_format_axis(double start, double step, int64_t first, int64_t count,
                              char* __restrict__ slots, uint8_t* __restrict__ len) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double v = __dadd_rn(start, __dmul_rn((double)(first + i), step));
        len[i] = (uint8_t)format_g17(v, slots + i * kFmtSlot);
    }
}

__global__ void k_format_values(const double* __restrict__ v, int64_t n, char* __restrict__ slots,
                                uint8_t* __restrict__ len) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        len[i] = (uint8_t)format_g17(v[i], slots + i * kFmtSlot);
}

__global__ void k_csv_row_len(const uint8_t* __restrict__ lat_len, const uint8_t* __restrict__ lon_len,
                              const uint8_t* __restrict__ val_len, int64_t n_lat, int64_t n_lon,
                              int64_t* __restrict__ row_len) {
    const int64_t n = n_lat * n_lon;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
         c += (int64_t)gridDim.x * blockDim.x)
        row_len[c] = (int64_t)lat_len[c / n_lon] + lon_len[c % n_lon] + val_len[c] + 3;
}

__device__ __forceinline__ char* put_slot(char* dst, const char* slot, int len) {
    for (int i = 0; i < len; ++i) dst[i] = slot[i];
    return dst + len;
}

// row c at out[base + end[c] - row_len(c)]: "<lat>,<lon>,<value>\n"
__global__ void k_csv_rows(const char* __restrict__ lat_s, const uint8_t* __restrict__ lat_len,
                           const char* __restrict__ lon_s, const uint8_t* __restrict__ lon_len,
                           const char* __restrict__ val_s, const uint8_t* __restrict__ val_len,
                           const int64_t* __restrict__ end, int64_t n_lat, int64_t n_lon,
                           char* __restrict__ out) {
    const int64_t n = n_lat * n_lon;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = c / n_lon, j = c % n_lon;
        const int la = lat_len[i], lo = lon_len[j], va = val_len[c];
        char* p = out + end[c] - (la + lo + va + 3);
        p = put_slot(p, lat_s + i * kFmtSlot, la);
        *p++ = ',';
        p = put_slot(p, lon_s + j * kFmtSlot, lo);
        *p++ = ',';
        p = put_slot(p, val_s + c * kFmtSlot, va);
        *p = '\n';
    }
}

// exact FP64 min / max (order-independent), per-block partials then one block
__global__ void k_minmax_partial(const double* __restrict__ v, int64_t n, double2* __restrict__ part) {
    double lo = v[0], hi = v[0];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        lo = fmin(lo, v[i]);
        hi = fmax(hi, v[i]);
    }
    __shared__ double slo[256], shi[256];
    slo[threadIdx.x] = lo;
    shi[threadIdx.x] = hi;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            slo[threadIdx.x] = fmin(slo[threadIdx.x], slo[threadIdx.x + s]);
            shi[threadIdx.x] = fmax(shi[threadIdx.x], shi[threadIdx.x + s]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = make_double2(slo[0], shi[0]);
}

__global__ void k_minmax_final(const double2* __restrict__ part, int n, double2* __restrict__ out) {
    double lo = part[0].x, hi = part[0].y;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        lo = fmin(lo, part[i].x);
        hi = fmax(hi, part[i].y);
    }
    __shared__ double slo[256], shi[256];
    slo[threadIdx.x] = lo;
    shi[threadIdx.x] = hi;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            slo[threadIdx.x] = fmin(slo[threadIdx.x], slo[threadIdx.x + s]);
            shi[threadIdx.x] = fmax(shi[threadIdx.x], shi[threadIdx.x + s]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = make_double2(slo[0], shi[0]);
}

// render_heatmap pixels (io.hpp:258-266): north row first, llround((v - lo) * scale),
// 16-bit big-endian; `scale` is computed by the host exactly as the reference
__global__ void k_heatmap(const double* __restrict__ v, int64_t n_lat, int64_t n_lon, double lo,
                          double scale, uint8_t* __restrict__ out) {
    const int64_t n = n_lat * n_lon;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = c / n_lon, j = c % n_lon;
        const double x = v[(n_lat - 1 - row) * n_lon + j];
        const uint32_t px = (uint32_t)llround(__dmul_rn(__dsub_rn(x, lo), scale));
        out[2 * c] = (uint8_t)((px >> 8) & 0xFF);
        out[2 * c + 1] = (uint8_t)(px & 0xFF);
    }
}

int grid_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    return (int)(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

}  // namespace

void launch_format_axis(double start, double step, int64_t first, int64_t count, char* slots,
                        uint8_t* len, cudaStream_t st) {
    k_format_axis<<<grid_for(count), 256, 0, st>>>(start, step, first, count, slots, len);
}

void launch_format_values(const double* v, int64_t n, char* slots, uint8_t* len, cudaStream_t st) {
    k_format_values<<<grid_for(n), 256, 0, st>>>(v, n, slots, len);
}

size_t csv_scan_temp_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, bytes, (const int64_t*)nullptr, (int64_t*)nullptr, n);
    return bytes;
}

void launch_csv_offsets(const uint8_t* lat_len, const uint8_t* lon_len, const uint8_t* val_len,
                        int64_t n_lat, int64_t n_lon, int64_t* row_len, int64_t* row_end,
                        void* temp, size_t temp_bytes, cudaStream_t st) {
    const int64_t n = n_lat * n_lon;
    k_csv_row_len<<<grid_for(n), 256, 0, st>>>(lat_len, lon_len, val_len, n_lat, n_lon, row_len);
    cub::DeviceScan::InclusiveSum(temp, temp_bytes, row_len, row_end, n, st);
}

void launch_csv_emit(const char* lat_s, const uint8_t* lat_len, const char* lon_s,
                     const uint8_t* lon_len, const char* val_s, const uint8_t* val_len,
                     const int64_t* row_end, int64_t n_lat, int64_t n_lon, char* out,
                     cudaStream_t st) {
    k_csv_rows<<<grid_for(n_lat * n_lon), 256, 0, st>>>(lat_s, lat_len, lon_s, lon_len, val_s,
                                                         val_len, row_end, n_lat, n_lon, out);
}

void launch_minmax(const double* v, int64_t n, double2* part, double2* out, cudaStream_t st) {
    const int blocks = 256;
    k_minmax_partial<<<blocks, 256, 0, st>>>(v, n, part);
    k_minmax_final<<<1, 256, 0, st>>>(part, blocks, out);
}

void launch_heatmap(const double* v, int64_t n_lat, int64_t n_lon, double lo, double scale,
                    uint8_t* out, cudaStream_t st) {
    k_heatmap<<<grid_for(n_lat * n_lon), 256, 0, st>>>(v, n_lat, n_lon, lo, scale, out);
}

}  // namespace dg
