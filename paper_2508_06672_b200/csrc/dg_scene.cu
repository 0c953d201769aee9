// Capture synthesis on the device (reference scene.hpp:200-310,
// waveform.hpp:124-204, fft.hpp:39-75). The host side (dg_scene.cpp) restates the
// scenario arithmetic (epochs, orbits, geometry, pads, delays, amplitudes, seeds)
// with the reference's own operation order; these kernels do the per-sample work:
//
//   k_waveform        transmit record of one (snapshot, emitter): spoofer (C/A chips x
//                     seeded nav bits, exact), tone / chirp / sawtooth (FP64 phase,
//                     device cos/sin)
//   fractional advance (scene.hpp:161-191) as a four-step FFT of N = N1 x N2 points,
//                     FP64, the record viewed as an [N1][N2] matrix:
//     k_fft_cols_fwd  Hann-tapered, zero-padded columns -> length-N1 DFTs, x w^(n2 k1)
//     k_fft_rows_fwd  rows -> length-N2 DFTs: position (k1, k2) holds X[k1 + N1 k2]
//                     (the forward spectrum is shared by every receiver)
//     k_fft_rows_inv  per receiver: x e^{i 2 pi f frac}, inverse row DFTs, x w^(-n2 k1)
//     k_fft_cols_inv  inverse column DFTs -> natural order, / N, and straight into the
//                     received samples amplitude * delayed[shift + k] * phasor_k
//   k_phasors         phasor_k by the reference's own recurrence (phasor *= rotation,
//                     exact complex products from the host's rotation)
//   k_noise_combine   per (snapshot, receiver): sum of the emitters' received samples in
//                     emitter order, plus sigma x Box-Muller on MT19937-64 (exact integer
//                     stream, twisted by a CTA in two parallel halves)
// Every complex product / sum is spelled with _rn intrinsics (no FMA contraction), so
// results differ from the reference only where a transcendental (cos, sin, log, sqrt
// of the Box-Muller radius) or the FFT's rounding differs: parity to tolerance.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dg_internal.cuh"

namespace dg {

namespace {

constexpr double kPi = 3.141592653589793;
constexpr int kFftThreads = 256;
constexpr int kColTile = 4;  // columns per CTA in the column passes

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {  // (ac - bd, ad + bc)
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
    return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
    return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
__device__ __forceinline__ double2 cscale(double s, double2 a) {
    return make_double2(__dmul_rn(s, a.x), __dmul_rn(s, a.y));
}
__device__ __forceinline__ double2 polar1(double th) {  // std::polar(1.0, th)
    double s, c;
    sincos(th, &s, &c);
    return make_double2(c, s);
}
// e^{sign 2 pi i j / m} for an exact integer ratio (sincospi: exact argument)
__device__ __forceinline__ double2 root(int64_t j, int64_t m, double sign) {
    double s, c;
    sincospi(sign * 2.0 * (double)(j % m) / (double)m, &s, &c);
    return make_double2(c, s);
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {  // waveform.hpp:38-43
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__device__ __forceinline__ int64_t floor_index(double v) {  // waveform.hpp:54-56
    return (int64_t)floor(__dadd_rn(v, 1e-6));
}

// waveform.hpp:115-120
__device__ __forceinline__ double chirp_phase(double t, double bw, double period) {
    const double cycles = __ddiv_rn(t, period);
    const double u = __dmul_rn(__dsub_rn(cycles, floor(cycles)), period);
    const double a = __dmul_rn(__dmul_rn(__ddiv_rn(bw, __dmul_rn(2.0, period)), u), u);
    const double b = __dmul_rn(__dmul_rn(0.5, bw), u);
    return __dmul_rn(2.0 * kPi, __dsub_rn(a, b));
}

__global__ void k_waveform(WaveParams w, double start, double ts, int64_t n,
                           const int8_t* __restrict__ chips, double2* __restrict__ out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const double t = __dadd_rn(start, __dmul_rn((double)k, ts));
        double2 v;
        if (w.kind == kWaveSpoofer) {  // waveform.hpp:127-146
            const int64_t ci = floor_index(__dmul_rn(t, 1.023e6));
            const int64_t wrapped = ((ci % 1023) + 1023) % 1023;
            const double chip = (double)chips[wrapped];
            const int64_t bi = floor_index(__dmul_rn(t, 50.0));
            const uint64_t h = splitmix64(w.seed ^ ((uint64_t)bi * 0xD1B54A32D192ED03ull));
            const double bit = (h >> 63) ? -1.0 : 1.0;
            v = make_double2(__dmul_rn(chip, bit), 0.0);
        } else if (w.kind == kWaveTone) {  // :149-159
            v = polar1(__dmul_rn(__dmul_rn(2.0 * kPi, w.a), t));
        } else if (w.kind == kWaveChirp) {  // :162-175
            v = polar1(chirp_phase(t, w.a, w.b));
        } else {  // sawtooth, :179-197
            const double full = __dmul_rn(2.0, w.b);
            const double cycles = __ddiv_rn(t, full);
            const double u = __dmul_rn(__dsub_rn(cycles, floor(cycles)), full);
            const bool first = u < w.b;
            const double ph = chirp_phase(first ? u : __dsub_rn(u, w.b), w.a, w.b);
            v = polar1(first ? ph : -ph);
        }
        out[k] = v;
    }
}

// In-place radix-2 DIF FFTs of `count` sequences of length m = 2^logm held in
// shared memory, element i of sequence c at x[i * cstride + c * estride];
// twiddles tw[j] = e^{sign 2 pi i j / m}, j < m/2. Output in bit-reversed order.
__device__ void smem_fft(double2* x, int logm, int count, int cstride, int estride,
                         const double2* tw) {
    const int m = 1 << logm;
    const int half = m >> 1;
    for (int h = half, st = 1; h >= 1; h >>= 1, st <<= 1) {
        const int lh = __ffs(h) - 1;
        for (int t = threadIdx.x; t < count * half; t += blockDim.x) {
            const int c = t >> (logm - 1), j = t & (half - 1);
            const int g = j >> lh, kk = j & (h - 1);
            const int i = (g << (lh + 1)) + kk;
            double2* p = x + c * estride;
            const double2 a = p[i * cstride], b = p[(i + h) * cstride];
            p[i * cstride] = cadd(a, b);
            p[(i + h) * cstride] = cmul(csub(a, b), tw[kk * st]);
        }
        __syncthreads();
    }
}

__device__ __forceinline__ int brev(int v, int bits) { return (int)(__brev((unsigned)v) >> (32 - bits)); }

__device__ void load_twiddles(double2* tw, int logm, double sign) {
    const int m = 1 << logm;
    for (int j = threadIdx.x; j < m / 2; j += blockDim.x) tw[j] = root(j, m, sign);
    __syncthreads();
}

// forward column pass: tile of kColTile columns n2 (all N1 rows) of the tapered,
// zero-padded record; DFT over n1; x w^(n2 k1) (sign -1); spectrum in place layout
__global__ void k_fft_cols_fwd(const double2* __restrict__ tx, int64_t n_tx, int guard,
                               int l1, int l2, double2* __restrict__ spec) {
    extern __shared__ double2 sm[];
    const int N1 = 1 << l1, N2 = 1 << l2;
    double2* x = sm;                      // [N1][kColTile]
    double2* tw = sm + N1 * kColTile;     // [N1 / 2]
    load_twiddles(tw, l1, -1.0);
    const int c0 = blockIdx.x * kColTile;
    for (int e = threadIdx.x; e < N1 * kColTile; e += blockDim.x) {
        const int r = e / kColTile, c = e % kColTile;
        const int64_t n = (int64_t)r * N2 + c0 + c;
        double2 v = make_double2(0.0, 0.0);
        if (n < n_tx) {
            v = tx[n];
            // Hann taper of the guard samples at both ends (scene.hpp:169-174)
            const int64_t i = n < guard ? n : (n >= n_tx - guard ? n_tx - 1 - n : -1);
            if (i >= 0) {
                const double w = __dmul_rn(
                    0.5, __dsub_rn(1.0, cos(__ddiv_rn(__dmul_rn(kPi, __dadd_rn((double)i, 0.5)),
                                                       (double)guard))));
                v = cscale(w, v);  // complex *= double
            }
        }
        x[e] = v;
    }
    __syncthreads();
    smem_fft(x, l1, kColTile, kColTile, 1, tw);
    const int64_t N = (int64_t)N1 << l2;
    for (int e = threadIdx.x; e < N1 * kColTile; e += blockDim.x) {
        const int k1 = e / kColTile, c = e % kColTile;
        const int n2 = c0 + c;
        const double2 v = x[brev(k1, l1) * kColTile + c];
        spec[(int64_t)k1 * N2 + n2] = cmul(v, root((int64_t)n2 * k1, N, -1.0));
    }
}

// forward row pass: row k1, DFT over n2 -> X[k1 + N1 k2] at (k1, k2)
__global__ void k_fft_rows_fwd(int l1, int l2, double2* __restrict__ spec) {
    extern __shared__ double2 sm[];
    const int N2 = 1 << l2;
    double2* x = sm;
    double2* tw = sm + N2;
    load_twiddles(tw, l2, -1.0);
    double2* row = spec + (int64_t)blockIdx.x * N2;
    for (int i = threadIdx.x; i < N2; i += blockDim.x) x[i] = row[i];
    __syncthreads();
    smem_fft(x, l2, 1, 1, 0, tw);
    for (int k2 = threadIdx.x; k2 < N2; k2 += blockDim.x) row[k2] = x[brev(k2, l2)];
}

// per receiver: the linear phase ramp (scene.hpp:177-185), inverse row DFT over
// k2, x w^(-n2 k1); into that receiver's work buffer
__global__ void k_fft_rows_inv(int l1, int l2, const double2* __restrict__ spec, double frac,
                               double2* __restrict__ work) {
    extern __shared__ double2 sm[];
    const int N1 = 1 << l1, N2 = 1 << l2;
    const int64_t N = (int64_t)N1 << l2;
    double2* x = sm;
    double2* tw = sm + N2;
    load_twiddles(tw, l2, 1.0);
    const int k1 = blockIdx.x;
    const double2* row = spec + (int64_t)k1 * N2;
    for (int k2 = threadIdx.x; k2 < N2; k2 += blockDim.x) {
        const int64_t k = k1 + (int64_t)N1 * k2;
        const double nf = __ddiv_rn((double)(k < N / 2 ? k : k - N), (double)N);
        x[k2] = cmul(row[k2], polar1(__dmul_rn(__dmul_rn(2.0 * kPi, nf), frac)));
    }
    __syncthreads();
    smem_fft(x, l2, 1, 1, 0, tw);
    double2* out = work + (int64_t)k1 * N2;
    for (int n2 = threadIdx.x; n2 < N2; n2 += blockDim.x)
        out[n2] = cmul(x[brev(n2, l2)], root((int64_t)n2 * k1, N, 1.0));
}

// inverse column pass: DFT over k1 -> x[N2 n1 + n2] in natural order, / N
// (fft.hpp:70-73), then received[k] = amplitude * delayed[shift + k] * phasor_k
// (scene.hpp:224-231) for the samples inside the receive window
__global__ void k_fft_cols_inv(int l1, int l2, const double2* __restrict__ work, int64_t shift,
                               int64_t n_out, double amplitude, const double2* __restrict__ phasor,
                               double2* __restrict__ recv) {
    extern __shared__ double2 sm[];
    const int N1 = 1 << l1, N2 = 1 << l2;
    const int64_t N = (int64_t)N1 << l2;
    const double scale = __ddiv_rn(1.0, (double)N);
    double2* x = sm;
    double2* tw = sm + N1 * kColTile;
    load_twiddles(tw, l1, 1.0);
    const int c0 = blockIdx.x * kColTile;
    for (int e = threadIdx.x; e < N1 * kColTile; e += blockDim.x) {
        const int r = e / kColTile, c = e % kColTile;
        x[e] = work[(int64_t)r * N2 + c0 + c];
    }
    __syncthreads();
    smem_fft(x, l1, kColTile, kColTile, 1, tw);
    for (int e = threadIdx.x; e < N1 * kColTile; e += blockDim.x) {
        const int n1 = e / kColTile, c = e % kColTile;
        const int64_t n = (int64_t)n1 * N2 + c0 + c;
        const int64_t k = n - shift;
        if (k < 0 || k >= n_out) continue;
        const double2 d = cscale(scale, x[brev(n1, l1) * kColTile + c]);
        recv[k] = cmul(cscale(amplitude, d), phasor[k]);
    }
}

// frac == 0: no advance (scene.hpp:164), straight from the transmit record
__global__ void k_receive_direct(const double2* __restrict__ tx, int64_t shift, int64_t n_out,
                                 double amplitude, const double2* __restrict__ phasor,
                                 double2* __restrict__ recv) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_out;
         k += (int64_t)gridDim.x * blockDim.x)
        recv[k] = cmul(cscale(amplitude, tx[shift + k]), phasor[k]);
}

// phasor_k = rotation^k by the reference's recurrence, one thread per record
__global__ void k_phasors(const double2* __restrict__ rotation, int n_rec, int64_t n_out,
                          double2* __restrict__ phasor) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rec) return;
    const double2 rot = rotation[r];
    double2 p = make_double2(1.0, 0.0);
    double2* out = phasor + (int64_t)r * n_out;
    for (int64_t k = 0; k < n_out; ++k) {
        out[k] = p;
        p = cmul(p, rot);
    }
}

// MT19937-64 (std::mt19937_64) state twist, 312 words, by the CTA: the first 156
// words depend only on old words, the rest on old words and the new first half
constexpr int kMtN = 312, kMtM = 156;
constexpr uint64_t kMtA = 0xB5026F5AA96619E9ull, kMtUpper = 0xFFFFFFFF80000000ull,
                   kMtLower = 0x7FFFFFFFull;

__device__ void mt_twist(uint64_t* x) {
    const int k = threadIdx.x;
    uint64_t nv = 0;
    if (k < kMtM) {
        const uint64_t y = (x[k] & kMtUpper) | (x[k + 1] & kMtLower);
        nv = x[k + kMtM] ^ (y >> 1) ^ ((y & 1) ? kMtA : 0);
    }
    __syncthreads();
    if (k < kMtM) x[k] = nv;
    __syncthreads();
    if (k >= kMtM && k < kMtN) {
        const uint64_t y = (x[k] & kMtUpper) | (x[(k + 1) % kMtN] & kMtLower);
        nv = x[k - kMtM] ^ (y >> 1) ^ ((y & 1) ? kMtA : 0);
    }
    __syncthreads();
    if (k >= kMtM && k < kMtN) x[k] = nv;
    __syncthreads();
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

// one CTA (>= 312 threads) per (snapshot, receiver): capture[k] = ((0 + recv_0[k]) +
// recv_1[k] + ...) + sigma * noise_k (scene.hpp:276-306)
__global__ void k_noise_combine(const uint64_t* __restrict__ seeds, int n_rx, int n_em,
                                const double2* __restrict__ recv, int64_t n, double sigma,
                                int add_noise, double2* __restrict__ caps, int64_t cap_stride) {
    __shared__ uint64_t x[kMtN];
    const int stream = blockIdx.x;  // s * n_rx + r
    const int s = stream / n_rx, r = stream % n_rx;
    double2* cap = caps + (int64_t)stream * cap_stride;
    if (add_noise && threadIdx.x == 0) {  // std::mersenne_twister_engine::seed
        uint64_t v = seeds[stream];
        x[0] = v;
        for (int i = 1; i < kMtN; ++i) {
            v = 6364136223846793005ull * (v ^ (v >> 62)) + (uint64_t)i;
            x[i] = v;
        }
    }
    __syncthreads();
    const int per = kMtN / 2;  // samples per twist (two draws each)
    for (int64_t base = 0; base < n; base += per) {
        if (add_noise) mt_twist(x);
        const int64_t k = base + threadIdx.x;
        if (threadIdx.x < per && k < n) {
            double2 acc = make_double2(0.0, 0.0);
            for (int e = 0; e < n_em; ++e)
                acc = cadd(acc, recv[(((int64_t)s * n_em + e) * n_rx + r) * n + k]);
            if (add_noise) {
                const uint64_t d1 = mt_temper(x[2 * threadIdx.x]);
                const uint64_t d2 = mt_temper(x[2 * threadIdx.x + 1]);
                const double u1 = __dmul_rn(__dadd_rn((double)(d1 >> 11), 1.0), 0x1.0p-53);
                const double u2 = __dmul_rn(__dadd_rn((double)(d2 >> 11), 1.0), 0x1.0p-53);
                const double rr = sqrt(-log(u1));
                const double2 p = polar1(__dmul_rn(2.0 * kPi, u2));
                const double2 g = make_double2(__dmul_rn(rr, p.x), __dmul_rn(rr, p.y));
                acc = cadd(acc, cscale(sigma, g));
            }
            cap[k] = acc;
        }
        __syncthreads();  // the next twist overwrites x
    }
}

inline int blocks_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    return (int)(b < 148 * 8 ? (b > 0 ? b : 1) : 148 * 8);
}

}  // namespace

void launch_waveform(const WaveParams& w, double start, double ts, int64_t n, const int8_t* chips,
                     double2* out, cudaStream_t st) {
    k_waveform<<<blocks_for(n), 256, 0, st>>>(w, start, ts, n, chips, out);
}

int fft_log2_max() { return 22; }

void launch_fractional_fwd(const double2* tx, int64_t n_tx, int guard, int l, double2* spec,
                           cudaStream_t st) {
    const int l1 = l / 2, l2 = l - l1;
    const size_t col_smem = ((size_t)(kColTile << l1) + (1 << (l1 - 1))) * sizeof(double2);
    const size_t row_smem = ((size_t)(1 << l2) + (1 << (l2 - 1))) * sizeof(double2);
    static size_t a0[64] = {}, a1[64] = {}, a2[64] = {}, a3[64] = {};
    ensure_smem(k_fft_cols_fwd, 200 << 10, a0);
    ensure_smem(k_fft_rows_fwd, 200 << 10, a1);
    ensure_smem(k_fft_rows_inv, 200 << 10, a2);
    ensure_smem(k_fft_cols_inv, 200 << 10, a3);
    k_fft_cols_fwd<<<(1 << l2) / kColTile, kFftThreads, col_smem, st>>>(tx, n_tx, guard, l1, l2,
                                                                          spec);
    k_fft_rows_fwd<<<1 << l1, kFftThreads, row_smem, st>>>(l1, l2, spec);
}

void launch_fractional_inv(const double2* spec, int l, double frac, int64_t shift, int64_t n_out,
                           double amplitude, const double2* phasor, double2* work, double2* recv,
                           cudaStream_t st) {
    const int l1 = l / 2, l2 = l - l1;
    const size_t col_smem = ((size_t)(kColTile << l1) + (1 << (l1 - 1))) * sizeof(double2);
    const size_t row_smem = ((size_t)(1 << l2) + (1 << (l2 - 1))) * sizeof(double2);
    k_fft_rows_inv<<<1 << l1, kFftThreads, row_smem, st>>>(l1, l2, spec, frac, work);
    k_fft_cols_inv<<<(1 << l2) / kColTile, kFftThreads, col_smem, st>>>(l1, l2, work, shift, n_out,
                                                                          amplitude, phasor, recv);
}

void launch_receive_direct(const double2* tx, int64_t shift, int64_t n_out, double amplitude,
                           const double2* phasor, double2* recv, cudaStream_t st) {
    k_receive_direct<<<blocks_for(n_out), 256, 0, st>>>(tx, shift, n_out, amplitude, phasor, recv);
}

void launch_phasors(const double2* rotation, int n_rec, int64_t n_out, double2* phasor,
                    cudaStream_t st) {
    k_phasors<<<(n_rec + 63) / 64, 64, 0, st>>>(rotation, n_rec, n_out, phasor);
}

void launch_noise_combine(const uint64_t* seeds, int n_snap, int n_rx, int n_em,
                          const double2* recv, int64_t n, double sigma, int add_noise,
                          double2* caps, int64_t cap_stride, cudaStream_t st) {
    k_noise_combine<<<n_snap * n_rx, 320, 0, st>>>(seeds, n_rx, n_em, recv, n, sigma, add_noise,
                                                   caps, cap_stride);
}

}  // namespace dg
