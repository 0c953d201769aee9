// sm_100a kernels of the B200 direct-geolocation engine.
//
// Reference (read-only, /root/reference/proj/include/digeo): the hot path is
// correlate.hpp:44-71 (Eq. 11) driven by geolocate.hpp:41-146, fed by
// geometry.hpp:51-83 and geodesy.hpp:82-92,182-207.
//
// Data layout in HBM:
//   grid      SoA double x[P], y[P], z[P]           (lat-major flat index)
//   captures  float2  [S][R][N] (FP32 hot path) + double2 [S][R][N] (FP64 refine)
//   per (snapshot, pair): d[P] int32, fdoa[P] f64, d-sorted candidate ids,
//   warp tasks, raw surface double [S*pairs][P], refine bitmap 1 bit/element.
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cstring>
#include <float.h>
#include <limits.h>
#include <math.h>
#include <stdint.h>

#include "dg_internal.cuh"

namespace dg {

namespace {

constexpr double kC = 299792458.0;      // geometry.hpp:32
constexpr double kTwoPi = 6.283185307179586;  // 2.0 * std::numbers::pi (exact doubling)
constexpr int kNoOverlap = INT_MIN;

inline int blocks_for(int64_t n, int threads, int64_t cap = 148LL * 64) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return (int)b;
}

// ---------------------------------------------------------------------------
// predict_geometry (geometry.hpp:51-64) in the reference's exact IEEE order:
// r = p_rx - c; rho = sqrt((x*x + y*y) + z*z); delay = rho / c;
// u = (1/rho) * r; doppler = -dot(u, v) / wl. No FMA contraction.
__device__ __forceinline__ bool geometry_exact(double cx, double cy, double cz, const dg_state& rx,
                                               double wl, double* delay, double* dop) {
    const double rx_ = __dsub_rn(rx.position.x, cx);
    const double ry = __dsub_rn(rx.position.y, cy);
    const double rz = __dsub_rn(rx.position.z, cz);
    const double rho =
        __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(rx_, rx_), __dmul_rn(ry, ry)), __dmul_rn(rz, rz)));
    *delay = __ddiv_rn(rho, kC);
    const double inv = __ddiv_rn(1.0, rho);
    const double ux = __dmul_rn(inv, rx_), uy = __dmul_rn(inv, ry), uz = __dmul_rn(inv, rz);
    const double dot = __dadd_rn(__dadd_rn(__dmul_rn(ux, rx.velocity.x), __dmul_rn(uy, rx.velocity.y)),
                                 __dmul_rn(uz, rx.velocity.z));
    *dop = __ddiv_rn(-dot, wl);
    return rho > 0.0;
}

// The same delay and Doppler with FMA contraction and a Newton-refined reciprocal
// square root instead of IEEE division / square root (a few ulp from the exact
// values): the candidate evaluation only needs FP32-class FDOA; the TDOA of a pair
// is taken from these only away from a rounding boundary (pair_tdoa_fast), and the
// FP64 refinement and the exact re-rank recompute both offsets with geometry_exact.
__device__ __forceinline__ bool geometry_fast(double cx, double cy, double cz, const dg_state& rx,
                                              double inv_wl, double* delay, double* dop) {
    const double rx_ = rx.position.x - cx, ry = rx.position.y - cy, rz = rx.position.z - cz;
    const double r2 = fma(rx_, rx_, fma(ry, ry, rz * rz));
    double inv = rsqrt(r2);
    inv = inv * fma(-0.5 * r2 * inv, inv, 1.5);  // one Newton step past rsqrt's ~1 ulp
    const double rho = r2 * inv;
    *delay = rho * (1.0 / kC);
    const double dot = fma(rx_, rx.velocity.x, fma(ry, rx.velocity.y, rz * rx.velocity.z));
    *dop = -(dot * inv) * inv_wl;
    return r2 > 0.0;
}
// llround((dj - di) fs) from the fast delays when the product is farther than
// 1e-6 + 1e-12 |t| samples from a half-integer (the fast-exact difference is below
// 1e-9 samples at any sample rate these runs use); otherwise -1 (recompute exactly)
__device__ __forceinline__ bool pair_tdoa_fast(double di, double dj, double fs, long long* tdoa) {
    const double t = (dj - di) * fs;
    const double a = fabs(t), f = a - floor(a);
    if (fabs(f - 0.5) <= 1e-6 + 1e-12 * a) return false;
    *tdoa = llround(t);
    return true;
}

// predict_pair_offsets (geometry.hpp:73-83): llround ties away from zero.
__device__ __forceinline__ bool offsets_exact(double cx, double cy, double cz, const PairGeom& g,
                                              double fs, double wl, long long* tdoa, double* fdoa) {
    double di, fi, dj, fj;
    const bool ok_i = geometry_exact(cx, cy, cz, g.rx_i, wl, &di, &fi);
    const bool ok_j = geometry_exact(cx, cy, cz, g.rx_j, wl, &dj, &fj);
    *tdoa = llround(__dmul_rn(__dsub_rn(dj, di), fs));
    *fdoa = __dsub_rn(fj, fi);
    return ok_i && ok_j;
}

// correlate_kernel (correlate.hpp:44-71) in the reference's exact order: one
// FP64 phasor recurrence, ascending k, double accumulators. Used only for the
// few elements whose FP32 value cannot meet the relative tolerance and for the
// near-peak re-rank; cos/sin are CUDA's (<= 1 ulp apart from glibc's).
// tg (nullable): {cos(step), sin(step), cos(phase0), sin(phase0)} from the host's
// libm (the reference's own std::cos / std::sin, exact_peak), so the chain is
// bit-identical to the reference's; without it CUDA's sincos (<= 1 ulp off).
__device__ __forceinline__ void chain_trig(long long kb, double fdoa, double fs,
                                           const double* tg, double* rot_re, double* rot_im,
                                           double* ph_re, double* ph_im) {
    if (tg) {
        *rot_re = tg[0];
        *rot_im = tg[1];
        *ph_re = tg[2];
        *ph_im = tg[3];
        return;
    }
    const double step = __ddiv_rn(__dmul_rn(kTwoPi, fdoa), fs);
    sincos(step, rot_im, rot_re);
    sincos(__dmul_rn(step, (double)kb), ph_im, ph_re);
}

__device__ double correlate_exact(const double2* __restrict__ y1, const double2* __restrict__ y2,
                                  int N, long long d, double fdoa, double fs,
                                  const double* tg = nullptr) {
    const long long kb = d < 0 ? -d : 0;
    const long long ke = (N - d) < N ? (N - d) : N;
    if (kb >= ke) return 0.0;
    double rot_im, rot_re, ph_im, ph_re;
    chain_trig(kb, fdoa, fs, tg, &rot_re, &rot_im, &ph_re, &ph_im);
    double acc_re = 0.0, acc_im = 0.0;
    const double2* b = y2 + d;
    // one reference iteration (correlate.hpp:59-69), operation order unchanged
    auto step_k = [&](const double2 a, const double2 bb) {
        const double b_re = bb.x, b_im = -bb.y;
        const double p_re = __dsub_rn(__dmul_rn(a.x, b_re), __dmul_rn(a.y, b_im));
        const double p_im = __dadd_rn(__dmul_rn(a.x, b_im), __dmul_rn(a.y, b_re));
        acc_re = __dadd_rn(acc_re, __dsub_rn(__dmul_rn(p_re, ph_re), __dmul_rn(p_im, ph_im)));
        acc_im = __dadd_rn(acc_im, __dadd_rn(__dmul_rn(p_re, ph_im), __dmul_rn(p_im, ph_re)));
        const double nr = __dsub_rn(__dmul_rn(ph_re, rot_re), __dmul_rn(ph_im, rot_im));
        ph_im = __dadd_rn(__dmul_rn(ph_re, rot_im), __dmul_rn(ph_im, rot_re));
        ph_re = nr;
    };
    // the loads of the next 8 samples are issued before the current 8 are
    // consumed, so the sequential FP64 chain never waits on memory
    constexpr int U = 8;
    long long k = kb;
    if (ke - kb >= 2 * U) {
        double2 na[U], nb[U];
#pragma unroll
        for (int i = 0; i < U; ++i) {
            na[i] = __ldg(y1 + k + i);
            nb[i] = __ldg(b + k + i);
        }
        for (; k + 2 * U <= ke; k += U) {
            // pull the lines 32 groups ahead into L1 so the register prefetch
            // below never waits on L2/HBM (one 128-B line per U samples)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(y1 + k + 32 * U));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(b + k + 32 * U));
            double2 ca[U], cb[U];
#pragma unroll
            for (int i = 0; i < U; ++i) {
                ca[i] = na[i];
                cb[i] = nb[i];
                na[i] = __ldg(y1 + k + U + i);
                nb[i] = __ldg(b + k + U + i);
            }
#pragma unroll
            for (int i = 0; i < U; ++i) step_k(ca[i], cb[i]);
        }
#pragma unroll
        for (int i = 0; i < U; ++i) step_k(na[i], nb[i]);
        k += U;
    }
    for (; k < ke; ++k) step_k(y1[k], b[k]);
    return __dsqrt_rn(__dadd_rn(__dmul_rn(acc_re, acc_re), __dmul_rn(acc_im, acc_im)));
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---------------------------------------------------------------------------
// K1: lattice ECEF (geodesy.hpp:82-92,182-207). The host supplies per-row
// A_i = (N_i + alt) * cos(lat_i), Z_i = (N_i (1 - e2) + alt) * sin(lat_i) and
// per-column cos/sin(lon_j) from libm, so x = A_i * cos(lon_j) etc. reproduce
// lla_to_ecef's doubles exactly (same operands, same single rounding).
__global__ void k_grid_ecef(const double* __restrict__ ra, const double* __restrict__ rz,
                            const double* __restrict__ cc, const double* __restrict__ cs,
                            int64_t n_lat, int64_t n_lon, double* __restrict__ x,
                            double* __restrict__ y, double* __restrict__ z) {
    const int64_t P = n_lat * n_lon;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = p / n_lon, j = p - i * n_lon;
        const double a = ra[i];
        x[p] = __dmul_rn(a, cc[j]);
        y[p] = __dmul_rn(a, cs[j]);
        z[p] = rz[i];
    }
}

// ---------------------------------------------------------------------------
// K2: per-point offsets (bit-exact) + TDOA histogram for the warp bucketing.
// Candidates whose shift leaves no overlap get S = 0 here (correlate.hpp:49).
// Per-thread running ranges of the overlapping candidates (StepRange).
struct RangeAcc {
    unsigned long long fmin = ~0ull, fmax = 0ull;
    int dmin = INT_MAX, dmax = INT_MIN;
    __device__ void flush(StepRange* r) {
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            fmin = min(fmin, __shfl_xor_sync(0xffffffffu, fmin, o));
            fmax = max(fmax, __shfl_xor_sync(0xffffffffu, fmax, o));
            dmin = min(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
            dmax = max(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        }
        if ((threadIdx.x & 31) == 0 && dmin <= dmax) {
            atomicMin(&r->fmin, fmin);
            atomicMax(&r->fmax, fmax);
            atomicMin(&r->dmin, dmin);
            atomicMax(&r->dmax, dmax);
        }
    }
};

// rank_out[p]: the histogram atomic's old value, this candidate's rank in its
// TDOA bin, so k_scatter places it without atomics
__device__ __forceinline__ void emit_point(int64_t p, long long tdoa, double fdoa, int N,
                                           int* d_out, int* rank_out, double* fdoa_out, int* hist,
                                           double* s_out, unsigned long long& ovl, RangeAcc& ra) {
    if (tdoa >= N || tdoa <= -N) {  // empty overlap (also catches llround overflow)
        d_out[p] = kNoOverlap;
        s_out[p] = 0.0;
    } else {
        const int d = (int)tdoa;
        d_out[p] = d;
        fdoa_out[p] = fdoa;
        rank_out[p] = atomicAdd(&hist[d + N - 1], 1);
        ovl += (unsigned long long)(N - (d < 0 ? -d : d));
        const unsigned long long k = f64_key(fdoa);
        ra.fmin = min(ra.fmin, k);
        ra.fmax = max(ra.fmax, k);
        ra.dmin = min(ra.dmin, d);
        ra.dmax = max(ra.dmax, d);
    }
}

__global__ void k_geometry_hist(const double* __restrict__ x, const double* __restrict__ y,
                                const double* __restrict__ z, int64_t P,
                                const PairGeom* __restrict__ pg, double fs, double wl, int N,
                                int* __restrict__ d_out, int* __restrict__ rank_out,
                                double* __restrict__ fdoa_out,
                                int* __restrict__ hist, double* __restrict__ s_out,
                                unsigned long long* __restrict__ overlap, int* __restrict__ err,
                                StepRange* __restrict__ range) {
    const PairGeom g = *pg;
    unsigned long long ovl = 0;
    RangeAcc ra;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        long long tdoa;
        double fdoa;
        if (!offsets_exact(x[p], y[p], z[p], g, fs, wl, &tdoa, &fdoa)) atomicExch(err, 1);
        emit_point(p, tdoa, fdoa, N, d_out, rank_out, fdoa_out, hist, s_out, ovl, ra);
    }
    ovl = warp_sum_u64(ovl);
    if ((threadIdx.x & 31) == 0 && ovl) atomicAdd(overlap, ovl);
    ra.flush(range);
}

// Phase A of a window of units in one pass: each thread loads its candidate
// once and predicts the offsets of every unit of the window, writing d[u][P],
// rank[u][P], fdoa[u][P], the per-unit TDOA histograms and S = 0 for candidates
// without overlap. The units come in groups that share receivers (the pairs of
// one snapshot: correlate_snapshot_all_pairs, geolocate.hpp:79-94), and every
// receiver's delay and Doppler (predict_geometry, geometry.hpp:51-64) is
// computed once per candidate and group, then differenced for each pair — the
// same operations as predict_pair_offsets on each pair, so bit-identical, with
// R instead of R(R-1) receiver evaluations per snapshot. The ranges are not
// reduced here: the bins come from the histograms (k_hist_range), B / R / the
// centre frequency from the FP32 lattice ranges (k_range_fp32).
constexpr int kGeoUnitsMax = 64;  // units per launch (shared-memory tables)
constexpr int kGeoRxMax = 8;      // receivers per group

// KR: receivers per group the launch needs (2 for two-receiver runs: no
// register tables beyond the pair)
template <int KR>
__global__ void __launch_bounds__(256)
k_geometry_units(const double* __restrict__ x, const double* __restrict__ y,
                 const double* __restrict__ z, int64_t P, const dg_state* __restrict__ rx,
                 int nrx, const GeoGroup* __restrict__ groups, int ng,
                 const int2* __restrict__ upair, int n, double fs, double wl, int N,
                 int* __restrict__ d_out, int* __restrict__ rank_out,
                 double* __restrict__ fdoa_out, int* __restrict__ hist, int nbins,
                 double* __restrict__ s_out, unsigned long long* __restrict__ overlap,
                 int* __restrict__ err) {
    __shared__ dg_state srx[2 * kGeoUnitsMax];
    __shared__ GeoGroup sgr[kGeoUnitsMax];
    __shared__ int2 sup[kGeoUnitsMax];
    for (int i = threadIdx.x; i < nrx * (int)(sizeof(dg_state) / 8); i += blockDim.x)
        reinterpret_cast<double*>(srx)[i] = reinterpret_cast<const double*>(rx)[i];
    for (int i = threadIdx.x; i < ng; i += blockDim.x) sgr[i] = groups[i];
    for (int i = threadIdx.x; i < n; i += blockDim.x) sup[i] = upair[i];
    __syncthreads();
    const double inv_wl = 1.0 / wl;
    unsigned long long ovl = 0;
    RangeAcc ra;  // not flushed: ranges come from k_hist_range / k_range_fp32
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        const double cx = x[p], cy = y[p], cz = z[p];
        for (int g = 0; g < ng; ++g) {
            const GeoGroup gr = sgr[g];
            double del[KR], dop[KR];
            bool ok[KR];
#pragma unroll
            for (int r = 0; r < KR; ++r)
                if (r < gr.nrx)
                    ok[r] = geometry_fast(cx, cy, cz, srx[gr.rx0 + r], inv_wl, &del[r], &dop[r]);
            for (int u = gr.u0; u < gr.u0 + gr.nu; ++u) {
                const int2 ij = sup[u];
                double di = 0.0, fi = 0.0, dj = 0.0, fj = 0.0;
                bool oki = true, okj = true;
#pragma unroll
                for (int r = 0; r < KR; ++r) {
                    if (r == ij.x) {
                        di = del[r];
                        fi = dop[r];
                        oki = ok[r];
                    }
                    if (r == ij.y) {
                        dj = del[r];
                        fj = dop[r];
                        okj = ok[r];
                    }
                }
                // predict_pair_offsets (geometry.hpp:73-83): llround ties away from zero;
                // exact delays where the fast ones sit near a rounding boundary
                long long tdoa;
                if (!pair_tdoa_fast(di, dj, fs, &tdoa)) {
                    double ei, ej, xi, xj;
                    geometry_exact(cx, cy, cz, srx[gr.rx0 + ij.x], wl, &ei, &xi);
                    geometry_exact(cx, cy, cz, srx[gr.rx0 + ij.y], wl, &ej, &xj);
                    tdoa = llround(__dmul_rn(__dsub_rn(ej, ei), fs));
                }
                const double fdoa = fj - fi;
                if (!(oki && okj)) atomicExch(err, 1);
                emit_point(p, tdoa, fdoa, N, d_out + (int64_t)u * P, rank_out + (int64_t)u * P,
                           fdoa_out + (int64_t)u * P, hist + (int64_t)u * nbins,
                           s_out + (int64_t)u * P, ovl, ra);
            }
        }
    }
    ovl = warp_sum_u64(ovl);
    if ((threadIdx.x & 31) == 0 && ovl) atomicAdd(overlap, ovl);
}

__global__ void k_predict_offsets(const double* __restrict__ x, const double* __restrict__ y,
                                  const double* __restrict__ z, int64_t P,
                                  const PairGeom* __restrict__ pg, double fs, double wl,
                                  dg_pair_offsets* __restrict__ out, int* __restrict__ err) {
    const PairGeom g = *pg;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        long long tdoa;
        double fdoa;
        if (!offsets_exact(x[p], y[p], z[p], g, fs, wl, &tdoa, &fdoa)) atomicExch(err, 1);
        dg_pair_offsets o;
        o.tdoa_samples = tdoa;
        o.fdoa_hz = fdoa;
        out[p] = o;
    }
}

__global__ void k_offsets_hist(const dg_pair_offsets* __restrict__ off, int64_t P, int N,
                               int* __restrict__ d_out, int* __restrict__ rank_out,
                               double* __restrict__ fdoa_out,
                               int* __restrict__ hist, double* __restrict__ s_out,
                               unsigned long long* __restrict__ overlap,
                               StepRange* __restrict__ range) {
    unsigned long long ovl = 0;
    RangeAcc ra;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        const dg_pair_offsets o = off[p];
        emit_point(p, o.tdoa_samples, o.fdoa_hz, N, d_out, rank_out, fdoa_out, hist, s_out, ovl,
                   ra);
    }
    ovl = warp_sum_u64(ovl);
    if ((threadIdx.x & 31) == 0 && ovl) atomicAdd(overlap, ovl);
    ra.flush(range);
}

// ---------------------------------------------------------------------------
// Planning ranges (not bit-exact; only used to choose the correlator's block
// length, moment count and centre frequency, which must not depend on how the
// lattice is partitioned): positions relative to the lattice centre in FP32.
__global__ void k_lattice_rel(const double* __restrict__ x, const double* __restrict__ y,
                              const double* __restrict__ z, int64_t P, double cx, double cy,
                              double cz, float4* __restrict__ out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x)
        out[p] = make_float4((float)(x[p] - cx), (float)(y[p] - cy), (float)(z[p] - cz), 0.f);
}

constexpr int kRangeThreads = 256;

__global__ void __launch_bounds__(kRangeThreads)
k_range_fp32(const float4* __restrict__ rel, int64_t P, const RxPairF32* __restrict__ rx,
             int n_steps, float fs_over_c, float inv_wl, StepRange* __restrict__ out) {
    __shared__ float red[4][kRangeThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int s = 0; s < n_steps; ++s) {
        const RxPairF32 g = rx[s];
        float fmn = INFINITY, fmx = -INFINITY, dmn = INFINITY, dmx = -INFINITY;
        for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
             p += (int64_t)gridDim.x * blockDim.x) {
            const float4 c = rel[p];
            const float ax = g.pi[0] - c.x, ay = g.pi[1] - c.y, az = g.pi[2] - c.z;
            const float bx = g.pj[0] - c.x, by = g.pj[1] - c.y, bz = g.pj[2] - c.z;
            // MUFU reciprocal square roots (~2 ulp): the planning margin is 1e-5
            // relative (fp32_fdoa_margin), the TDOA margin 2 samples
            const float si = ax * ax + ay * ay + az * az, sj = bx * bx + by * by + bz * bz;
            const float qi = rsqrtf(si), qj = rsqrtf(sj);
            const float ri = si * qi, rj = sj * qj;
            const float di = -(ax * g.vi[0] + ay * g.vi[1] + az * g.vi[2]) * qi;
            const float dj = -(bx * g.vj[0] + by * g.vj[1] + bz * g.vj[2]) * qj;
            const float f = (dj - di) * inv_wl;
            const float t = (rj - ri) * fs_over_c;
            fmn = fminf(fmn, f);
            fmx = fmaxf(fmx, f);
            dmn = fminf(dmn, t);
            dmx = fmaxf(dmx, t);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            fmn = fminf(fmn, __shfl_xor_sync(0xffffffffu, fmn, o));
            fmx = fmaxf(fmx, __shfl_xor_sync(0xffffffffu, fmx, o));
            dmn = fminf(dmn, __shfl_xor_sync(0xffffffffu, dmn, o));
            dmx = fmaxf(dmx, __shfl_xor_sync(0xffffffffu, dmx, o));
        }
        if (lane == 0) {
            red[0][warp] = fmn;
            red[1][warp] = fmx;
            red[2][warp] = dmn;
            red[3][warp] = dmx;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < kRangeThreads / 32; ++w) {
                fmn = fminf(fmn, red[0][w]);
                fmx = fmaxf(fmx, red[1][w]);
                dmn = fminf(dmn, red[2][w]);
                dmx = fmaxf(dmx, red[3][w]);
            }
            if (fmn <= fmx) {
                atomicMin(&out[s].fmin, f64_key((double)fmn));
                atomicMax(&out[s].fmax, f64_key((double)fmx));
                atomicMin(&out[s].dmin, (int)floorf(dmn) - 2);
                atomicMax(&out[s].dmax, (int)ceilf(dmx) + 2);
            }
        }
        __syncthreads();
    }
}

// Exact TDOA range of each step of a window: the first and last non-empty
// bin of its histogram. The buckets are planned over these bins, so every
// candidate lands in a planned bin whatever the error of the FP32 planning pass
// (which now only sets B, R and the centre frequency). Grid (chunks, steps):
// each CTA scans kHistRangeChunk bins and folds its extremes into the step's
// range with atomics (k_range_init sets the empty range first).
constexpr int kHistRangeThreads = 512;
constexpr int kHistRangeChunk = 16 * kHistRangeThreads;

__global__ void k_range_init(StepRange* __restrict__ out, int n_steps) {
    for (int s = threadIdx.x; s < n_steps; s += blockDim.x) {
        StepRange r;
        r.fmin = ~0ull;
        r.fmax = 0ull;
        r.dmin = INT_MAX;
        r.dmax = INT_MIN;
        out[s] = r;
    }
}

__global__ void __launch_bounds__(kHistRangeThreads)
k_hist_range(const int* __restrict__ hist, int nbins, int N, StepRange* __restrict__ out) {
    __shared__ int red[2][kHistRangeThreads / 32];
    const int* h = hist + (int64_t)blockIdx.y * nbins;
    const int b0 = blockIdx.x * kHistRangeChunk;
    int lo = INT_MAX, hi = INT_MIN;
#pragma unroll
    for (int j = 0; j < kHistRangeChunk / kHistRangeThreads; ++j) {
        const int b = b0 + j * kHistRangeThreads + threadIdx.x;
        if (b < nbins && h[b]) {
            lo = min(lo, b);
            hi = max(hi, b);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        red[0][warp] = lo;
        red[1][warp] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kHistRangeThreads / 32; ++w) {
            lo = min(lo, red[0][w]);
            hi = max(hi, red[1][w]);
        }
        if (lo <= hi) {
            atomicMin(&out[blockIdx.y].dmin, lo - (N - 1));
            atomicMax(&out[blockIdx.y].dmax, hi - (N - 1));
        }
    }
}

// Exclusive prefix sums of |y|^2 per capture, FP64 (one CTA per capture):
// E[c][k] = sum_{i<k} |y_c[i]|^2. A bucket's ||z||_2^2 estimate is then
// sum_b E1_b E2_b / len_b over its blocks (exact for constant-envelope
// signals), the moment path's refinement floor (k_evaluate*).
constexpr int kEnergyThreads = 1024;

__global__ void __launch_bounds__(kEnergyThreads)
k_energy_prefix(const double2* __restrict__ y, int64_t stride, int64_t N, double* __restrict__ out) {
    __shared__ double sh[kEnergyThreads];
    const double2* yc = y + (int64_t)blockIdx.x * stride;
    double* o = out + (int64_t)blockIdx.x * (N + 1);
    const int t = threadIdx.x;
    const int64_t per = (N + kEnergyThreads - 1) / kEnergyThreads;
    const int64_t k0 = min(N, t * per), k1 = min(N, k0 + per);
    double s = 0.0;
    for (int64_t k = k0; k < k1; ++k) s = fma(yc[k].x, yc[k].x, fma(yc[k].y, yc[k].y, s));
    sh[t] = s;
    __syncthreads();
    for (int off = 1; off < kEnergyThreads; off <<= 1) {  // inclusive Hillis-Steele scan
        const double v = t >= off ? sh[t - off] : 0.0;
        __syncthreads();
        sh[t] += v;
        __syncthreads();
    }
    double run = sh[t] - s;  // exclusive prefix of this thread's range
    for (int64_t k = k0; k < k1; ++k) {
        o[k] = run;
        run = fma(yc[k].x, yc[k].x, fma(yc[k].y, yc[k].y, run));
    }
    if (t == kEnergyThreads - 1) o[N] = sh[t];
}

// ---------------------------------------------------------------------------
// Bucketing over the step's TDOA range only (bins [bin0, bin0 + nbins)):
// exclusive scans of per-d counts, per-d warp-task counts and non-empty bins,
// then scatter candidate ids by d, cut each d-bucket into warp tasks and emit
// one Bucket per non-empty bin.
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 8;

__global__ void __launch_bounds__(kScanThreads)
k_scan(const int* __restrict__ hist, int nbins, int ts, int* __restrict__ off,
       int* __restrict__ toff, int* __restrict__ boff, int* __restrict__ cursor,
       int* __restrict__ n_tasks, int* __restrict__ n_buckets) {
    __shared__ int ws[3][32];
    __shared__ int carry[3];
    if (threadIdx.x < 3) carry[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int base = 0; base < nbins; base += kScanThreads * kScanItems) {
        int v[kScanItems];
        int tot[3] = {0, 0, 0};
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) {
            const int idx = base + threadIdx.x * kScanItems + i;
            v[i] = idx < nbins ? hist[idx] : 0;
            tot[0] += v[i];
            tot[1] += (v[i] + ts - 1) / ts;
            tot[2] += v[i] ? 1 : 0;
        }
        int inc[3] = {tot[0], tot[1], tot[2]};  // inclusive warp scans
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int x = __shfl_up_sync(0xffffffffu, inc[c], o);
                if (lane >= o) inc[c] += x;
            }
        }
        if (lane == 31)
#pragma unroll
            for (int c = 0; c < 3; ++c) ws[c][warp] = inc[c];
        __syncthreads();
        if (warp == 0) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                int a = ws[c][lane];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int x = __shfl_up_sync(0xffffffffu, a, o);
                    if (lane >= o) a += x;
                }
                ws[c][lane] = a;
            }
        }
        __syncthreads();
        int e[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) e[c] = carry[c] + (warp ? ws[c][warp - 1] : 0) + inc[c] - tot[c];
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) {
            const int idx = base + threadIdx.x * kScanItems + i;
            if (idx < nbins) {
                off[idx] = e[0];
                cursor[idx] = e[0];
                toff[idx] = e[1];
                boff[idx] = e[2];
            }
            e[0] += v[i];
            e[1] += (v[i] + ts - 1) / ts;
            e[2] += v[i] ? 1 : 0;
        }
        __syncthreads();
        if (threadIdx.x < 3) carry[threadIdx.x] += ws[threadIdx.x][31];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *n_tasks = carry[1];
        *n_buckets = carry[2];
    }
}

// sfdoa (nullable): the candidates' FDOA in the same bucket order, so the
// candidate evaluators read contiguous values instead of gathering fdoa[p].
// Each candidate goes to its bin's start plus its rank in the bin (taken by
// the geometry pass's histogram atomic): no atomics here, a streaming pass.
// Candidates whose bin lies outside the planned bins [bin0, bin0 + nbins) are
// skipped (another part of a split step owns them; their offsets are unset).
__global__ void k_scatter(const int* __restrict__ d, const int* __restrict__ rank, int64_t P, int N,
                          int bin0, int nbins, const int* __restrict__ off,
                          int* __restrict__ sorted, const double* __restrict__ fdoa,
                          double* __restrict__ sfdoa) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int dd = d[p];
        if (dd == kNoOverlap || (unsigned)(dd + N - 1 - bin0) >= (unsigned)nbins) continue;
        const int pos = off[dd + N - 1] + rank[p];
        sorted[pos] = (int)p;
        if (sfdoa) sfdoa[pos] = fdoa[p];
    }
}

// hist/off/toff/boff are offset to bin0 (d = bin0 + b - (N - 1))
__global__ void k_build_tasks(int* __restrict__ hist, int nbins, int bin0, int N, int ts,
                              const int* __restrict__ off, const int* __restrict__ toff,
                              const int* __restrict__ boff, Task* __restrict__ tasks,
                              Bucket* __restrict__ buckets, int* __restrict__ ubin, int B) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nbins; b += gridDim.x * blockDim.x) {
        const int cnt = hist[b];
        if (B > 0) ubin[b] = cnt ? boff[b] : -1;
        if (!cnt) continue;
        hist[b] = 0;  // ready for the next (snapshot, pair)
        const int d = bin0 + b - (N - 1);
        const int t0 = toff[b], s0 = off[b], u = boff[b];
        if (B > 0) {
            Bucket bk;
            bk.d = d;
            bk.start = s0;
            bk.count = cnt;
            // blocks aligned to absolute sample index (k_moments): those meeting
            // the overlap [kb, ke)
            const int kb = d < 0 ? -d : 0, ke = d > 0 ? N - d : N;
            bk.nb = (ke - 1) / B - kb / B + 1;
            buckets[u] = bk;
        }
        for (int t = 0; ts * t < cnt; ++t) {
            Task tk;
            tk.d = d;
            tk.start = s0 + ts * t;
            tk.count = min(ts, cnt - ts * t);
            tk.pad = u;
            tasks[t0 + t] = tk;
        }
    }
}

// ---------------------------------------------------------------------------
// Refinement: compact the flag bitmap and re-evaluate those elements exactly.
__global__ void k_count_flags(const uint32_t* __restrict__ bits, int64_t n_words,
                              unsigned long long* __restrict__ count) {
    unsigned long long c = 0;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_words;
         w += (int64_t)gridDim.x * blockDim.x)
        c += __popc(bits[w]);
    c = warp_sum_u64(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

__global__ void k_compact_flags(const uint32_t* __restrict__ bits, int64_t n_words,
                                int64_t* __restrict__ list, unsigned long long* __restrict__ cur) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_words;
         w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t b = bits[w];
        if (!b) continue;
        unsigned long long pos = atomicAdd(cur, (unsigned long long)__popc(b));
        while (b) {
            const int i = __ffs(b) - 1;
            b &= b - 1;
            list[pos++] = w * 32 + i;
        }
    }
}

__device__ __forceinline__ double exact_element(const RefineCtx& c, int64_t sp, int64_t p,
                                                const double* tg) {
    if (c.offsets) {
        const dg_pair_offsets o = c.offsets[p];
        return correlate_exact(c.y64, c.y64 + c.stride, c.N, o.tdoa_samples, o.fdoa_hz, c.fs, tg);
    }
    const int64_t s = sp / c.pairs, pr = sp - s * c.pairs;
    long long tdoa;
    double fdoa;
    offsets_exact(c.x[p], c.y[p], c.z[p], c.pg[sp], c.fs, c.wl, &tdoa, &fdoa);
    const int ri = c.pair_rx[2 * pr], rj = c.pair_rx[2 * pr + 1];
    const double2* y1 = c.y64 + (s * c.R + ri) * c.stride;
    const double2* y2 = c.y64 + (s * c.R + rj) * c.stride;
    return correlate_exact(y1, y2, c.N, tdoa, fdoa, c.fs, tg);
}

// the exact offsets of every re-rank chain (cell ci, step sp) -> out[ci * SP + sp],
// for the host's libm phasor values (chain_trig)
__global__ void k_chain_offsets(const int* __restrict__ cells, int n, int SP, RefineCtx c,
                                dg_pair_offsets* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)n * SP;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ci = i / SP, sp = i - ci * SP;
        const int64_t p = cells[ci];
        dg_pair_offsets o;
        if (c.offsets) {
            o = c.offsets[p];
        } else {
            long long tdoa;
            offsets_exact(c.x[p], c.y[p], c.z[p], c.pg[sp], c.fs, c.wl, &tdoa, &o.fdoa_hz);
            o.tdoa_samples = tdoa;
        }
        out[i] = o;
    }
}

// Eq. 11 in FP64 for one element, split across a group of T threads (a warp, or
// a whole 256-thread CTA for long captures): thread t takes samples kb + t + T j
// with its own phasor (FP64 sincos of the exact FP64-reduced start phase, FP64
// recurrence by e^{i 2 pi T nu}); warp butterflies, then the warp sums in order.
// Agrees with the reference's single recurrence to ~1e-12 relative — far inside
// the 1e-4 contract the refinement exists to meet. T is chosen from N alone
// (refine_group), so every partition of a run computes the same bits.
constexpr int kRefThreads = 256;

template <int T>
__device__ double correlate_fp64_group(const double2* __restrict__ y1,
                                       const double2* __restrict__ y2, int N, long long d,
                                       double fdoa, double fs) {
    const int t = threadIdx.x % T, lane = threadIdx.x & 31;
    const long long kb = d < 0 ? -d : 0;
    const long long ke = (N - d) < N ? (N - d) : N;
    double acc_re = 0.0, acc_im = 0.0;
    if (kb < ke) {
        const double nu = fdoa / fs;
        const long long k0 = kb + t;
        const double ph0 = nu * (double)k0;
        double pr, pi_, rr, ri;
        sincospi(2.0 * (ph0 - rint(ph0)), &pi_, &pr);
        const double st = nu * (double)T;
        sincospi(2.0 * (st - rint(st)), &ri, &rr);
        const double2* b = y2 + d;
        for (long long k = k0; k < ke; k += T) {
            const double2 a = __ldg(y1 + k), bb = __ldg(b + k);
            const double zr = a.x * bb.x + a.y * bb.y, zi = a.y * bb.x - a.x * bb.y;
            acc_re += zr * pr - zi * pi_;
            acc_im += zr * pi_ + zi * pr;
            const double nr = pr * rr - pi_ * ri;
            pi_ = pr * ri + pi_ * rr;
            pr = nr;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        acc_re += __shfl_xor_sync(0xffffffffu, acc_re, o);
        acc_im += __shfl_xor_sync(0xffffffffu, acc_im, o);
    }
    if constexpr (T > 32) {
        __shared__ double part[2][T / 32];
        const int warp = threadIdx.x >> 5;
        if (lane == 0) {
            part[0][warp] = acc_re;
            part[1][warp] = acc_im;
        }
        __syncthreads();
        acc_re = acc_im = 0.0;
#pragma unroll
        for (int w = 0; w < T / 32; ++w) {
            acc_re += part[0][w];
            acc_im += part[1][w];
        }
        __syncthreads();  // `part` is reused by the next element
    }
    return sqrt(acc_re * acc_re + acc_im * acc_im);
}

// threads per element: the whole CTA for long captures (few, long chains), a warp
// otherwise; a function of N only
inline bool refine_cta(int N) { return N >= 131072; }

template <int T>
__global__ void __launch_bounds__(kRefThreads)
k_refine(const int64_t* __restrict__ list, int64_t n, RefineCtx c) {
    const int per = kRefThreads / T;
    for (int64_t i = (int64_t)blockIdx.x * per + threadIdx.x / T; i < n;
         i += (int64_t)gridDim.x * per) {
        const int64_t e = list[i];
        const int64_t sp = e / c.P, p = e - sp * c.P;
        double v;
        if (c.offsets) {
            const dg_pair_offsets o = c.offsets[p];
            v = correlate_fp64_group<T>(c.y64, c.y64 + c.stride, c.N, o.tdoa_samples, o.fdoa_hz,
                                        c.fs);
        } else {
            const int64_t s = sp / c.pairs, pr = sp - s * c.pairs;
            long long tdoa;
            double fdoa;
            offsets_exact(c.x[p], c.y[p], c.z[p], c.pg[sp], c.fs, c.wl, &tdoa, &fdoa);
            const int ri = c.pair_rx[2 * pr], rj = c.pair_rx[2 * pr + 1];
            v = correlate_fp64_group<T>(c.y64 + (s * c.R + ri) * c.stride,
                                        c.y64 + (s * c.R + rj) * c.stride, c.N, tdoa, fdoa, c.fs);
        }
        if (threadIdx.x % T == 0) c.raw[e] = v;
    }
}

// Batched refinement on a side stream (overlaps the FP32 correlation of later
// steps): `list` holds indices relative to element `base` of a bitmap laid out
// one P32-element row per step (P32 = P rounded up to 32), `count` is on the
// device (k_compact_flags), raw surfaces are dense [step][P].
template <int T>
__global__ void __launch_bounds__(kRefThreads)
k_refine_rows(const int64_t* __restrict__ list, const unsigned long long* __restrict__ count,
              int64_t base, int64_t P32, RefineCtx c) {
    const int64_t n = (int64_t)*count;
    const int per = kRefThreads / T;
    for (int64_t i = (int64_t)blockIdx.x * per + threadIdx.x / T; i < n;
         i += (int64_t)gridDim.x * per) {
        const int64_t e = base + list[i];
        const int64_t row = e / P32, p = e - row * P32;
        const int64_t sp = c.unit_step ? c.unit_step[row] : row;  // global step of the row
        const int64_t s = sp / c.pairs, pr = sp - s * c.pairs;
        long long tdoa;
        double fdoa;
        offsets_exact(c.x[p], c.y[p], c.z[p], c.pg[sp], c.fs, c.wl, &tdoa, &fdoa);
        const int ri = c.pair_rx[2 * pr], rj = c.pair_rx[2 * pr + 1];
        const double v = correlate_fp64_group<T>(c.y64 + (s * c.R + ri) * c.stride,
                                                 c.y64 + (s * c.R + rj) * c.stride, c.N, tdoa,
                                                 fdoa, c.fs);
        if (threadIdx.x % T == 0) c.raw[row * c.P + p] = v;
    }
}

// ---------------------------------------------------------------------------
// Accumulation (correlate_snapshot_all_pairs + accumulate_grids order).
__global__ void k_combine_pairs(const double* __restrict__ raw, int S, int pairs, int64_t P,
                                double* __restrict__ grids) {
    const int64_t total = (int64_t)S * P;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = i / P, p = i - s * P;
        const double* r = raw + s * pairs * P + p;
        double g = r[0];
        for (int q = 1; q < pairs; ++q) g = __dadd_rn(g, r[q * P]);
        grids[i] = g;
    }
}

// steps[step[u]][i] += units[u][i] over the units in order (multi-GPU slabs:
// the parts of a step hold disjoint candidates, so the sum is exact)
__global__ void k_sum_units(const double* __restrict__ units, int U, int64_t n,
                            const int* __restrict__ step, double* __restrict__ steps) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        for (int u = 0; u < U; ++u) {
            double* o = steps + (int64_t)step[u] * n + i;
            *o = __dadd_rn(*o, units[(int64_t)u * n + i]);
        }
}

__global__ void k_scale(double* __restrict__ v, int64_t P, const double* __restrict__ median) {
    const double m = *median;
    if (!(m > 0.0)) return;  // geolocate.hpp:120
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
         i += (int64_t)gridDim.x * blockDim.x)
        v[i] = __ddiv_rn(v[i], m);
}

// first: acc = g_0 + g_1 + ... (accumulate_grids, snapshot order); otherwise the
// chunk continues a running sum: acc = acc + g_0 + ... (the same additions in
// the same order, so a run accumulated chunk by chunk is bit-identical)
__global__ void k_accumulate(const double* __restrict__ grids, int S, int64_t P,
                             double* __restrict__ acc, int first) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        double a = first ? grids[p] : __dadd_rn(acc[p], grids[p]);
        for (int s = 1; s < S; ++s) a = __dadd_rn(a, grids[(int64_t)s * P + p]);
        acc[p] = a;
    }
}

__device__ __forceinline__ double warp_max(double v) {
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__global__ void k_max_partial(const double* __restrict__ v, int64_t P, double* __restrict__ part) {
    __shared__ double sm[32];
    double m = -DBL_MAX;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
         i += (int64_t)gridDim.x * blockDim.x)
        m = fmax(m, v[i]);
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : -DBL_MAX;
        m = warp_max(m);
        if (threadIdx.x == 0) part[blockIdx.x] = m;
    }
}

__global__ void k_max_final(const double* __restrict__ part, int n, double* __restrict__ out) {
    __shared__ double sm[32];
    double m = -DBL_MAX;
    for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, part[i]);
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : -DBL_MAX;
        m = warp_max(m);
        if (threadIdx.x == 0) *out = m;
    }
}

// Near-peak cells for the exact re-rank: every cell whose fast value is >= thr,
// counted, then listed in ascending flat index (CUB select, stable) so the
// candidate set never depends on atomic order.
__global__ void k_count_ge(const double* __restrict__ v, int64_t P, double thr,
                           unsigned long long* __restrict__ count) {
    unsigned long long c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
         i += (int64_t)gridDim.x * blockDim.x)
        c += v[i] >= thr ? 1ull : 0ull;
    c = warp_sum_u64(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

struct GeThreshold {
    const double* v;
    double thr;
    __device__ __forceinline__ bool operator()(const int& i) const { return v[i] >= thr; }
};

// cells[i] = the i-th selected cell; keys[i] = its fast value's bit pattern
// (order-preserving for v >= 0) for the descending sort of large selections
__global__ void k_gather_keys(const double* __restrict__ v, const int* __restrict__ cells, int n,
                              unsigned long long* __restrict__ keys) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        keys[i] = (unsigned long long)__double_as_longlong(v[cells[i]]);
}

// the exact values of the re-ranked cells written into a surface
__global__ void k_patch_cells(const int* __restrict__ cells, int n, const double* __restrict__ val,
                              double* __restrict__ surf) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        surf[cells[i]] = val[i];
}

// lowest flat index whose value equals the maximum (std::max_element on the
// fast surface; accumulate-only calls of sharded runs)
__global__ void k_first_max(const double* __restrict__ v, int64_t P, const double* __restrict__ vmax,
                            unsigned long long* __restrict__ idx) {
    const double m = *vmax;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
         i += (int64_t)gridDim.x * blockDim.x)
        if (v[i] == m) atomicMin(idx, (unsigned long long)i);
}

// Exact re-evaluation of the near-peak candidates into a private buffer
// ex[ci * SP + sp] (the returned surfaces are left untouched so they stay
// independent of how the grid is partitioned).
// Each (cell, snapshot-pair) is one sequential FP64 chain of N_ov iterations
// (the reference's order, bit-exact). With few items, one item per warp (lane
// 0 only) spreads the chains over SM sub-partitions so each runs at its own
// FP64 pipe's rate instead of sharing it: `stride` threads per item.
__global__ void k_rerank(const int* __restrict__ cells, const int* __restrict__ n_cells, int cap,
                         int SP, RefineCtx c, double* __restrict__ ex, int stride) {
    const int n = min(*n_cells, cap);
    const int64_t total = (int64_t)n * SP;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t % stride) return;
    for (int64_t i = t / stride; i < total; i += (int64_t)gridDim.x * blockDim.x / stride) {
        const int64_t ci = i / SP, sp = i - ci * SP;
        ex[i] = exact_element(c, sp, cells[ci], c.trig ? c.trig + 4 * i : nullptr);
    }
}

// The same exact chains with the work of one chain spread over the four warps of
// a CTA (bit-identical: every FP64 operation and its order are the reference's,
// only the thread that executes it changes). Tiles of kRrT samples, three stages
// in flight: in iteration t, warp 2 lane 0 runs the phasor recurrence for tile
// t+1 (the critical chain: a dependent DMUL + DADD per sample), warp 1 forms the
// products p_k = y1[k] conj(y2[k+d]) of tile t+1 (all of a lane's loads issued
// before its arithmetic: one memory latency per tile), warp 3 the terms
// q_k = p_k ph_k of tile t, and warp 0 lane 0 adds the terms of tile t-1 in
// sample order (acc += q_k: two independent DADDs per sample).
constexpr int kRrT = 256;
constexpr int kRrThreads = 128;

__device__ void exact_chain_cta(const double2* __restrict__ y1, const double2* __restrict__ y2,
                                int N, long long d, double fdoa, double fs, const double* tg,
                                double* out) {
    __shared__ double2 pbuf[2][kRrT], hbuf[2][kRrT], qbuf[2][kRrT];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long kb = d < 0 ? -d : 0;
    const long long ke = (N - d) < N ? (N - d) : N;
    if (kb >= ke) {
        if (tid == 0) *out = 0.0;
        return;
    }
    double rot_im, rot_re, ph_im, ph_re;
    chain_trig(kb, fdoa, fs, tg, &rot_re, &rot_im, &ph_re, &ph_im);
    double acc_re = 0.0, acc_im = 0.0;
    const double2* b = y2 + d;
    const long long n = ke - kb;
    const int ntile = (int)((n + kRrT - 1) / kRrT);
    auto tile_len = [&](int t) { return (int)min((long long)kRrT, n - (long long)t * kRrT); };
    auto products = [&](int t) {  // warp 1: p of tile t into pbuf[t & 1]
        const long long k0 = kb + (long long)t * kRrT;
        const int len = tile_len(t), bf = t & 1;
        constexpr int J = kRrT / 32;
        double2 a[J], bb[J];
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int i = lane + 32 * j;
            if (i < len) {
                a[j] = __ldg(y1 + k0 + i);
                bb[j] = __ldg(b + k0 + i);
            }
        }
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int i = lane + 32 * j;
            if (i < len) {
                const double b_re = bb[j].x, b_im = -bb[j].y;
                pbuf[bf][i] =
                    make_double2(__dsub_rn(__dmul_rn(a[j].x, b_re), __dmul_rn(a[j].y, b_im)),
                                 __dadd_rn(__dmul_rn(a[j].x, b_im), __dmul_rn(a[j].y, b_re)));
            }
        }
    };
    auto phasors = [&](int t) {  // warp 2 lane 0: ph of tile t into hbuf[t & 1]
        const int len = tile_len(t), bf = t & 1;
#pragma unroll 4
        for (int i = 0; i < len; ++i) {
            hbuf[bf][i] = make_double2(ph_re, ph_im);
            const double nr = __dsub_rn(__dmul_rn(ph_re, rot_re), __dmul_rn(ph_im, rot_im));
            ph_im = __dadd_rn(__dmul_rn(ph_re, rot_im), __dmul_rn(ph_im, rot_re));
            ph_re = nr;
        }
    };
    if (warp == 1) products(0);
    else if (warp == 2 && lane == 0) phasors(0);
    __syncthreads();
    for (int t = 0; t <= ntile; ++t) {
        if (warp == 2) {
            if (lane == 0 && t + 1 < ntile) phasors(t + 1);
        } else if (warp == 1) {
            if (t + 1 < ntile) products(t + 1);
        } else if (warp == 3) {
            if (t < ntile) {  // terms of tile t (its p and ph were written last iteration)
                const int len = tile_len(t), bf = t & 1;
                for (int i = lane; i < len; i += 32) {
                    const double2 pk = pbuf[bf][i], hk = hbuf[bf][i];
                    qbuf[bf][i] =
                        make_double2(__dsub_rn(__dmul_rn(pk.x, hk.x), __dmul_rn(pk.y, hk.y)),
                                     __dadd_rn(__dmul_rn(pk.x, hk.y), __dmul_rn(pk.y, hk.x)));
                }
            }
        } else if (lane == 0 && t > 0) {  // warp 0: sum the terms of tile t-1
            const int len = tile_len(t - 1), bf = (t - 1) & 1;
#pragma unroll 8
            for (int i = 0; i < len; ++i) {
                const double2 q = qbuf[bf][i];
                acc_re = __dadd_rn(acc_re, q.x);
                acc_im = __dadd_rn(acc_im, q.y);
            }
        }
        __syncthreads();
    }
    if (tid == 0)
        *out = __dsqrt_rn(__dadd_rn(__dmul_rn(acc_re, acc_re), __dmul_rn(acc_im, acc_im)));
}

__global__ void __launch_bounds__(kRrThreads)
k_rerank_cta(const int* __restrict__ cells, const int* __restrict__ n_cells, int cap, int SP,
             RefineCtx c, double* __restrict__ ex) {
    const int n = min(*n_cells, cap);
    const int64_t total = (int64_t)n * SP;
    for (int64_t i = blockIdx.x; i < total; i += gridDim.x) {
        const int64_t ci = i / SP, sp = i - ci * SP;
        const int64_t p = cells[ci];
        const double2 *y1, *y2;
        long long tdoa;
        double fdoa;
        if (c.offsets) {
            tdoa = c.offsets[p].tdoa_samples;
            fdoa = c.offsets[p].fdoa_hz;
            y1 = c.y64;
            y2 = c.y64 + c.stride;
        } else {
            const int64_t s = sp / c.pairs, pr = sp - s * c.pairs;
            offsets_exact(c.x[p], c.y[p], c.z[p], c.pg[sp], c.fs, c.wl, &tdoa, &fdoa);
            y1 = c.y64 + (s * c.R + c.pair_rx[2 * pr]) * c.stride;
            y2 = c.y64 + (s * c.R + c.pair_rx[2 * pr + 1]) * c.stride;
        }
        exact_chain_cta(y1, y2, c.N, tdoa, fdoa, c.fs, c.trig ? c.trig + 4 * i : nullptr, ex + i);
        __syncthreads();
    }
}

// per candidate: pair sums (correlate_snapshot_all_pairs), optional median
// scaling, accumulation over snapshots in order (accumulate_grids)
__global__ void k_recombine_cells(const int* __restrict__ n_cells, int cap,
                                  const double* __restrict__ ex, int S, int pairs,
                                  const double* __restrict__ medians, double* __restrict__ acc_ex,
                                  double* __restrict__ grid_ex) {
    const int n = min(*n_cells, cap);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double* r = ex + (int64_t)i * S * pairs;
        double a = 0.0;
        for (int s = 0; s < S; ++s) {
            double g = r[s * pairs];
            for (int q = 1; q < pairs; ++q) g = __dadd_rn(g, r[s * pairs + q]);
            if (medians && medians[s] > 0.0) g = __ddiv_rn(g, medians[s]);
            grid_ex[(int64_t)i * S + s] = g;
            a = s ? __dadd_rn(a, g) : g;
        }
        acc_ex[i] = a;
    }
}

// single block: exact max over the re-ranked cells, lowest flat index on ties
// (std::max_element keeps the first maximum)
__global__ void k_argmax_cells(const int* __restrict__ cells, const int* __restrict__ n_cells,
                               int cap, const double* __restrict__ acc_ex,
                               long long* __restrict__ best_idx, double* __restrict__ best_val) {
    __shared__ double sv[1024];
    __shared__ long long si[1024];
    const int n = min(*n_cells, cap);
    double bv = -DBL_MAX;
    long long bi = LLONG_MAX;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const long long p = cells[i];
        const double v = acc_ex[i];
        if (v > bv || (v == bv && p < bi)) {
            bv = v;
            bi = p;
        }
    }
    sv[threadIdx.x] = bv;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int s = blockDim.x / 2; s; s >>= 1) {
        if (threadIdx.x < s) {
            const double v = sv[threadIdx.x + s];
            const long long p = si[threadIdx.x + s];
            if (v > sv[threadIdx.x] || (v == sv[threadIdx.x] && p < si[threadIdx.x])) {
                sv[threadIdx.x] = v;
                si[threadIdx.x] = p;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *best_idx = si[0];
        *best_val = sv[0];
    }
}

// ---------------------------------------------------------------------------
// Median (geolocate.hpp:115-122: nth_element at size/2) by 8-bit radix select
// over the IEEE bit patterns (order-preserving for S >= 0).
// state[0] = prefix, state[1] = remaining rank
__global__ void k_radix_hist(const double* __restrict__ v, int64_t P, int shift,
                             const unsigned long long* __restrict__ state,
                             unsigned* __restrict__ hist) {
    __shared__ unsigned sh[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const unsigned long long prefix = state[0];
    const unsigned long long hi_mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = (unsigned long long)__double_as_longlong(v[i]);
        if ((key & hi_mask) == (prefix & hi_mask)) atomicAdd(&sh[(key >> shift) & 255], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

__global__ void k_radix_pick(unsigned* __restrict__ hist, int shift,
                             unsigned long long* __restrict__ state, double* __restrict__ out) {
    if (threadIdx.x == 0) {
        unsigned long long rank = state[1], cum = 0;
        int digit = 255;
        for (int i = 0; i < 256; ++i) {
            if (cum + hist[i] > rank) {
                digit = i;
                break;
            }
            cum += hist[i];
        }
        state[0] |= (unsigned long long)digit << shift;
        state[1] = rank - cum;
        if (shift == 0) *out = __longlong_as_double((long long)state[0]);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
}

// ---------------------------------------------------------------------------
// detect_emitters (correlate.hpp:127-201)
__device__ __forceinline__ double warp_sumd(double v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// fixed-shape tree reductions (deterministic); mode 0: sum v, mode 1: sum (v-mean)^2
__global__ void k_sum_partial(const double* __restrict__ v, int64_t P, const double* __restrict__ stats,
                              int mode, double* __restrict__ part) {
    __shared__ double sm[32];
    const double mean = mode ? stats[0] : 0.0;
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double x = v[i];
        s += mode ? (x - mean) * (x - mean) : x;
    }
    s = warp_sumd(s);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
        s = warp_sumd(s);
        if (threadIdx.x == 0) part[blockIdx.x] = s;
    }
}

__global__ void k_sum_final(const double* __restrict__ part, int n, int64_t P, int mode,
                            double* __restrict__ stats) {
    __shared__ double sm[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
    s = warp_sumd(s);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
        s = warp_sumd(s);
        if (threadIdx.x == 0) {
            const double m = s / (double)P;
            if (mode == 0) {
                stats[0] = m;
            } else {
                stats[1] = m;
                stats[2] = sqrt(m);
            }
        }
    }
}

__global__ void k_local_max(const double* __restrict__ v, int64_t n_lat, int64_t n_lon,
                            const double* __restrict__ stats, double k_sigma,
                            DetCand* __restrict__ cands, int* __restrict__ n_cands, int cap) {
    const double sigma = stats[2];
    if (sigma == 0.0) return;
    const double thr = stats[0] + k_sigma * sigma;
    const int64_t P = n_lat * n_lon;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        const double x = v[p];
        if (x <= thr) continue;
        const int64_t i = p / n_lon, j = p - i * n_lon;
        bool is_max = true;
        for (int di = -1; di <= 1 && is_max; ++di)
            for (int dj = -1; dj <= 1 && is_max; ++dj) {
                if (!di && !dj) continue;
                const int64_t ni = i + di, nj = j + dj;
                if (ni < 0 || ni >= n_lat || nj < 0 || nj >= n_lon) continue;
                if (v[ni * n_lon + nj] > x) is_max = false;
            }
        if (!is_max) continue;
        const int pos = atomicAdd(n_cands, 1);
        if (pos < cap) {
            DetCand c;
            c.score = x;
            c.key = (long long)i * 1000000LL + j;
            c.ilat = (int)i;
            c.ilon = (int)j;
            cands[pos] = c;
        }
    }
}

// single block: sort by (score desc, key asc) then greedy Chebyshev exclusion
__device__ __forceinline__ bool cand_before(const DetCand& a, const DetCand& b) {
    if (a.score != b.score) return a.score > b.score;
    return a.key < b.key;
}

__global__ void k_greedy(const DetCand* __restrict__ cands, const int* __restrict__ n_cands,
                         int cap, int radius, const double* __restrict__ stats, int64_t n_lon,
                         dg_emitter_estimate* __restrict__ out, int* __restrict__ n_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    DetCand* c = reinterpret_cast<DetCand*>(smem);
    const int n = min(*n_cands, cap);
    int m = 1;
    while (m < n) m <<= 1;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        if (i < n) {
            c[i] = cands[i];
        } else {
            c[i].score = -DBL_MAX;
            c[i].key = LLONG_MAX;
        }
    }
    __syncthreads();
    for (int k = 2; k <= m; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < m; i += blockDim.x) {
                const int l = i ^ j;
                if (l > i) {
                    const bool up = (i & k) == 0;
                    const bool swap = up ? cand_before(c[l], c[i]) : cand_before(c[i], c[l]);
                    if (swap) {
                        const DetCand t = c[i];
                        c[i] = c[l];
                        c[l] = t;
                    }
                }
            }
            __syncthreads();
        }
    // the greedy pass (correlate.hpp:177-199): candidate i (in sorted order) is
    // kept iff no kept candidate before it lies within the Chebyshev radius.
    // Blocks of 32 candidates in order: (A) all threads test the block against
    // the kept list of the earlier blocks (one rejection bit per candidate);
    // (B) warp 0 resolves the block itself: each lane's mask of conflicting
    // earlier lanes, then the 32-step keep rule on bit masks, and appends the
    // kept ones. A single warp walking the candidates one by one is
    // latency-bound (~800 cycles per candidate at C3).
    unsigned char* stat = reinterpret_cast<unsigned char*>(c + m);  // 1 kept, 2 rejected
    unsigned short* klist = reinterpret_cast<unsigned short*>(stat + ((m + 15) & ~15));
    __shared__ unsigned rejmask;
    __shared__ int nkept;
    if (threadIdx.x == 0) {
        rejmask = 0;
        nkept = 0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (int base = 0; base < n; base += 32) {
        const int nb = min(32, n - base);
        const int nk = nkept;
        unsigned my = 0;
        for (int k = threadIdx.x; k < nk; k += blockDim.x) {  // (A)
            const DetCand& kc = c[klist[k]];
            const int kl = kc.ilat, kn = kc.ilon;
            for (int q = 0; q < nb; ++q)
                if (max(abs(kl - c[base + q].ilat), abs(kn - c[base + q].ilon)) <= radius)
                    my |= 1u << q;
        }
        if (my) atomicOr(&rejmask, my);
        __syncthreads();
        if (threadIdx.x < 32) {  // (B)
            const int i = base + lane;
            const bool valid = lane < nb;
            const bool alive = valid && !((rejmask >> lane) & 1u);
            unsigned pm = 0;  // earlier lanes of this block within the radius
            if (alive) {
                const int li = c[i].ilat, ni = c[i].ilon;
                for (int q = 0; q < lane; ++q)
                    if (max(abs(li - c[base + q].ilat), abs(ni - c[base + q].ilon)) <= radius)
                        pm |= 1u << q;
            }
            const unsigned am = __ballot_sync(0xffffffffu, alive);
            unsigned kept = 0;
#pragma unroll
            for (int q = 0; q < 32; ++q) {
                const unsigned pmq = __shfl_sync(0xffffffffu, pm, q);
                if (((am >> q) & 1u) && !(pmq & kept)) kept |= 1u << q;
            }
            const bool keep = (kept >> lane) & 1u;
            if (valid) stat[i] = keep ? 1 : 2;
            if (keep) klist[nk + __popc(kept & ((1u << lane) - 1))] = (unsigned short)i;
            __syncwarp();
            if (lane == 0) {
                nkept = nk + __popc(kept);
                rejmask = 0;
            }
        }
        __syncthreads();
    }
    // kept candidates in sorted order (one warp, ballot compaction)
    if (threadIdx.x < 32) {
        int acc = 0;
        for (int base = 0; base < n; base += 32) {
            const int i = base + lane;
            const bool keep = i < n && stat[i] == 1;
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const DetCand cur = c[i];
                dg_emitter_estimate e;
                e.lat_deg = (double)cur.ilat;  // lattice coordinates filled in on the host
                e.lon_deg = (double)cur.ilon;
                e.alt_m = 0.0;
                e.grid_index = (int64_t)cur.ilat * n_lon + cur.ilon;
                e.score = cur.score;
                e.score_zsigma = (cur.score - stats[0]) / stats[2];
                out[acc + __popc(bal & ((1u << lane) - 1))] = e;
            }
            acc += __popc(bal);
        }
        if (lane == 0) *n_out = acc;
    }
}

__global__ void k_f64_to_f32(const double2* __restrict__ in, float2* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double2 v = in[i];
        out[i] = make_float2((float)v.x, (float)v.y);
    }
}

// captures [n_caps][N] (contiguous, as uploaded) -> the padded slots of both
// resident copies, pads zeroed: slot c element i holds sample i - pad
template <typename T>
__global__ void k_stage_captures(const T* __restrict__ in, int64_t n_caps, int64_t N,
                                 int64_t stride, int64_t pad, double2* __restrict__ y64,
                                 float2* __restrict__ y32) {
    const int64_t n = n_caps * stride;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i / stride, k = i - c * stride - pad;
        double2 v = make_double2(0.0, 0.0);
        if (k >= 0 && k < N) {
            const T w = in[c * N + k];
            v = make_double2((double)w.x, (double)w.y);
        }
        y64[i] = v;
        y32[i] = make_float2((float)v.x, (float)v.y);
    }
}

__global__ void k_f32_to_f64(const float2* __restrict__ in, double2* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float2 v = in[i];
        out[i] = make_double2((double)v.x, (double)v.y);
    }
}

}  // namespace

// ===========================================================================
// launchers
void launch_grid_ecef(const double* ra, const double* rz, const double* cc, const double* cs,
                      int64_t n_lat, int64_t n_lon, double* x, double* y, double* z,
                      cudaStream_t st) {
    k_grid_ecef<<<blocks_for(n_lat * n_lon, 256), 256, 0, st>>>(ra, rz, cc, cs, n_lat, n_lon, x, y,
                                                               z);
}

void launch_geometry_hist(const double* x, const double* y, const double* z, int64_t P,
                          const PairGeom* pg, double fs, double wl, int N, int* d_out,
                          int* rank_out, double* fdoa_out, int* hist, double* s_out,
                          unsigned long long* overlap, int* err, StepRange* range,
                          cudaStream_t st) {
    k_geometry_hist<<<blocks_for(P, 256), 256, 0, st>>>(x, y, z, P, pg, fs, wl, N, d_out, rank_out,
                                                        fdoa_out, hist, s_out, overlap, err, range);
}

void launch_geometry_units(const double* x, const double* y, const double* z, int64_t P,
                           const PairGeom* pg, int n, double fs, double wl, int N, int* d_out,
                           int* rank_out, double* fdoa_out, int* hist, int nbins, double* s_out,
                           unsigned long long* overlap, int* err, GeoScratch* ws,
                           cudaStream_t st) {
    const auto same = [](const dg_state& a, const dg_state& b) {
        return std::memcmp(&a, &b, sizeof(dg_state)) == 0;
    };
    for (int s0 = 0; s0 < n; s0 += kGeoUnitsMax) {
        const int m = n - s0 < kGeoUnitsMax ? n - s0 : kGeoUnitsMax;
        // host: group consecutive units whose receivers fit one table (the pairs
        // of one snapshot), receivers deduplicated bitwise
        GeoScratch& h = ws[s0 / kGeoUnitsMax];
        h.nrx = h.ng = 0;
        for (int u = 0; u < m; ++u) {
            const PairGeom& g = pg[s0 + u];
            GeoGroup* cur = h.ng ? &h.groups[h.ng - 1] : nullptr;
            auto find = [&](const dg_state& st) {
                for (int r = 0; cur && r < cur->nrx; ++r)
                    if (same(h.rx[cur->rx0 + r], st)) return r;
                return -1;
            };
            int a = find(g.rx_i), b = find(g.rx_j);
            const int need = (a < 0) + (b < 0 && !same(g.rx_i, g.rx_j));
            // a new group unless this unit shares a receiver with the current one
            // (pairs of one snapshot) and its receivers fit the table
            if (!cur || (a < 0 && b < 0) || cur->nrx + need > kGeoRxMax) {
                h.groups[h.ng++] = GeoGroup{h.nrx, 0, u, 0};
                cur = &h.groups[h.ng - 1];
                a = b = -1;
            }
            if (a < 0) {
                h.rx[h.nrx++] = g.rx_i;
                a = cur->nrx++;
            }
            if (b < 0) {
                b = same(g.rx_i, g.rx_j) ? a : -1;
                if (b < 0) {
                    h.rx[h.nrx++] = g.rx_j;
                    b = cur->nrx++;
                }
            }
            h.upair[u] = make_int2(a, b);
            cur->nu++;
        }
        cudaMemcpyAsync(h.d_rx, h.rx, h.nrx * sizeof(dg_state), cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(h.d_groups, h.groups, h.ng * sizeof(GeoGroup), cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(h.d_upair, h.upair, m * sizeof(int2), cudaMemcpyHostToDevice, st);
        int kr = 2;
        for (int g = 0; g < h.ng; ++g) kr = std::max(kr, h.groups[g].nrx);
        auto kern = kr <= 2 ? k_geometry_units<2> : kr <= 4 ? k_geometry_units<4>
                                                             : k_geometry_units<kGeoRxMax>;
        kern<<<blocks_for(P, 256, 148LL * 8), 256, 0, st>>>(
            x, y, z, P, h.d_rx, h.nrx, h.d_groups, h.ng, h.d_upair, m, fs, wl, N,
            d_out + (int64_t)s0 * P, rank_out + (int64_t)s0 * P, fdoa_out + (int64_t)s0 * P,
            hist + (int64_t)s0 * nbins, nbins, s_out + (int64_t)s0 * P, overlap, err);
    }
}

void launch_energy_prefix(const double2* y, int64_t stride, int64_t n_caps, int64_t N,
                          double* out, cudaStream_t st) {
    if (n_caps > 0) k_energy_prefix<<<(int)n_caps, kEnergyThreads, 0, st>>>(y, stride, N, out);
}

void launch_hist_range(const int* hist, int nbins, int n_steps, int N, StepRange* out,
                       cudaStream_t st) {
    k_range_init<<<1, 256, 0, st>>>(out, n_steps);
    const int chunks = (nbins + kHistRangeChunk - 1) / kHistRangeChunk;
    k_hist_range<<<dim3(chunks, n_steps), kHistRangeThreads, 0, st>>>(hist, nbins, N, out);
}

void launch_predict_offsets(const double* x, const double* y, const double* z, int64_t P,
                            const PairGeom* pg, double fs, double wl, dg_pair_offsets* out, int* err,
                            cudaStream_t st) {
    k_predict_offsets<<<blocks_for(P, 256), 256, 0, st>>>(x, y, z, P, pg, fs, wl, out, err);
}

void launch_offsets_hist(const dg_pair_offsets* off, int64_t P, int N, int* d_out,
                         int* rank_out, double* fdoa_out, int* hist, double* s_out,
                         unsigned long long* overlap, StepRange* range, cudaStream_t st) {
    k_offsets_hist<<<blocks_for(P, 256), 256, 0, st>>>(off, P, N, d_out, rank_out, fdoa_out, hist,
                                                       s_out, overlap, range);
}

void launch_lattice_rel(const double* x, const double* y, const double* z, int64_t P, double cx,
                        double cy, double cz, float4* out, cudaStream_t st) {
    k_lattice_rel<<<blocks_for(P, 256), 256, 0, st>>>(x, y, z, P, cx, cy, cz, out);
}

void launch_range_fp32(const float4* rel, int64_t P, const RxPairF32* rx, int n_steps, double fs,
                       double wl, StepRange* out, cudaStream_t st) {
    if (P <= 0 || n_steps <= 0) return;
    k_range_fp32<<<blocks_for(P, kRangeThreads, 148LL * 8), kRangeThreads, 0, st>>>(
        rel, P, rx, n_steps, (float)(fs / kC), (float)(1.0 / wl), out);
}

void launch_bucket(int* hist, int bin0, int nb, int N, int* off, int* toff, int* boff,
                   int* cursor, int* n_tasks, int* n_buckets, const int* d, const int* rank,
                   int64_t P, int* sorted, Task* tasks, Bucket* buckets, int* ubin, int B,
                   cudaStream_t st, const double* fdoa, double* sfdoa) {
    const int ts = correlate_task_size();
    k_scan<<<1, kScanThreads, 0, st>>>(hist + bin0, nb, ts, off + bin0, toff + bin0, boff + bin0,
                                       cursor + bin0, n_tasks, n_buckets);
    k_scatter<<<blocks_for(P, 256), 256, 0, st>>>(d, rank, P, N, bin0, nb, off, sorted, fdoa, sfdoa);
    k_build_tasks<<<blocks_for(nb, 256), 256, 0, st>>>(hist + bin0, nb, bin0, N, ts, off + bin0,
                                                      toff + bin0, boff + bin0, tasks, buckets, ubin, B);
}

void launch_count_flags(const uint32_t* bits, int64_t n_words, unsigned long long* count,
                        cudaStream_t st) {
    k_count_flags<<<blocks_for(n_words, 256), 256, 0, st>>>(bits, n_words, count);
}

void launch_compact_flags(const uint32_t* bits, int64_t n_words, int64_t* list,
                          unsigned long long* cursor, cudaStream_t st) {
    k_compact_flags<<<blocks_for(n_words, 256), 256, 0, st>>>(bits, n_words, list, cursor);
}

void launch_refine_rows(const uint32_t* bits, int64_t row0, int64_t row1, int64_t P32,
                        int64_t* list, unsigned long long* count, RefineCtx ctx, cudaStream_t st) {
    const int64_t w0 = row0 * (P32 / 32), nw = (row1 - row0) * (P32 / 32);
    cudaMemsetAsync(count, 0, sizeof(unsigned long long), st);
    k_compact_flags<<<blocks_for(nw, 256, 148LL * 8), 256, 0, st>>>(bits + w0, nw, list, count);
    if (refine_cta(ctx.N))
        k_refine_rows<kRefThreads><<<148 * 8, kRefThreads, 0, st>>>(list, count, row0 * P32, P32,
                                                                    ctx);
    else
        k_refine_rows<32><<<148 * 16, kRefThreads, 0, st>>>(list, count, row0 * P32, P32, ctx);
}

void launch_refine(const int64_t* list, int64_t n, RefineCtx ctx, cudaStream_t st) {
    if (n <= 0) return;
    if (refine_cta(ctx.N))
        k_refine<kRefThreads><<<(int)std::min<int64_t>(n, 148 * 8), kRefThreads, 0, st>>>(list, n,
                                                                                         ctx);
    else
        k_refine<32><<<blocks_for(n * 32, kRefThreads, 148LL * 16), kRefThreads, 0, st>>>(list, n,
                                                                                         ctx);
}

void launch_combine_pairs(const double* raw, int S, int pairs, int64_t P, double* grids,
                          cudaStream_t st) {
    k_combine_pairs<<<blocks_for((int64_t)S * P, 256), 256, 0, st>>>(raw, S, pairs, P, grids);
}

void launch_sum_units(const double* units, int U, int64_t n, const int* step, double* steps,
                      cudaStream_t st) {
    if (U > 0 && n > 0) k_sum_units<<<blocks_for(n, 256), 256, 0, st>>>(units, U, n, step, steps);
}

void launch_scale(double* v, int64_t P, const double* median, cudaStream_t st) {
    k_scale<<<blocks_for(P, 256), 256, 0, st>>>(v, P, median);
}

void launch_accumulate(const double* grids, int S, int64_t P, double* acc, cudaStream_t st,
                       bool first) {
    k_accumulate<<<blocks_for(P, 256), 256, 0, st>>>(grids, S, P, acc, first ? 1 : 0);
}

void launch_max(const double* v, int64_t P, double* partial, int n_partial, double* out,
                cudaStream_t st) {
    k_max_partial<<<n_partial, 256, 0, st>>>(v, P, partial);
    k_max_final<<<1, 1024, 0, st>>>(partial, n_partial, out);
}

void launch_count_ge(const double* v, int64_t P, double thr, unsigned long long* count,
                     cudaStream_t st) {
    k_count_ge<<<blocks_for(P, 256, 148LL * 8), 256, 0, st>>>(v, P, thr, count);
}

size_t select_ge_temp_bytes(int64_t P, int n_sel) {
    size_t a = 0, b = 0;
    cub::DeviceSelect::If(nullptr, a, thrust::counting_iterator<int>(0), (int*)nullptr,
                          (int*)nullptr, (int)P, GeThreshold{nullptr, 0.0});
    cub::DeviceRadixSort::SortPairsDescending(nullptr, b, (const unsigned long long*)nullptr,
                                              (unsigned long long*)nullptr, (const int*)nullptr,
                                              (int*)nullptr, n_sel);
    return std::max(a, b);
}

void launch_select_ge(const double* v, int64_t P, double thr, int* cells, int* n_out, void* temp,
                      size_t temp_bytes, cudaStream_t st) {
    cub::DeviceSelect::If(temp, temp_bytes, thrust::counting_iterator<int>(0), cells, n_out,
                          (int)P, GeThreshold{v, thr}, st);
}

void launch_sort_by_value(const double* v, const int* cells, int n, unsigned long long* keys,
                          unsigned long long* keys_out, int* cells_out, void* temp,
                          size_t temp_bytes, cudaStream_t st) {
    k_gather_keys<<<blocks_for(n, 256), 256, 0, st>>>(v, cells, n, keys);
    // radix sort is stable: equal values keep ascending flat index
    cub::DeviceRadixSort::SortPairsDescending(temp, temp_bytes, keys, keys_out, cells, cells_out, n,
                                              0, 64, st);
}

void launch_patch_cells(const int* cells, int n, const double* val, double* surf, cudaStream_t st) {
    if (n > 0) k_patch_cells<<<blocks_for(n, 256), 256, 0, st>>>(cells, n, val, surf);
}

void launch_first_max(const double* v, int64_t P, const double* vmax, unsigned long long* idx,
                      cudaStream_t st) {
    k_first_max<<<blocks_for(P, 256, 148LL * 8), 256, 0, st>>>(v, P, vmax, idx);
}

void launch_rerank(const int* cells, const int* n_cells, int cap, int n_items_hint, int SP,
                   RefineCtx ctx, double* ex, cudaStream_t st) {
    const int64_t items = (int64_t)std::min(n_items_hint, cap) * SP;
    if (items <= 148 * 16) {  // one four-warp CTA per chain
        k_rerank_cta<<<(int)std::max<int64_t>(items, 1), kRrThreads, 0, st>>>(cells, n_cells, cap, SP,
                                                                      ctx, ex);
        return;
    }
    k_rerank<<<blocks_for((int64_t)cap * SP, 64, 148LL * 64), 64, 0, st>>>(cells, n_cells, cap,
                                                                           SP, ctx, ex, 1);
}

void launch_chain_offsets(const int* cells, int n, int SP, RefineCtx ctx, dg_pair_offsets* out,
                          cudaStream_t st) {
    k_chain_offsets<<<blocks_for((int64_t)n * SP, 128), 128, 0, st>>>(cells, n, SP, ctx, out);
}

void launch_recombine_cells(const int* n_cells, int cap, const double* ex, int S, int pairs,
                            const double* medians, double* acc_ex, double* grid_ex,
                            cudaStream_t st) {
    k_recombine_cells<<<blocks_for(cap, 128), 128, 0, st>>>(n_cells, cap, ex, S, pairs, medians,
                                                            acc_ex, grid_ex);
}

void launch_argmax_cells(const int* cells, const int* n_cells, int cap, const double* acc_ex,
                         long long* best_idx, double* best_val, cudaStream_t st) {
    k_argmax_cells<<<1, 1024, 0, st>>>(cells, n_cells, cap, acc_ex, best_idx, best_val);
}

void launch_median(const double* v, int64_t P, unsigned* hist, unsigned long long* state,
                   double* out, cudaStream_t st) {
    // state must hold {0, P/2}; hist zeroed
    for (int shift = 56; shift >= 0; shift -= 8) {
        k_radix_hist<<<blocks_for(P, 256, 148LL * 8), 256, 0, st>>>(v, P, shift, state, hist);
        k_radix_pick<<<1, 256, 0, st>>>(hist, shift, state, out);
    }
}

void launch_mean_var(const double* v, int64_t P, double* partial, int n_partial, double* stats,
                     cudaStream_t st) {
    k_sum_partial<<<n_partial, 256, 0, st>>>(v, P, stats, 0, partial);
    k_sum_final<<<1, 1024, 0, st>>>(partial, n_partial, P, 0, stats);
    k_sum_partial<<<n_partial, 256, 0, st>>>(v, P, stats, 1, partial);
    k_sum_final<<<1, 1024, 0, st>>>(partial, n_partial, P, 1, stats);
}

void launch_local_max(const double* v, int64_t n_lat, int64_t n_lon, const double* stats,
                      double k_sigma, DetCand* cands, int* n_cands, int cap, cudaStream_t st) {
    k_local_max<<<blocks_for(n_lat * n_lon, 256), 256, 0, st>>>(v, n_lat, n_lon, stats, k_sigma,
                                                               cands, n_cands, cap);
}

void launch_greedy(const DetCand* cands, const int* n_cands, int cap, int radius,
                   const double* stats, int64_t n_lon, dg_emitter_estimate* out, int* n_out,
                   cudaStream_t st) {
    int m = 1;
    while (m < cap) m <<= 1;
    // candidates, statuses, kept list
    const size_t smem = (size_t)m * sizeof(DetCand) + ((m + 15) & ~15) + (size_t)m * 2;
    cudaFuncSetAttribute(k_greedy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_greedy<<<1, 1024, smem, st>>>(cands, n_cands, cap, radius, stats, n_lon, out, n_out);
}

void launch_f64_to_f32(const double2* in, float2* out, int64_t n, cudaStream_t st) {
    k_f64_to_f32<<<blocks_for(n, 256), 256, 0, st>>>(in, out, n);
}

void launch_stage_captures(const void* in, bool f64, int64_t n_caps, int64_t N, int64_t stride,
                           int64_t pad, double2* y64, float2* y32, cudaStream_t st) {
    const int64_t n = n_caps * stride;
    if (f64)
        k_stage_captures<double2><<<blocks_for(n, 256), 256, 0, st>>>(
            static_cast<const double2*>(in), n_caps, N, stride, pad, y64, y32);
    else
        k_stage_captures<float2><<<blocks_for(n, 256), 256, 0, st>>>(
            static_cast<const float2*>(in), n_caps, N, stride, pad, y64, y32);
}

void launch_f32_to_f64(const float2* in, double2* out, int64_t n, cudaStream_t st) {
    k_f32_to_f64<<<blocks_for(n, 256), 256, 0, st>>>(in, out, n);
}

}  // namespace dg
