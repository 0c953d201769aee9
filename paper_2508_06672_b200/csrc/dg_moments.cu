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
//               M_m[b] on FFMA2 with the Chebyshev table broadcast from smem (the
//               direct sums: B < 256, the FFMA2 evaluator, or tuning moment_fft = 0;
//               otherwise dg_moments_fft.cu computes the same moments by FFTs)
//   k_evaluate  one warp = up to 64 candidates of one bucket (2 per lane):
//               J_m(x) by series + backward recurrence (FP64), block loop on
//               FFMA2 with the bucket's moments as broadcast loads, Horner in
//               FP32 within groups of G blocks, FP64-reduced anchors, FP64 sum.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <type_traits>

#include "dg_device.cuh"
#include "dg_internal.cuh"

namespace dg {

namespace {

constexpr int kEvalStages = 3;  // bucket-moment buffers in k_evaluate's TMA ring
inline size_t evaluate_smem(int nbmax, int R) {
    return kEvalStages * (size_t)nbmax * R * sizeof(float2);
}
constexpr int kMomThreads = 512;
constexpr int kMomRun = 16;  // sample pairs per first-level FP32 sum in k_moments
constexpr int kMomWarps = kMomThreads / 32;

// y1c[k] = fp32(y1[k] e^{i 2 pi nu_c k}) (FP64 math), and y2 into a zero-padded
// array (data at the even offset padf), so k_moments' window copies start
// 16-byte aligned and never leave the allocation.
__global__ void k_center(const double2* __restrict__ y, const float2* __restrict__ y2, int N,
                         const double* __restrict__ nu_c, float2* __restrict__ y1c,
                         float2* __restrict__ y2p, int padf) {
    const double nc = *nu_c;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
        const double ph = nc * (double)k;
        double s, c;
        sincospi(2.0 * (ph - rint(ph)), &s, &c);
        const double2 v = y[k];
        y1c[k] = make_float2((float)(v.x * c - v.y * s), (float)(v.x * s + v.y * c));
        const float2 w = y2[k];
        y2p[padf + k] = w;
    }
}

// Moments of all d-buckets, blocks aligned to ABSOLUTE sample index (block b
// covers y1 samples [bB, (b+1)B); a bucket uses the blocks meeting its
// overlap, masked to it), so buckets with neighbouring d share the same y1
// rows and overlapping y2 windows. Work item = (group of G = 128 consecutive
// TDOA values starting at an even d0, chunk of CB = 4 absolute blocks);
// persistent grid, one 16-warp CTA per SM:
//   stage   per block row: y1c[bB .. +B) and the y2 window [bB+d0 .. +B+G+2)
//           (zero-padded array) by per-row TMA bulk copies; double-buffered
//           with full/empty mbarriers (item k+1 lands while item k is
//           computed; no __syncthreads)
//   compute warp w = (block w / 4, TDOA values d0 + 32 (w % 4) + lane): one
//           block per warp, so the y1 samples are warp-uniform broadcasts
//           (one shared-memory wavefront per LDS.128) and the y2 samples of
//           the 32 lanes are 32 consecutive words (conflict-free); each lane
//           runs its whole block: z = y1c conj(y2) in registers, folded by
//           T_m(-t) = (-1)^m T_m(t) (R/2 FFMA2 per sample), Chebyshev rows
//           broadcast; moments written directly
// Per two folded sample pairs a warp reads 2 (y1) + 8 (y2) + R/2 (table)
// shared-memory wavefronts (8 + 8 + R/2 with the 8-blocks-per-warp mapping of
// r01, where the y1 reads were 4-way redundant across quarter-warps); L2 -> SM
// traffic is (B + (B + G)) samples per block row for G buckets.
template <int B, int R>
struct MomLayout {
    static constexpr int WG = 4;                        // 32-value TDOA groups per item
    static constexpr int CB = kMomWarps / WG;           // blocks per item
    static constexpr int G = 32 * WG;                   // TDOA values per item
    static constexpr int RP = (2 * R + 3) / 4 * 4;      // table row: T_m(t_j), T_m(t_j+1) pairs
    static constexpr int RS1 = B;                       // y1 row (float2): broadcast reads
    static constexpr int W2 = B + G + 2;                // y2 window samples copied
    static constexpr int RS2 = W2;                      // consecutive lanes: consecutive words
    static constexpr size_t table_floats = (size_t)B / 4 * RP;  // one row per two folded pairs
    static constexpr size_t stage_f2 = (size_t)CB * (RS1 + RS2);  // one buffer
    static constexpr size_t smem = ((table_floats * sizeof(float) + 15) & ~(size_t)15) +
                                   2 * stage_f2 * sizeof(float2);
    static_assert(W2 % 2 == 0 && RS1 % 2 == 0, "16-byte rows");
    static_assert(smem <= 227 * 1024 - 64, "k_moments stage exceeds shared memory");
};

__device__ __forceinline__ float2 cmulc(float4 a, float4 b, int hi) {  // a * conj(b), one sample
    const float ax = hi ? a.z : a.x, ay = hi ? a.w : a.y;
    const float bx = hi ? b.z : b.x, by = hi ? b.w : b.y;
    return make_float2(fmaf(ax, bx, ay * by), fmaf(ay, bx, -(ax * by)));
}

template <int B, int R>
__global__ void __launch_bounds__(kMomThreads, 1)
k_moments(const Bucket* __restrict__ buckets, const int* __restrict__ ubin, int bin0,
          int nbins, int bin_lo, int ngroups, int cpb, const float* __restrict__ tcheb,
          const float2* __restrict__ y1c, const float2* __restrict__ y2p, int padf, int N,
          float2* __restrict__ mom, int nbmax) {
    static_assert(B % 64 == 0 && B <= 768, "block length");
    static_assert(R % 2 == 0 && R <= kMaxMoments, "moment count");
    static_assert(kMomThreads % 32 == 0, "mapping");
    using L = MomLayout<B, R>;
    constexpr int CB = L::CB, WG = L::WG, G = L::G;
    constexpr int RP = L::RP, RS1 = L::RS1, RS2 = L::RS2, W2 = L::W2;
    extern __shared__ float4 smem4[];
    float* ts = reinterpret_cast<float*>(smem4);  // [B/2][RP]
    float2* stage = reinterpret_cast<float2*>(reinterpret_cast<char*>(smem4) +
                                              ((L::table_floats * sizeof(float) + 15) & ~15));
    __shared__ uint64_t full[2], empty[2];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int blk = warp / WG;              // block row of the item (warp-uniform)
    const int t = 32 * (warp % WG) + lane;  // TDOA slot in the group
    const int nitems = ngroups * cpb;
    const int nblk_abs = (N + B - 1) / B;

    auto issue = [&](int it, int buf) {  // warp 0: TMA rows of item `it` into `buf`
        const int g = it / cpb, c = it - g * cpb;
        const int d0 = bin_lo + g * G - (N - 1);
        const int nrow = max(0, min(CB, nblk_abs - c * CB));
        float2* st = stage + (size_t)buf * L::stage_f2;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (lane == 0) mbar_expect_tx(&full[buf], (uint32_t)(nrow * (B + W2) * sizeof(float2)));
        __syncwarp();
        for (int i = lane; i < 2 * nrow; i += 32) {
            const int r = i >> 1;
            const int k0 = (c * CB + r) * B;
            if ((i & 1) == 0)
                tma_load_1d(st + r * RS1, y1c + k0, B * sizeof(float2), &full[buf]);
            else
                tma_load_1d(st + CB * RS1 + r * RS2, y2p + padf + k0 + d0,
                            W2 * sizeof(float2), &full[buf]);
        }
    };

    for (int i = tid; i < B / 4 * RP; i += kMomThreads) {  // row r: pairs 2r, 2r + 1
        const int r = i / RP, q = i % RP;
        ts[i] = q < 2 * R ? tcheb[(2 * r + (q & 1)) * kMaxMoments + (q >> 1)] : 0.f;
    }
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        mbar_init(&empty[0], kMomWarps);
        mbar_init(&empty[1], kMomWarps);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int item = blockIdx.x;
    if (warp == 0 && item < nitems) issue(item, 0);
    for (int k = 0; item < nitems; ++k, item += gridDim.x) {
        const int buf = k & 1;
        const int nitem = item + gridDim.x;
        if (warp == 0 && nitem < nitems) {
            if (k >= 1) mbar_wait(&empty[buf ^ 1], ((k - 1) >> 1) & 1);  // item k-1 done
            issue(nitem, buf ^ 1);
        }
        const int g = item / cpb, c = item - g * cpb;
        const int bin = bin_lo + g * G + t;
        const int u = (bin >= bin0 && bin < bin0 + nbins) ? ubin[bin - bin0] : -1;
        const int d = bin - (N - 1);
        const int kb = d < 0 ? -d : 0, ke = d > 0 ? N - d : N;
        const int bf = kb / B, bl = (ke - 1) / B;      // the bucket's absolute block range
        const int babs = c * CB + blk;
        const bool active = u >= 0 && babs >= bf && babs <= bl;
        const int lo = kb - babs * B, hi = ke - babs * B;  // valid j in [lo, hi)
        // warps whose blocks all lie inside their buckets' overlaps skip the
        // per-sample masks (all but the first / last block of each bucket)
        const bool interior = __all_sync(0xffffffffu, !active || (lo <= 0 && hi >= B));
        mbar_wait(&full[buf], (k >> 1) & 1);
        if (active) {
            const float2* st = stage + (size_t)buf * L::stage_f2;
            const float2* r1 = st + blk * RS1;
            // y2 samples [bB + d ..) start at offset t of the window row
            const float2* r2 = st + CB * RS1 + blk * RS2 + t;
            // two-level accumulation: sums of 16 pairs, then their sum, so the
            // FP32 rounding of coherent partial sums stays ~16x below one
            // sequential 256-pair run
            float2 acc[R];
#pragma unroll
            for (int m = 0; m < R; ++m) acc[m] = make_float2(0.f, 0.f);
            // the block loop, compiled twice: warps whose blocks lie inside their
            // buckets' overlaps run it without the per-sample masks
            auto run = [&](auto masked) {
                constexpr bool kMasked = decltype(masked)::value;
                for (int j0 = 0; j0 < B / 2; j0 += kMomRun) {
                    float2 part[R];
#pragma unroll
                    for (int m = 0; m < R; ++m) part[m] = make_float2(0.f, 0.f);
#pragma unroll
                    for (int j = j0; j < j0 + kMomRun; j += 2) {  // samples j, j+1 (front), B-2-j, B-1-j (back)
                        const float4 f1 = *reinterpret_cast<const float4*>(r1 + j);
                        const float4 g1 = *reinterpret_cast<const float4*>(r1 + B - 2 - j);
                        const float2 fa = r2[j], fb = r2[j + 1], ga = r2[B - 2 - j], gb = r2[B - 1 - j];
                        const float4 f2 = make_float4(fa.x, fa.y, fb.x, fb.y);
                        const float4 g2 = make_float4(ga.x, ga.y, gb.x, gb.y);
                        float2 z0 = cmulc(f1, f2, 0), z1 = cmulc(f1, f2, 1);
                        float2 w1 = cmulc(g1, g2, 0), w0 = cmulc(g1, g2, 1);
                        if constexpr (kMasked) {
                            const float2 zero = make_float2(0.f, 0.f);
                            if (!(j >= lo && j < hi)) z0 = zero;
                            if (!(j + 1 >= lo && j + 1 < hi)) z1 = zero;
                            if (!(B - 2 - j >= lo && B - 2 - j < hi)) w1 = zero;
                            if (!(B - 1 - j >= lo && B - 1 - j < hi)) w0 = zero;
                        }
                        // pair j: (z0, w0); pair j+1: (z1, w1)
                        const float2 u0 = add2(z0, w0), v0 = sub2(z0, w0);
                        const float2 u1 = add2(z1, w1), v1 = sub2(z1, w1);
                        // (T_m(t_j), T_m(t_j+1)) for m = 2qq, 2qq + 1 in one LDS.128
                        const float4* tr = reinterpret_cast<const float4*>(ts + (j >> 1) * RP);
#pragma unroll
                        for (int qq = 0; qq < R / 2; ++qq) {
                            const float4 t = tr[qq];
                            part[2 * qq] = ffma2(u1, t.y, ffma2(u0, t.x, part[2 * qq]));
                            part[2 * qq + 1] = ffma2(v1, t.w, ffma2(v0, t.z, part[2 * qq + 1]));
                        }
                    }
#pragma unroll
                    for (int m = 0; m < R; ++m) {
                        acc[m].x += part[m].x;
                        acc[m].y += part[m].y;
                    }
                }
            };
            if (interior)
                run(std::false_type{});
            else
                run(std::true_type{});
            // odd moments are stored times i, so a candidate's block value is one
            // real-weighted sum  C_b = sum_m c_m M'_m  (k_evaluate)
            const int rb = babs - bf;
            float2* dst = mom + ((size_t)u * nbmax + rb) * R;
#pragma unroll
            for (int m = 0; m < R; ++m)
                dst[m] = (m & 1) ? make_float2(-acc[m].y, acc[m].x) : acc[m];
            if (babs == bl) {  // zero rows up to a multiple of kEvalG (k_evaluate's groups)
                const int nb = bl - bf + 1;
                for (int z = nb * R; z < pad_blocks(nb) * R; ++z)
                    mom[(size_t)u * nbmax * R + z] = make_float2(0.f, 0.f);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[buf]);
    }
}

constexpr int kEvalWarps = 4;
constexpr int kEvalNC = 2;                              // candidates per lane
constexpr int kEvalPass = 32 * kEvalWarps * kEvalNC;   // candidates per CTA pass

// One CTA per d-bucket from a dynamic queue; the bucket's moments are staged
// in shared memory by one TMA bulk copy into a double buffer run as a
// producer/consumer pipeline (full/empty mbarriers): thread 0 claims and
// prefetches bucket k+1 while the warps evaluate bucket k, and each warp
// releases a buffer on its own, so no warp waits for the others at a bucket
// boundary. Each lane evaluates kEvalNC candidates:
//   C_b = sum_m c_m M'_m[b]                       (R FFMA2, broadcast LDS.128)
//   group g of G blocks:  A += Re(W_j) C_b, V += Im(W_j) C_b, e += C_b o C_b
//   acc += a_g (A + iV),  a_{g+1} = a_g e^{i 2 pi nu B G}   (FP64 recurrence)
// W_j = e^{i 2 pi nu B j} (j < G) are rounded once from FP64 phases.
template <int R, int G>
__global__ void __launch_bounds__(32 * kEvalWarps, 4)
k_evaluate(const Bucket* __restrict__ buckets, const int* __restrict__ n_buckets,
           int* __restrict__ queue, const int* __restrict__ sorted,
           const double* __restrict__ fdoa, double fs, const double* __restrict__ nu_c_p, int B,
           const float2* __restrict__ mom, int nbmax, double* __restrict__ s_out,
           uint32_t* __restrict__ flag_bits, int64_t flag_base, float tau, float tau_noise,
           const double* __restrict__ e1, const double* __restrict__ e2, int N) {
    extern __shared__ float4 smem4[];
    __shared__ uint64_t full[kEvalStages], empty[kEvalStages];
    __shared__ int slot_u[kEvalStages];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nbk = *n_buckets;
    const double nu_c = *nu_c_p;
    const size_t buf_f4 = (size_t)nbmax * R / 2;

    // thread 0 only: claim bucket k into its ring slot. The slot is free once
    // every warp released item k - kEvalStages; `block` = wait for that,
    // otherwise give up (returns false) so the producer never idles a warp.
    auto produce = [&](int k, bool block) -> bool {
        const int sl = k % kEvalStages;
        if (k >= kEvalStages) {
            const uint32_t par = ((k / kEvalStages) - 1) & 1;
            if (block)
                mbar_wait(&empty[sl], par);
            else if (!mbar_test(&empty[sl], par))
                return false;
        }
        const int u = atomicAdd(queue, 1);
        slot_u[sl] = u;
        if (u < nbk) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const uint32_t bytes = (uint32_t)pad_blocks(buckets[u].nb) * R * sizeof(float2);
            mbar_expect_tx(&full[sl], bytes);
            tma_load_1d(smem4 + sl * buf_f4, mom + (size_t)u * nbmax * R, bytes, &full[sl]);
        } else {
            mbar_arrive(&full[sl]);  // end of queue: complete the phase with no data
        }
        return true;
    };
    if (tid == 0) {
        for (int i = 0; i < kEvalStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kEvalWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int produced = 0;  // thread 0: buckets claimed so far
    if (tid == 0)
        for (; produced < kEvalStages; ++produced) produce(produced, false);

    for (int k = 0;; ++k) {
        // the ring runs up to kEvalStages buckets ahead; thread 0 blocks only
        // if bucket k itself is not claimed yet
        if (tid == 0) {
            for (; produced <= k; ++produced) produce(produced, true);
            while (produced < k + kEvalStages && produce(produced, false)) ++produced;
        }
        const int sl = k % kEvalStages;
        mbar_wait(&full[sl], (k / kEvalStages) & 1);
        const int u = slot_u[sl];
        if (u >= nbk) break;
        const Bucket bk = buckets[u];
        const int nb = bk.nb;
        const float4* mb = smem4 + sl * buf_f4;
        // Q_m^2 = sum_b |M_m[b]|^2 of the bucket: the scale of the moments' own
        // FP32 rounding, which every candidate of a coherent bucket inherits
        // through its coefficients a_m; per warp,
        // fixed-order reductions
        float qm2[R];
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const float2* mb2 = reinterpret_cast<const float2*>(mb);
            float q2 = 0.f;
            for (int b = lane; b < nb; b += 32) {
                const float2 v = mb2[b * R + m];
                q2 = fmaf(v.x, v.x, fmaf(v.y, v.y, q2));
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) q2 += __shfl_xor_sync(0xffffffffu, q2, o);
            qm2[m] = q2;
        }
        // ||z||_2^2 of the bucket (the floor of the error scale), per warp
        double zfloor = bucket_z2_part(e1, e2, N, bk.d, B, lane, 32);
#pragma unroll
        for (int o = 16; o; o >>= 1) zfloor += __shfl_xor_sync(0xffffffffu, zfloor, o);
        const RefineBucket rfb =
            refine_bucket(zfloor, bucket_coherence(qm2, R, zfloor), tau, tau_noise);

        for (int base = warp * 32 * kEvalNC; base < bk.count; base += kEvalPass) {
            int p[kEvalNC];
            double nu[kEvalNC];
            float cf[kEvalNC][R];
            float wtr[kEvalNC][G], wti[kEvalNC][G];
            double sr[kEvalNC], si[kEvalNC];  // e^{i 2 pi nu B G}
            double qe2[kEvalNC];               // sum_m a_m^2 Q_m^2
#pragma unroll
            for (int c = 0; c < kEvalNC; ++c) {
                const int slot = base + 32 * c + lane;
                p[c] = slot < bk.count ? sorted[bk.start + slot] : -1;
                nu[c] = p[c] >= 0 ? fma(fdoa[p[c]], 1.0 / fs, -nu_c) : 0.0;
                double jv[R];
                bessel_j<R>(3.141592653589793 * nu[c] * (double)B, jv);
                // a_m M_m = (2 - delta_m0) (-1)^(m/2) J_m M'_m  (M' = i^(m mod 2) M)
                float qa = 0.f, qb = 0.f;
#pragma unroll
                for (int m = 0; m < R; ++m) {
                    cf[c][m] = (float)((m == 0 ? 1.0 : 2.0) * (((m >> 1) & 1) ? -1.0 : 1.0) * jv[m]);
                    if (m & 1)
                        qb = fmaf(cf[c][m] * cf[c][m], qm2[m], qb);
                    else
                        qa = fmaf(cf[c][m] * cf[c][m], qm2[m], qa);
                }
                qe2[c] = (double)qa + (double)qb;
                // W_j = W_1^j by an FP64 recurrence from one FP64 sincospi (error
                // ~1e-15), each rounded once to FP32; e^{i 2 pi nu B G} = W_G
                const double x1 = nu[c] * (double)B;
                double w1r, w1i;
                sincospi(2.0 * (x1 - rint(x1)), &w1i, &w1r);
                double pr = 1.0, pi_ = 0.0;
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    wtr[c][j] = (float)pr;
                    wti[c][j] = (float)pi_;
                    const double nr = fma(pr, w1r, -pi_ * w1i);
                    pi_ = fma(pr, w1i, pi_ * w1r);
                    pr = nr;
                }
                sr[c] = pr;
                si[c] = pi_;
            }
            double acc_re[kEvalNC], acc_im[kEvalNC], en[kEvalNC], ar[kEvalNC], ai[kEvalNC];
#pragma unroll
            for (int c = 0; c < kEvalNC; ++c) {
                acc_re[c] = acc_im[c] = en[c] = ai[c] = 0.0;
                ar[c] = 1.0;
            }
            const int ng = pad_blocks(nb) / G;
            const float4* mg = mb;
            for (int g = 0; g < ng; ++g, mg += G * (R / 2)) {
                float2 A[kEvalNC], V[kEvalNC], E2[kEvalNC];
#pragma unroll
                for (int c = 0; c < kEvalNC; ++c)
                    A[c] = V[c] = E2[c] = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    {
                        float4 mv[R / 2];
#pragma unroll
                        for (int q = 0; q < R / 2; ++q) mv[q] = mg[j * (R / 2) + q];
#pragma unroll
                        for (int c = 0; c < kEvalNC; ++c) {
                            // two chains (odd / even m), smallest terms first
                            float2 Co = make_float2(0.f, 0.f), Ce = make_float2(0.f, 0.f);
#pragma unroll
                            for (int q = R / 2 - 1; q >= 0; --q) {
                                Co = ffma2(make_float2(mv[q].z, mv[q].w), cf[c][2 * q + 1], Co);
                                Ce = ffma2(make_float2(mv[q].x, mv[q].y), cf[c][2 * q], Ce);
                            }
                            const float2 C = add2(Ce, Co);
                            A[c] = ffma2(C, wtr[c][j], A[c]);
                            V[c] = ffma2(C, wti[c][j], V[c]);
                            E2[c] = ffma2v(C, C, E2[c]);
                        }
                    }
                }
#pragma unroll
                for (int c = 0; c < kEvalNC; ++c) {
                    const double hr = (double)(A[c].x - V[c].y), hi = (double)(A[c].y + V[c].x);
                    acc_re[c] = fma(ar[c], hr, fma(-ai[c], hi, acc_re[c]));
                    acc_im[c] = fma(ar[c], hi, fma(ai[c], hr, acc_im[c]));
                    en[c] += (double)(E2[c].x + E2[c].y);
                    const double nr = fma(ar[c], sr[c], -ai[c] * si[c]);
                    ai[c] = fma(ar[c], si[c], ai[c] * sr[c]);
                    ar[c] = nr;
                }
            }
            // FP32 error scale of this candidate: max(sqrt(sum_b |C_b|^2),
            // sqrt(sum_m a_m^2 Q_m^2)); below tau of it the
            // value is re-evaluated in FP64
#pragma unroll
            for (int c = 0; c < kEvalNC; ++c) {
                if (p[c] < 0) continue;
                const double s2 = acc_re[c] * acc_re[c] + acc_im[c] * acc_im[c];
                s_out[p[c]] = sqrt(s2);
                if (refine_moment(s2, en[c], qe2[c], rfb)) {
                    const int64_t e = flag_base + p[c];
                    atomicOr(&flag_bits[e >> 5], 1u << (e & 31));
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[sl]);
    }
}

// algorithmic work of one step in FP32x2 operations (the numerators of bench.py's
// rooflines): moments per bucket-block B/2 (R + 6): R moment MACs per folded
// sample pair, two complex products (2 each) and the fold (2); candidates
// count*nb*(R+3) on the block loop, count*nb*3 plus the MMA FLOPs (work[2]) on
// the tensor-core path (six BF16 MMAs of 128 x np x 16 per 128-candidate tile)
__global__ void k_work_count(const Bucket* __restrict__ buckets, const int* __restrict__ n_buckets,
                             int B, int R, int tc, unsigned long long* __restrict__ work) {
    unsigned long long a = 0, b = 0, c = 0;
    for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < *n_buckets;
         u += gridDim.x * blockDim.x) {
        const Bucket bk = buckets[u];
        a += (unsigned long long)bk.nb * (B / 2) * (R + 6);
        if (tc) {
            b += (unsigned long long)bk.count * bk.nb * 3;
            const unsigned long long tiles = (bk.count + 127) / 128;
            const unsigned long long np = 32ull * ((bk.nb + 15) / 16);
            c += tiles * 6ull * 2ull * 128ull * np * 16ull;
        } else {
            b += (unsigned long long)bk.count * bk.nb * (R + 3);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if ((threadIdx.x & 31) == 0 && (a || b || c)) {
        atomicAdd(&work[0], a);
        atomicAdd(&work[1], b);
        atomicAdd(&work[2], c);
    }
}

struct MomArgs {
    const Bucket* buckets;
    const int* ubin;
    int bin0, nbins, bin_lo, ngroups, cpb;
    const float* tcheb;
    const float2 *y1c, *y2p;
    int padf, N;
    float2* mom;
    int nbmax;
};

template <int B, int R>
void moments_variant(MomArgs a, int sm_count, cudaStream_t st) {
    using L = MomLayout<B, R>;
    // groups of G TDOA values starting at an even d (16-byte aligned y2 windows)
    a.bin_lo = ((a.bin0 - (a.N - 1)) & 1) ? a.bin0 - 1 : a.bin0;
    a.ngroups = (a.bin0 + a.nbins - a.bin_lo + L::G - 1) / L::G;
    a.cpb = ((a.N + B - 1) / B + L::CB - 1) / L::CB;
    auto kern = k_moments<B, R>;
    const size_t smem = MomLayout<B, R>::smem;
    static size_t attr[64] = {};
    ensure_smem(kern, smem, attr);
    const int items = a.ngroups * a.cpb;
    const int grid = items < sm_count ? (items > 0 ? items : 1) : sm_count;
    kern<<<grid, kMomThreads, smem, st>>>(a.buckets, a.ubin, a.bin0, a.nbins, a.bin_lo, a.ngroups,
                                          a.cpb, a.tcheb, a.y1c, a.y2p, a.padf, a.N, a.mom,
                                          a.nbmax);
}

template <int B>
void moments_b(int R, const MomArgs& a, int sm_count, cudaStream_t st) {
    switch (R) {
        case 8: moments_variant<B, 8>(a, sm_count, st); break;
        case 10: moments_variant<B, 10>(a, sm_count, st); break;
        case 12: moments_variant<B, 12>(a, sm_count, st); break;
        case 14: moments_variant<B, 14>(a, sm_count, st); break;
        default: moments_variant<B, 16>(a, sm_count, st); break;
    }
}

template <int R>
void evaluate_variant(const Bucket* buckets, const int* n_buckets, int* queue, int max_buckets,
                      const int* sorted, const double* fdoa, double fs, const double* nu_c, int B,
                      const float2* mom, int nbmax, double* s_out, uint32_t* flag_bits,
                      int64_t flag_base, float tau, float tau_noise, const double* e1,
                      const double* e2, int N, int sm_count, cudaStream_t st) {
    auto kern = k_evaluate<R, kEvalG>;
    const size_t smem = evaluate_smem(nbmax, R);
    static size_t attr[64] = {};
    ensure_smem(kern, smem, attr);
    int grid = sm_count * 4;
    if (grid > max_buckets) grid = max_buckets > 0 ? max_buckets : 1;
    kern<<<grid, 32 * kEvalWarps, smem, st>>>(buckets, n_buckets, queue, sorted, fdoa, fs, nu_c,
                                              B, mom, nbmax, s_out, flag_bits, flag_base, tau,
                                              tau_noise, e1, e2, N);
}

}  // namespace

void launch_center(const double2* y, const float2* y2, int N, const double* nu_c, float2* y1c,
                   float2* y2p, int padf, cudaStream_t st) {
    int blocks = (N + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    k_center<<<blocks, 256, 0, st>>>(y, y2, N, nu_c, y1c, y2p, padf);
}

void launch_work_count(const Bucket* buckets, const int* n_buckets, int B, int R, int tc,
                       unsigned long long* work, cudaStream_t st) {
    k_work_count<<<64, 256, 0, st>>>(buckets, n_buckets, B, R, tc, work);
}


void launch_moments(int B, int R, const Bucket* buckets, const int* ubin, int bin0, int nbins,
                    int N, const float* tcheb, const float2* y1c, const float2* y2p, int padf,
                    float2* mom, int nbmax, int sm_count, cudaStream_t st) {
    MomArgs a;
    a.buckets = buckets;
    a.ubin = ubin;
    a.bin0 = bin0;
    a.nbins = nbins;
    a.tcheb = tcheb;
    a.y1c = y1c;
    a.y2p = y2p;
    a.padf = padf;
    a.N = N;
    a.mom = mom;
    a.nbmax = nbmax;
    switch (B) {
        case 64: moments_b<64>(R, a, sm_count, st); break;
        case 128: moments_b<128>(R, a, sm_count, st); break;
        case 256: moments_b<256>(R, a, sm_count, st); break;
        case 640: moments_b<640>(R, a, sm_count, st); break;
        case 768: moments_b<768>(R, a, sm_count, st); break;
        default: moments_b<512>(R, a, sm_count, st); break;
    }
}

size_t evaluate_smem_bytes(int nbmax, int R) { return evaluate_smem(nbmax, R); }

void launch_evaluate(int R, const Bucket* buckets, const int* n_buckets, int* queue,
                     int max_buckets, const int* sorted, const double* fdoa, double fs,
                     const double* nu_c, int B, const float2* mom, int nbmax, double* s_out,
                     uint32_t* flag_bits, int64_t flag_base, float tau, float tau_noise,
                     const double* e1, const double* e2, int N, int sm_count, cudaStream_t st) {
#define DG_EVAL_CASE(RR)                                                                    \
    evaluate_variant<RR>(buckets, n_buckets, queue, max_buckets, sorted, fdoa, fs, nu_c, B, \
                         mom, nbmax, s_out, flag_bits, flag_base, tau, tau_noise, e1, e2, N,   \
                         sm_count, st)
    switch (R) {
        case 8: DG_EVAL_CASE(8); break;
        case 10: DG_EVAL_CASE(10); break;
        case 12: DG_EVAL_CASE(12); break;
        case 14: DG_EVAL_CASE(14); break;
        default: DG_EVAL_CASE(16); break;
    }
#undef DG_EVAL_CASE
}

}  // namespace dg
