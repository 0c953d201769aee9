// C ABI of the B200 direct-geolocation engine (include/b200geo.h).
//
// Host orchestration only: validation mirrors the reference's exceptions
// (messages kept verbatim where the reference has them), every numeric step
// runs in the kernels of dg_kernels.cu. Reference paths are relative to
// /root/reference/proj/include/digeo.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <new>
#include <numbers>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "b200geo.h"
#include "dg_host.hpp"
#include "dg_internal.cuh"

using namespace dg;

std::string& dg::last_error() {
    thread_local std::string s;
    return s;
}

namespace {

// geodesy.hpp:31-38
constexpr double kA = 6378137.0;
constexpr double kF = 1.0 / 298.257223563;
constexpr double kE2 = kF * (2.0 - kF);
constexpr double kC = 299792458.0;
inline double deg2rad(double d) { return d * std::numbers::pi / 180.0; }

std::string fmt_double(double v) { return std::to_string(v); }

// GeodeticCoord::validate (geodesy.hpp:69-78)
void validate_geodetic(double lat, double lon, double alt) {
    if (!(lat >= -90.0 && lat <= 90.0))
        raise(DG_EINVAL, "GeodeticCoord: lat_deg out of [-90, 90]: " + fmt_double(lat));
    if (!(lon >= -180.0 && lon < 180.0))
        raise(DG_EINVAL, "GeodeticCoord: lon_deg out of [-180, 180): " + fmt_double(lon));
    if (!std::isfinite(alt)) raise(DG_EINVAL, "GeodeticCoord: alt_m not finite");
}

}  // namespace

struct dg_session {
    dg_engine* eng = nullptr;
    int64_t N = 0, stride = 0;
    double fs = 0;
    std::unique_ptr<DevMem> y32;  // float2 [2][stride]
    std::unique_ptr<DevMem> y64;  // double2 [2][stride]
    std::unique_ptr<DevMem> e64;  // double [2][N+1]: prefix sums of |y|^2
    cudaStream_t st = nullptr;
    ~dg_session() {
        if (st) cudaStreamDestroy(st);
    }
};


namespace {


// ---------------------------------------------------------------------------
// Correlator planning. A (snapshot, pair) "step" runs either the block-moment
// correlator (dg_moments.cu) with block length B and R moments, or the direct
// FFMA2 correlator (dg_correlate.cu) when no (B, R) meets the truncation bound
// (very wide FDOA ranges) or when the direct form is cheaper (few candidates
// per TDOA bucket). See DESIGN.md section 4.
// One work unit of a run: the (snapshot, pair) step sp over the whole grid, or
// part `part` of `parts` of it (the candidates of a contiguous range of its
// TDOA buckets, cost-balanced on the step's histogram; the other candidates
// are left 0 so the parts of a step sum to the whole step exactly).
struct StepUnit {
    int sp = 0, part = 0, parts = 1;
};

struct StepPlan {
    bool empty = true;    // no candidate overlaps: every S is 0 (already written)
    bool direct = false;
    int B = 0, R = 0, nbmax = 0, cpb = 0;
    int bin0 = 0, nbins = 0;
    double nu_c = 0.0;
};

// |e^{ixt} - sum_{m<R} a_m T_m(t)| <= 2 (x/2)^R / R! / (1 - (x/2)^2/(R+1)), |t| <= 1
double jacobi_anger_tail(double x, int R) {
    const double h = std::fabs(x) * 0.5;
    double t = 2.0;
    for (int m = 1; m <= R; ++m) t *= h / m;
    const double q = h * h / (R + 1);
    return q < 1.0 ? t / (1.0 - q) : INFINITY;
}

// Truncation budget. Per block the Jacobi-Anger remainder is bounded by
// tail(x, R) times the block's L1 norm, and a product stream that repeats with
// the block length (e.g. a chirp product tone aliasing onto B) can add those
// remainders coherently, so a candidate's truncation error is only bounded by
// tail * ||z||_1 <= tail * sqrt(N) ||z||_2, while unrefined values are at least
// tau ||z||_2 (the refinement test's floor). tail <= kTailBudget tau / sqrt(N)
// keeps that term below 1e-5 relative, half the 2e-5 margin the error model
// holds (tests/test_gpu_error_model.py): 9e-10 at N = 50,000 (C3: B = 512 with
// R = 14, or B = 640 with R = 16; the planner's cost model picks).
constexpr double kTailBudget = 1e-5;
// Largest Jacobi-Anger argument x = pi h B the planner admits. Past it the
// coefficients a_m(x) grow and the block sums cancel more, so the FP32
// evaluation error of sidelobe candidates in coherent buckets rises faster
// than the refinement test tracks (measured on +40 dB tone / chirp scenes:
// B = 768 at x = 3.5 reached 1.4e-4, B = 640 at x = 2.9 stayed at 3e-5;
// tests/test_gpu_error_model.py).
constexpr double kMomentXMax = 3.0;
constexpr size_t kEvalSmemMax = 200 * 1024;  // k_evaluate stages two buckets of moments
constexpr int kMomentR[] = {8, 10, 12, 14, 16};
constexpr int kMomentB[] = {768, 640, 512, 256, 128, 64};

// `r`: the exact range of the candidates being correlated (bins, emptiness).
// `a` (nullable): the FP32 planning range of the whole lattice with its FDOA
// margin; when given, B / R / nu_c depend only on it, so every slab of a
// lattice computes every cell bit-identically.
StepPlan plan_step(const StepRange& r, const StepRange* a, double a_margin_hz, int64_t P_plan,
                   int N, double fs, const dg_tuning& tn) {
    StepPlan pl;
    if (r.dmin > r.dmax) return pl;
    pl.empty = false;
    pl.bin0 = r.dmin + N - 1;
    pl.nbins = r.dmax - r.dmin + 1;
    double nu_lo = f64_from_key(r.fmin) / fs, nu_hi = f64_from_key(r.fmax) / fs;
    double d_span = pl.nbins;
    if (a && a->dmin <= a->dmax) {
        const double alo = (f64_from_key(a->fmin) - a_margin_hz) / fs;
        const double ahi = (f64_from_key(a->fmax) + a_margin_hz) / fs;
        // the exact range lies inside the planning range unless FP32 erred
        // beyond its margin; then widen (correct, no longer partition-proof)
        nu_lo = std::min(nu_lo, alo);
        nu_hi = std::max(nu_hi, ahi);
        d_span = std::max(1, std::min(a->dmax, N - 1) - std::max(a->dmin, 1 - N) + 1);
    }
    pl.nu_c = 0.5 * (nu_lo + nu_hi);
    const double half = 0.5 * (nu_hi - nu_lo) * (1.0 + 1e-9) + 1e-15;
    const double avg = (double)P_plan / d_span;  // candidates per TDOA bucket (approx.)
    const double tail_max = kTailBudget * kMomentRefineTau / std::sqrt((double)N);
    // costs in FP32x2-MAC units per bucket: direct ~2.3 per candidate-sample;
    // moments R per sample (x1.5 for smem traffic) + (R + 5) per candidate-block
    double best = 2.3 * avg * N;
    const int forceB = tn.moment_block, forceR = tn.moment_count;
    pl.direct = true;
    if (tn.correlator == DG_CORRELATOR_DIRECT) return pl;
    if (tn.correlator == DG_CORRELATOR_MOMENTS) best = INFINITY;
    for (int B : kMomentB) {
        if (forceB && B != forceB) continue;
        const double x = M_PI * half * B;
        if (x > kMomentXMax) continue;
        for (int R : kMomentR) {
            if (forceR && R != forceR) continue;
            // a forced R is used only where it meets the truncation bound too
            if (jacobi_anger_tail(x, R) > tail_max) continue;
            if (evaluate_smem_bytes(((N + B - 1) / B + kEvalG - 1) / kEvalG * kEvalG, R) >
                kEvalSmemMax)
                break;
            const double cost = 1.5 * R * N + avg * ((double)N / B) * (R + 3);
            if (cost < best) {
                best = cost;
                pl.direct = false;
                pl.B = B;
                pl.R = R;
            }
            break;  // smallest admissible R for this B
        }
    }
    if (!pl.direct) {
        pl.nbmax = ((N + pl.B - 1) / pl.B + kEvalG - 1) / kEvalG * kEvalG;
    }
    return pl;
}

// Chebyshev tables T_m(t_j), t_j = (2j - (B-1))/B, for every supported B:
// [B][kMaxMoments] floats each, FP64 recurrence then one rounding.
std::vector<float> chebyshev_table(int B) {
    std::vector<float> t((size_t)B * kMaxMoments);
    for (int j = 0; j < B; ++j) {
        const double x = (2.0 * j - (B - 1)) / B;
        double tm1 = 1.0, tm = x;
        t[(size_t)j * kMaxMoments] = 1.0f;
        t[(size_t)j * kMaxMoments + 1] = (float)x;
        for (int m = 2; m < kMaxMoments; ++m) {
            const double tn = 2.0 * x * tm - tm1;
            tm1 = tm;
            tm = tn;
            t[(size_t)j * kMaxMoments + m] = (float)tn;
        }
    }
    return t;
}

// ---------------------------------------------------------------------------
// The per-(snapshot, pair) pipeline shared by correlate_batch, correlate_snapshot
// and the full driver. Phase A (geometry) runs for a window of steps into
// per-slot d/fdoa/histogram/range buffers; one synchronisation reads the
// ranges and plans every step; phase B buckets and correlates each step.
std::vector<RxPairF32> rx_pairs_f32(const dg_grid* g, const PairGeom* pg, int n);
double fp32_fdoa_margin(const PairGeom* pg, int n, double wl);

// Per-step working set of the bucket/moments/evaluate stages. Two lanes on two
// streams let step i+1's latency-bound bucketing (scan, scatter, task build)
// and moments overlap step i's evaluation.
struct Lane {
    cudaStream_t st = nullptr;
    bool own_stream = false;
    int *sorted = nullptr, *off = nullptr, *toff = nullptr, *boff = nullptr, *cursor = nullptr,
        *n_tasks = nullptr, *n_buckets = nullptr, *queue = nullptr, *ubin = nullptr;
    Task* tasks = nullptr;
    Bucket* buckets = nullptr;
    float2 *y1c = nullptr, *y2p = nullptr;
    float2* af = nullptr;  // FFT path: per (block, moment) spectra of the y1 blocks
    float* fe = nullptr;   // FFT path: per (window, block, moment) correlation mean squares
    int* fqueue = nullptr;  // FFT path: work queue + per-block spectrum counters
    float* qf = nullptr;   // FFT path: their sums over each bucket's blocks [bucket][16]
    float2* mom = nullptr;
    size_t mom_cap = 0;
    unsigned long long* work = nullptr;  // [2]: moment / evaluate FP32x2 MACs
    cudaEvent_t done = nullptr;
    ~Lane() {
        if (done) cudaEventDestroy(done);
        if (own_stream && st) cudaStreamDestroy(st);
    }
};

struct Pipeline {
    int64_t P = 0;
    int N = 0, nbins = 0, max_tasks = 0, slots = 0, sm_count = 148, n_lanes = 1;
    int *d = nullptr, *rank = nullptr, *hist = nullptr, *err = nullptr;
    double* fdoa = nullptr;
    StepRange* range = nullptr;
    double* nu_c = nullptr;  // [slots]
    int padf = 0;            // zero padding in front of each lane's y2p
    Lane lanes[2];
    cudaEvent_t window_ready = nullptr;
    unsigned long long* overlap = nullptr;
    static constexpr int kTables = 6;  // the block lengths of kMomentB
    const float* tcheb[kTables] = {};   // [B][kMaxMoments] (k_moments)
    const float* tchebT[kTables] = {};  // [kMaxMoments][B] (k_mfft: coalesced per moment)
    const float* tcheb_for(int B, bool transposed = false) const {
        for (int i = 0; i < kTables; ++i)
            if (kMomentB[i] == B) return transposed ? tchebT[i] : tcheb[i];
        raise(DG_ERUNTIME, "b200: no Chebyshev table for this block length");
    }
    std::vector<StepPlan> plans;
    int64_t launches = 0, direct_steps = 0;
    // the engine's tuning (dg_engine_set_tuning), copied once per call:
    // refinement threshold of the block-moment path (error-model studies use a
    // huge value to re-evaluate every element exactly) and whether the
    // candidate block sums run on the tensor cores (dg_evaluate_tc.cu) or the
    // FFMA2 block loop (k_evaluate)
    dg_tuning tn{};
    float tau = kMomentRefineTau, tau_direct = kRefineTau, tau_noise = kNoiseRefineTau;
    bool use_tc = true;
    bool use_fft = false;  // block moments as FFT cross-correlations (tuning moment_fft)
    float fft_kappa = kFftRefineKappa;
    int64_t fft_steps = 0;
    double fft_flop = 0.0;  // FFT moments: 5 L log2 L per FFT + 6 L per spectrum product

    ~Pipeline() {
        if (window_ready) cudaEventDestroy(window_ready);
    }

    // lanes: 2 overlap consecutive steps; 1 serialises them (profiled runs, so
    // each kernel's CUDA-event time is its own)
    void init(Scratch& sc, dg_engine* eng, int64_t P_, int64_t N_, int n_steps, int max_lanes = 2,
              cudaStream_t lane1 = nullptr) {
        const int sms = eng->sm_count;
        {
            std::lock_guard<std::mutex> lk(eng->tables_mu);
            tn = eng->tuning;
        }
        tau = tn.refine_tau > 0.0 ? (float)tn.refine_tau : kMomentRefineTau;
        tau_direct = tn.direct_refine_tau > 0.0 ? (float)tn.direct_refine_tau : kRefineTau;
        tau_noise = tn.noise_refine_tau > 0.0 ? (float)tn.noise_refine_tau : kNoiseRefineTau;
        use_tc = tn.evaluate_tensor != 0;
        use_fft = tn.moment_fft != 0;
        fft_kappa = tn.fft_refine_kappa > 0.0 ? (float)tn.fft_refine_kappa : kFftRefineKappa;
        if (P_ > INT32_MAX) raise(DG_EINVAL, "b200: more than 2^31-1 candidates in one call");
        if (N_ > INT32_MAX / 2) raise(DG_EINVAL, "b200: capture longer than 2^30 samples");
        P = P_;
        N = (int)N_;
        sm_count = sms;
        nbins = 2 * N - 1;
        const int64_t mt = P / correlate_task_size() + std::min<int64_t>(P, nbins) + 1;
        max_tasks = (int)std::min<int64_t>(mt, INT32_MAX);
        // phase-A window: per-slot d + fdoa + histogram, within ~4 GB
        const int64_t per_slot = 16 * P + 4 * (int64_t)nbins + 64;
        slots = (int)std::max<int64_t>(1, std::min<int64_t>(n_steps, (4ll << 30) / per_slot));
        d = sc.alloc<int>((size_t)P * slots);
        rank = sc.alloc<int>((size_t)P * slots);
        fdoa = sc.alloc<double>((size_t)P * slots);
        hist = sc.alloc<int>((size_t)nbins * slots);
        range = sc.alloc<StepRange>(slots);
        nu_c = sc.alloc<double>(slots);
        err = sc.alloc<int>(1);
        overlap = sc.alloc<unsigned long long>(1);
        CK(cudaMemsetAsync(hist, 0, sizeof(int) * nbins * slots, sc.st));
        CK(cudaMemsetAsync(err, 0, sizeof(int), sc.st));
        CK(cudaMemsetAsync(overlap, 0, sizeof(unsigned long long), sc.st));
        n_lanes = n_steps > 1 ? std::max(1, std::min(2, max_lanes)) : 1;
        lane1_ = lane1;
        eng_ = eng;
    }

    // the correlation lanes' working sets (after the first geometry launch, so
    // the geometry pass does not wait for this host work)
    cudaStream_t lane1_ = nullptr;
    dg_engine* eng_ = nullptr;
    void init_lanes(Scratch& sc) {
        dg_engine* eng = eng_;
        cudaStream_t lane1 = lane1_;
        // centred y1 (k_moments' row copies may run one block past N) and y2 in a
        // zero-padded array: its window copies reach from N samples before to
        // N + 1200 samples after the data
        padf = (N + 65) & ~1;  // even: window copies start 16-byte aligned
        const size_t ylen = (size_t)padf + 2 * (size_t)N + 1280;
        for (int l = 0; l < n_lanes; ++l) {
            Lane& L = lanes[l];
            if (l == 0) {
                L.st = sc.st;
            } else if (lane1) {
                L.st = lane1;
            } else {
                CK(cudaStreamCreateWithFlags(&L.st, cudaStreamNonBlocking));
                L.own_stream = true;
            }
            CK(cudaEventCreateWithFlags(&L.done, cudaEventDisableTiming));
            L.sorted = sc.alloc<int>(P);
            L.tasks = sc.alloc<Task>(max_tasks);
            L.buckets = sc.alloc<Bucket>(std::min<int64_t>(P, nbins));
            L.off = sc.alloc<int>(nbins);
            L.toff = sc.alloc<int>(nbins);
            L.boff = sc.alloc<int>(nbins);
            L.cursor = sc.alloc<int>(nbins);
            L.ubin = sc.alloc<int>(nbins);
            L.n_tasks = sc.alloc<int>(1);
            L.n_buckets = sc.alloc<int>(1);
            L.queue = sc.alloc<int>(1);
            L.work = sc.alloc<unsigned long long>(3);
            L.y1c = sc.alloc<float2>(N + 768 + 64);  // + one block (B <= 768)
            L.y2p = sc.alloc<float2>(ylen);
            CK(cudaMemsetAsync(L.y2p, 0, ylen * sizeof(float2), sc.st));
            CK(cudaMemsetAsync(L.work, 0, 3 * sizeof(unsigned long long), sc.st));
            if (use_fft) {  // the largest block count the FFT path takes (B = 256)
                L.af = sc.alloc<float2>(moments_fft_af_bytes(N, 256, kMaxMoments) /
                                        sizeof(float2));
                L.fe = sc.alloc<float>(moments_fft_fe_floats(N, 256, kMaxMoments));
                L.fqueue = sc.alloc<int>((size_t)N / 256 + 2);
                L.qf = sc.alloc<float>((size_t)std::min<int64_t>(P, nbins) * kMaxMoments);
            }
        }
        CK(cudaEventCreateWithFlags(&window_ready, cudaEventDisableTiming));
        static_assert(sizeof(kMomentB) / sizeof(kMomentB[0]) == kTables, "tables");
        size_t off[kTables], total = 0;
        for (int i = 0; i < kTables; ++i) {
            off[i] = total;
            total += (size_t)kMomentB[i] * kMaxMoments;
        }
        const size_t offT = total;  // the transposed copies follow, same offsets
        {
            std::lock_guard<std::mutex> lk(eng->tables_mu);
            if (!eng->tables) {
                std::vector<float> all;
                for (int i = 0; i < kTables; ++i) {
                    auto t = chebyshev_table(kMomentB[i]);
                    all.insert(all.end(), t.begin(), t.end());
                }
                for (int i = 0; i < kTables; ++i) {
                    const int B = kMomentB[i];
                    for (int m = 0; m < kMaxMoments; ++m)
                        for (int j = 0; j < B; ++j)
                            all.push_back(all[off[i] + (size_t)j * kMaxMoments + m]);
                }
                auto mem = std::make_unique<DevMem>(all.size() * sizeof(float));
                CK(cudaMemcpy(mem->p, all.data(), all.size() * sizeof(float),
                              cudaMemcpyHostToDevice));
                eng->tables = std::move(mem);
            }
        }
        for (int i = 0; i < kTables; ++i) {
            tcheb[i] = static_cast<const float*>(eng->tables->p) + off[i];
            tchebT[i] = static_cast<const float*>(eng->tables->p) + offT + off[i];
        }
    }

    int* d_slot(int s) const { return d + (size_t)s * P; }
    int* rank_slot(int s) const { return rank + (size_t)s * P; }
    double* fdoa_slot(int s) const { return fdoa + (size_t)s * P; }
    int* hist_slot(int s) const { return hist + (size_t)s * nbins; }

    void reset_ranges(Scratch& sc, int n) {
        std::vector<StepRange> h(n);
        for (auto& r : h) step_range_init(&r);
        CK(cudaMemcpyAsync(range, h.data(), n * sizeof(StepRange), cudaMemcpyHostToDevice, sc.st));
        CK(cudaStreamSynchronize(sc.st));
    }

    // one synchronisation: read the window's ranges (and the lattice planning
    // ranges `approx`, nullable), plan each step, upload nu_c, size the moment
    // buffers; the lanes then wait for `window_ready` (main stream)
    // exact_ranges: `range` holds the exact FDOA and TDOA ranges of each step;
    // otherwise (the windowed geometry pass) only its TDOA range, reduced from
    // the step's histogram (k_hist_range), and the FDOA range is the planning one
    // units (nullable): a unit with parts > 1 keeps only its share of the
    // step's bins, split where the cumulative planner cost of the histogram's
    // buckets crosses part / parts of the total (the same split on every rank:
    // the histograms are bit-exact)
    void plan_window(Scratch& sc, int n, double fs, const StepRange* approx = nullptr,
                     double margin_hz = 0.0, int64_t P_plan = 0, bool exact_ranges = true,
                     const std::vector<StepUnit>* units = nullptr) {
        std::vector<StepRange> h(n), ha(approx ? n : 0);
        if (!exact_ranges && !approx) raise(DG_ERUNTIME, "b200: plan without FDOA range");
        CK(cudaMemcpyAsync(h.data(), range, n * sizeof(StepRange), cudaMemcpyDeviceToHost, sc.st));
        if (approx)
            CK(cudaMemcpyAsync(ha.data(), approx, n * sizeof(StepRange), cudaMemcpyDeviceToHost,
                               sc.st));
        CK(cudaStreamSynchronize(sc.st));
        plans.assign(n, StepPlan{});
        std::vector<double> nc(n);
        size_t need = 0;
        for (int i = 0; i < n; ++i) {
            if (!exact_ranges) {  // exact bins, planning FDOA range
                h[i].fmin = ha[i].fmin;
                h[i].fmax = ha[i].fmax;
            }
            plans[i] = plan_step(h[i], approx ? &ha[i] : nullptr, margin_hz, approx ? P_plan : P, N,
                                 fs, tn);
            if (units && (*units)[i].parts > 1 && !plans[i].empty)
                split_bins(sc, i, (*units)[i].part, (*units)[i].parts, plans[i]);
            nc[i] = plans[i].nu_c;
            const StepPlan& pl = plans[i];
            if (!pl.empty && !pl.direct)
                need = std::max(need, (size_t)std::min<int64_t>(P, pl.nbins) * pl.nbmax * pl.R);
        }
        for (int l = 0; l < n_lanes; ++l)
            if (need > lanes[l].mom_cap) {
                lanes[l].mom = sc.alloc<float2>(need);
                lanes[l].mom_cap = need;
            }
        CK(cudaMemcpyAsync(nu_c, nc.data(), n * sizeof(double), cudaMemcpyHostToDevice, sc.st));
        CK(cudaStreamSynchronize(sc.st));
        CK(cudaEventRecord(window_ready, sc.st));
        for (int l = 1; l < n_lanes; ++l) CK(cudaStreamWaitEvent(lanes[l].st, window_ready, 0));
    }

    void split_bins(Scratch& sc, int slot, int part, int parts, StepPlan& pl) const {
        std::vector<int> h(pl.nbins);
        CK(cudaMemcpyAsync(h.data(), hist_slot(slot) + pl.bin0, pl.nbins * sizeof(int),
                           cudaMemcpyDeviceToHost, sc.st));
        CK(cudaStreamSynchronize(sc.st));
        // planner cost of each non-empty bin (plan_step's model)
        std::vector<double> cum(pl.nbins + 1, 0.0);
        for (int b = 0; b < pl.nbins; ++b) {
            double c = 0.0;
            if (h[b] > 0)
                c = pl.direct ? 2.3 * h[b] * (double)N
                              : 1.5 * pl.R * (double)N + h[b] * ((double)N / pl.B) * (pl.R + 3);
            cum[b + 1] = cum[b] + c;
        }
        const double total = cum[pl.nbins];
        auto cut = [&](int k) {  // first bin whose cumulative cost reaches k / parts
            if (k <= 0) return 0;
            if (k >= parts) return pl.nbins;
            const double t = total * k / parts;
            return (int)(std::lower_bound(cum.begin() + 1, cum.end(), t) - cum.begin());
        };
        const int lo = cut(part), hi = std::max(lo, cut(part + 1));
        pl.bin0 += lo;
        pl.nbins = hi - lo;
        if (pl.nbins <= 0) pl.empty = true;
    }

    void wait_event(cudaEvent_t e) {
        for (int l = 0; l < n_lanes; ++l) CK(cudaStreamWaitEvent(lanes[l].st, e, 0));
    }

    // the main stream waits for every lane (end of a window / of the call)
    void join(Scratch& sc) {
        for (int l = 1; l < n_lanes; ++l) {
            CK(cudaEventRecord(lanes[l].done, lanes[l].st));
            CK(cudaStreamWaitEvent(sc.st, lanes[l].done, 0));
        }
    }

    // FP32 planning ranges over the full lattice of `g` for steps pg[0..n)
    // (run after the geometry pass: beside it, at one CTA per SM, this pass was
    // slower than the two in sequence)
    std::vector<RxPairF32> h_rx;  // members: alive until plan_window synchronises
    std::vector<StepRange> h_init;
    StepRange* lattice_ranges(Scratch& sc, const dg_grid* g, const PairGeom* pg_host,
                              int n, double fs, double wl) {
        h_rx = rx_pairs_f32(g, pg_host, n);
        h_init.assign(n, StepRange{});
        for (auto& r : h_init) step_range_init(&r);
        auto* rx_dev = sc.alloc<RxPairF32>(n);
        auto* out = sc.alloc<StepRange>(n);
        CK(cudaMemcpyAsync(rx_dev, h_rx.data(), n * sizeof(RxPairF32), cudaMemcpyHostToDevice,
                           sc.st));
        CK(cudaMemcpyAsync(out, h_init.data(), n * sizeof(StepRange), cudaMemcpyHostToDevice,
                           sc.st));
        launch_range_fp32(g->rel32(), g->full_size, rx_dev, n, fs, wl, out, sc.st);
        launches += 1;
        return out;
    }

    cudaStream_t lane_stream(int s) const { return lanes[s % n_lanes].st; }

    // phase B for slot s on lane s % n_lanes. y1_64 is the exact capture
    // (centring source).
    // e1 / e2: the captures' |y|^2 prefix sums (launch_energy_prefix)
    void correlate(int s, const double2* y1_64, const float2* y1, const float2* y2,
                   const double* e1, const double* e2, double fs, double* s_out, uint32_t* bits,
                   int64_t flag_base, cudaEvent_t ev0, cudaEvent_t ev1, cudaEvent_t ev2) {
        const StepPlan& pl = plans[s];
        Lane& L = lanes[s % n_lanes];
        cudaStream_t st = L.st;
        if (pl.empty) {
            for (cudaEvent_t e : {ev0, ev1, ev2})
                if (e) CK(cudaEventRecord(e, st));
            return;
        }
        if (pl.direct) {
            launch_bucket(hist_slot(s), pl.bin0, pl.nbins, N, L.off, L.toff, L.boff, L.cursor,
                          L.n_tasks, L.n_buckets, d_slot(s), rank_slot(s), P, L.sorted, L.tasks,
                          L.buckets,
                          L.ubin, 0, st);
            if (ev0) CK(cudaEventRecord(ev0, st));
            if (ev1) CK(cudaEventRecord(ev1, st));
            launch_correlate(L.tasks, L.n_tasks, max_tasks, L.sorted, fdoa_slot(s), y1, y2, N, fs,
                             s_out, bits, flag_base, tau_direct, st);
            launches += 4;
            ++direct_steps;
        } else {
            launch_bucket(hist_slot(s), pl.bin0, pl.nbins, N, L.off, L.toff, L.boff, L.cursor,
                          L.n_tasks, L.n_buckets, d_slot(s), rank_slot(s), P, L.sorted, L.tasks,
                          L.buckets,
                          L.ubin, pl.B, st);
            launch_center(y1_64, y2, N, nu_c + s, L.y1c, L.y2p, padf, st);
            if (ev0) CK(cudaEventRecord(ev0, st));
            const bool tc = use_tc && evaluate_tc_supported(pl.nbmax, pl.R);
            // FFT moments only where the tensor-core evaluator carries their error term
            FftErr fx{nullptr, 0.f};
            // (k_mfft addresses moment rows in 32-bit: a bound no realistic run reaches)
            const bool fft_fits =
                std::min<int64_t>(P, pl.nbins) * (int64_t)pl.nbmax * pl.R < (int64_t)INT32_MAX;
            if (use_fft && tc && fft_fits && moments_fft_supported(pl.B)) {
                launch_moments_fft(pl.B, pl.R, L.ubin, pl.bin0, pl.nbins, N, tcheb_for(pl.B, true),
                                   L.y1c, L.y2p, padf, L.mom, pl.nbmax, L.af, L.fe, L.fqueue,
                                   sm_count, st);
                launch_fft_bucket_energy(L.buckets, L.n_buckets,
                                         (int)std::min<int64_t>(P, pl.nbins), L.fe, pl.bin0,
                                         kFftLen - pl.B, (N + pl.B - 1) / pl.B, N, pl.B, pl.R,
                                         L.qf, st);
                fx = FftErr{L.qf, fft_kappa};
                ++fft_steps;
                {
                    const double Lf = kFftLen, fftf = 5.0 * Lf * 10.0;  // log2 1024 = 10
                    const int G = kFftLen - pl.B, nblk = (N + pl.B - 1) / pl.B;
                    const int ngr = (pl.bin0 + pl.nbins - 1) / G - pl.bin0 / G + 1;
                    fft_flop += (double)nblk * pl.R * fftf +
                                (double)ngr * nblk * ((1.0 + pl.R) * fftf + pl.R * 6.0 * Lf);
                }
            } else {
                launch_moments(pl.B, pl.R, L.buckets, L.ubin, pl.bin0, pl.nbins, N,
                               tcheb_for(pl.B), L.y1c, L.y2p, padf, L.mom, pl.nbmax, sm_count, st);
            }
            if (ev1) CK(cudaEventRecord(ev1, st));
            CK(cudaMemsetAsync(L.queue, 0, sizeof(int), st));
            if (tc)
                launch_evaluate_tc(fx, pl.R, L.buckets, L.n_buckets, L.queue,
                                   (int)std::min<int64_t>(P, pl.nbins), L.sorted, fdoa_slot(s), fs,
                                   nu_c + s, pl.B, L.mom, pl.nbmax, s_out, bits, flag_base, tau,
                                   tau_noise, e1, e2, N, sm_count, st);
            else
                launch_evaluate(pl.R, L.buckets, L.n_buckets, L.queue,
                                (int)std::min<int64_t>(P, pl.nbins), L.sorted, fdoa_slot(s), fs,
                                nu_c + s, pl.B, L.mom, pl.nbmax, s_out, bits, flag_base, tau,
                                tau_noise, e1, e2, N, sm_count, st);
            launch_work_count(L.buckets, L.n_buckets, pl.B, pl.R, tc ? 1 : 0, L.work, st);
            launches += fx.qf ? 8 : 7;  // + k_fft_bucket_energy
        }
        if (ev2) CK(cudaEventRecord(ev2, st));
    }
};

// compact the refine bitmap and re-evaluate flagged elements exactly
int64_t run_refine(Scratch& sc, const uint32_t* bits, int64_t n_elems, const RefineCtx& ctx,
                   int64_t* launches) {
    const int64_t n_words = (n_elems + 31) / 32;
    auto* cnt = sc.alloc<unsigned long long>(2);
    CK(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), sc.st));
    launch_count_flags(bits, n_words, cnt, sc.st);
    unsigned long long n = 0;
    CK(cudaMemcpyAsync(&n, cnt, sizeof n, cudaMemcpyDeviceToHost, sc.st));
    CK(cudaStreamSynchronize(sc.st));
    *launches += 1;
    if (n == 0) return 0;
    auto* list = sc.alloc<int64_t>(n);
    launch_compact_flags(bits, n_words, list, cnt + 1, sc.st);
    launch_refine(list, (int64_t)n, ctx, sc.st);
    *launches += 2;
    return (int64_t)n;
}

// Refinement of batches of steps on a side stream: a batch (up to K steps)
// starts once those steps' correlators finished (events on their lanes) and
// runs on the FP64 pipes while the lanes correlate later steps.
// K = 0: everything refined at the end on the main stream (profiled runs).
struct SideRefine {
    static constexpr int kSerialBatch = 10;  // steps per batch of the K = 0 mode
    Scratch& sc;
    int steps, K;
    int64_t P, P32;
    cudaStream_t rs = nullptr;
    std::vector<cudaEvent_t> ev;
    int64_t* list = nullptr;
    unsigned long long* counts = nullptr;  // one per batch
    int next = 0, batches = 0;
    int64_t launches = 0;
    bool own_rs = false;
    SideRefine(Scratch& s, int n_steps, int64_t P_, int64_t P32_, int K_, cudaStream_t side)
        : sc(s), steps(n_steps), K(K_), P(P_), P32(P32_) {
        const int nb = steps;  // at most one batch per step
        counts = sc.alloc<unsigned long long>(nb);
        CK(cudaMemsetAsync(counts, 0, nb * sizeof(unsigned long long), sc.st));
        list = sc.alloc<int64_t>((size_t)std::min(K > 0 ? K : kSerialBatch, steps) * P32);
        if (K > 0) {
            rs = side;
            if (!rs) {
                CK(cudaStreamCreateWithFlags(&rs, cudaStreamNonBlocking));
                own_rs = true;
            }
            ev.resize(steps);
            for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            // list/counts were allocated on the main stream
            cudaEvent_t ready;
            CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
            CK(cudaEventRecord(ready, sc.st));
            CK(cudaStreamWaitEvent(rs, ready, 0));
            cudaEventDestroy(ready);
        }
    }
    ~SideRefine() {
        for (auto e : ev) cudaEventDestroy(e);
        if (own_rs && rs) cudaStreamDestroy(rs);
    }
    void launch_batch(const uint32_t* bits, const RefineCtx& ctx, int r0, int r1,
                      cudaStream_t st) {
        launch_refine_rows(bits, r0, r1, P32, list, counts + batches, ctx, st);
        ++batches;
        launches += 2;
    }
    void step_done(int s, cudaStream_t lane, const uint32_t* bits, const RefineCtx& ctx) {
        if (K <= 0) return;
        CK(cudaEventRecord(ev[s], lane));
        // batches of K steps, shrinking towards the end (a batch is due once it
        // holds as many steps as remain after it), so the refinement left after
        // the last correlation is about one step's
        if (s + 1 - next >= std::min(K, steps - 1 - s)) {
            for (int i = next; i <= s; ++i) CK(cudaStreamWaitEvent(rs, ev[i], 0));
            launch_batch(bits, ctx, next, s + 1, rs);
            next = s + 1;
        }
    }
    void finish(const uint32_t* bits, const RefineCtx& ctx) {
        if (K <= 0) {  // profiled runs: everything at the end, on the main stream
            for (int r0 = 0; r0 < steps; r0 += kSerialBatch)
                launch_batch(bits, ctx, r0, std::min(steps, r0 + kSerialBatch), sc.st);
            return;
        }
        if (next < steps) {
            for (int i = next; i < steps; ++i) CK(cudaStreamWaitEvent(rs, ev[i], 0));
            launch_batch(bits, ctx, next, steps, rs);
            next = steps;
        }
        cudaEvent_t done;
        CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
        CK(cudaEventRecord(done, rs));
        CK(cudaStreamWaitEvent(sc.st, done, 0));
        cudaEventDestroy(done);
    }
};

void check_err_flag(Scratch& sc, const int* err) {
    int h = 0;
    CK(cudaMemcpyAsync(&h, err, sizeof h, cudaMemcpyDeviceToHost, sc.st));
    CK(cudaStreamSynchronize(sc.st));
    if (h) raise(DG_EINVAL, "predict_geometry: candidate coincides with receiver");
}

std::unique_ptr<dg_session> make_session(dg_engine* eng, int64_t n1, double fs1, int64_t n2,
                                         double fs2) {
    // check_pair (backend.hpp:221-228) via BasebandCapture::validate (capture.hpp:42-46)
    if (n1 <= 0 || n2 <= 0) raise(DG_EINVAL, "BasebandCapture: no samples");
    if (!(fs1 > 0.0) || !(fs2 > 0.0)) raise(DG_EINVAL, "BasebandCapture: sample_rate_hz <= 0");
    if (fs1 != fs2) raise(DG_EINVAL, "backend stage: sample rates differ");
    if (n1 != n2) raise(DG_EINVAL, "backend stage: sample counts differ");
    set_device(eng);
    auto s = std::make_unique<dg_session>();
    s->eng = eng;
    s->N = n1;
    s->stride = capture_stride(n1);
    s->fs = fs1;
    s->y32 = std::make_unique<DevMem>(2 * s->stride * sizeof(float2));
    s->y64 = std::make_unique<DevMem>(2 * s->stride * sizeof(double2));
    CK(cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking));
    CK(cudaMemsetAsync(s->y32->p, 0, s->y32->bytes, s->st));
    CK(cudaMemsetAsync(s->y64->p, 0, s->y64->bytes, s->st));
    return s;
}

// FP32 centre-relative copy of a freshly built full lattice (planning only)
void finish_lattice(dg_grid* g, cudaStream_t st) {
    const int64_t n = g->size();
    g->full_size = n;
    const int64_t mid = n / 2;
    double c[3];
    CK(cudaMemcpyAsync(&c[0], g->x + mid, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&c[1], g->y + mid, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&c[2], g->z + mid, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    g->cx = c[0];
    g->cy = c[1];
    g->cz = c[2];
    g->rel = std::make_shared<DevMem>(n * sizeof(float4));
    launch_lattice_rel(g->x, g->y, g->z, n, g->cx, g->cy, g->cz,
                       static_cast<float4*>(g->rel->p), st);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
}

// per-step receiver pairs relative to the lattice centre, FP32
std::vector<RxPairF32> rx_pairs_f32(const dg_grid* g, const PairGeom* pg, int n) {
    std::vector<RxPairF32> out(n);
    for (int i = 0; i < n; ++i) {
        const dg_state& a = pg[i].rx_i;
        const dg_state& b = pg[i].rx_j;
        RxPairF32& r = out[i];
        r.pi[0] = (float)(a.position.x - g->cx);
        r.pi[1] = (float)(a.position.y - g->cy);
        r.pi[2] = (float)(a.position.z - g->cz);
        r.vi[0] = (float)a.velocity.x;
        r.vi[1] = (float)a.velocity.y;
        r.vi[2] = (float)a.velocity.z;
        r.pj[0] = (float)(b.position.x - g->cx);
        r.pj[1] = (float)(b.position.y - g->cy);
        r.pj[2] = (float)(b.position.z - g->cz);
        r.vj[0] = (float)b.velocity.x;
        r.vj[1] = (float)b.velocity.y;
        r.vj[2] = (float)b.velocity.z;
    }
    return out;
}

// FDOA error bound of the FP32 planning geometry: 1e-5 of the largest
// possible Doppler difference (|v_i| + |v_j|) / wl, plus 1 mHz
double fp32_fdoa_margin(const PairGeom* pg, int n, double wl) {
    double m = 0.0;
    for (int i = 0; i < n; ++i) {
        auto norm = [](const dg_ecef& v) { return std::sqrt(v.x * v.x + v.y * v.y + v.z * v.z); };
        m = std::max(m, (norm(pg[i].rx_i.velocity) + norm(pg[i].rx_j.velocity)) / wl);
    }
    return 1e-5 * m + 1e-3;
}

}  // namespace

// ===========================================================================
extern "C" {

const char* dg_last_error(void) { return last_error().c_str(); }
int dg_abi_version(void) { return DG_ABI_VERSION; }

void dg_options_default(dg_options* o) {
    std::memset(o, 0, sizeof *o);
    o->k_sigma = 5.0;
    o->exclusion_radius_cells = 5;
    o->detect = 1;
    o->patch_peak = 1;
}

void dg_tuning_default(dg_tuning* t) {
    std::memset(t, 0, sizeof *t);
    t->correlator = DG_CORRELATOR_AUTO;
    t->evaluate_tensor = 1;
    t->moment_fft = 1;
}

int dg_engine_set_tuning(dg_engine* e, const dg_tuning* t) {
    return guard([&] {
        if (!e || !t) raise(DG_EINVAL, "null argument");
        if (t->correlator < DG_CORRELATOR_AUTO || t->correlator > DG_CORRELATOR_MOMENTS)
            raise(DG_EINVAL, "dg_tuning: unknown correlator mode " + std::to_string(t->correlator));
        if (t->moment_block &&
            std::find(std::begin(kMomentB), std::end(kMomentB), t->moment_block) == std::end(kMomentB))
            raise(DG_EINVAL, "dg_tuning: unsupported moment block " + std::to_string(t->moment_block));
        if (t->moment_count &&
            std::find(std::begin(kMomentR), std::end(kMomentR), t->moment_count) == std::end(kMomentR))
            raise(DG_EINVAL, "dg_tuning: unsupported moment count " + std::to_string(t->moment_count));
        if (!(t->refine_tau >= 0.0) || !std::isfinite(t->refine_tau))
            raise(DG_EINVAL, "dg_tuning: refine_tau must be finite and >= 0");
        if (!(t->noise_refine_tau >= 0.0) || !std::isfinite(t->noise_refine_tau))
            raise(DG_EINVAL, "dg_tuning: noise_refine_tau must be finite and >= 0");
        if (t->noise_refine_tau > 0.0 && t->noise_refine_tau < kNoiseRefineTau &&
            !t->allow_weaker_refine)
            raise(DG_EINVAL, "dg_tuning: noise_refine_tau below the default " +
                                 std::to_string(kNoiseRefineTau) +
                                 " weakens the 1e-4 contract (set allow_weaker_refine)");
        if (t->surface_budget_bytes < 0)
            raise(DG_EINVAL, "dg_tuning: surface_budget_bytes < 0");
        if (t->moment_fft != 0 && t->moment_fft != 1)
            raise(DG_EINVAL, "dg_tuning: moment_fft must be 0 or 1");
        if (!(t->fft_refine_kappa >= 0.0) || !std::isfinite(t->fft_refine_kappa))
            raise(DG_EINVAL, "dg_tuning: fft_refine_kappa must be finite and >= 0");
        if (t->fft_refine_kappa > 0.0 && t->fft_refine_kappa < kFftRefineKappa &&
            !t->allow_weaker_refine)
            raise(DG_EINVAL, "dg_tuning: fft_refine_kappa below the default weakens the 1e-4 "
                             "contract (set allow_weaker_refine)");
        if (!(t->direct_refine_tau >= 0.0) || !std::isfinite(t->direct_refine_tau))
            raise(DG_EINVAL, "dg_tuning: direct_refine_tau must be finite and >= 0");
        if (t->direct_refine_tau > 0.0 && t->direct_refine_tau < kRefineTau &&
            !t->allow_weaker_refine)
            raise(DG_EINVAL, "dg_tuning: direct_refine_tau below the default " +
                                 std::to_string(kRefineTau) +
                                 " weakens the 1e-4 contract (set allow_weaker_refine)");
        if (t->refine_tau > 0.0 && t->refine_tau < kMomentRefineTau && !t->allow_weaker_refine)
            raise(DG_EINVAL, "dg_tuning: refine_tau below the default " +
                                 std::to_string(kMomentRefineTau) +
                                 " weakens the 1e-4 contract (set allow_weaker_refine)");
        std::lock_guard<std::mutex> lk(e->tables_mu);
        e->tuning = *t;
        for (dg_engine* p : e->peers) {
            std::lock_guard<std::mutex> lp(p->tables_mu);
            p->tuning = *t;
        }
    });
}

int dg_engine_get_tuning(const dg_engine* e, dg_tuning* t) {
    return guard([&] {
        if (!e || !t) raise(DG_EINVAL, "null argument");
        *t = e->tuning;
    });
}

int dg_engine_create(int device, dg_engine** out) {
    return guard([&] {
        int n = 0;
        CK(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n)
            raise(DG_EINVAL, "dg_engine_create: device " + std::to_string(device) +
                                 " out of range (" + std::to_string(n) + " visible)");
        CK(cudaSetDevice(device));
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10)
            raise(DG_ERUNTIME, std::string("b200: sm_100a build cannot run on ") + prop.name);
        // keep freed stream-ordered scratch (per-run surfaces, GBs at C3/C5)
        // mapped in the pool instead of returning it to the driver at every sync
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t keep = UINT64_MAX;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        auto e = std::make_unique<dg_engine>();
        e->device = device;
        e->sm_count = prop.multiProcessorCount;
        dg_tuning_default(&e->tuning);
        CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&e->upload, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&e->lane, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&e->refine, cudaStreamNonBlocking));
        *out = e.release();
    });
}

int dg_device_count(int* n) {
    return guard([&] {
        if (!n) raise(DG_EINVAL, "null argument");
        CK(cudaGetDeviceCount(n));
    });
}

int dg_engine_create_multi(const int* devices, int n, dg_engine** out) {
    return guard([&] {
        if (!devices || n < 1 || !out) raise(DG_EINVAL, "dg_engine_create_multi: no devices");
        dg_engine* first = nullptr;
        if (int rc = dg_engine_create(devices[0], &first)) raise(rc, last_error());
        std::unique_ptr<dg_engine> e(first);
        for (int k = 1; k < n; ++k) {
            dg_engine* p = nullptr;
            if (int rc = dg_engine_create(devices[k], &p)) raise(rc, last_error());
            e->peers.push_back(p);
            p->tuning = e->tuning;
        }
        // peer access between distinct devices (NVLink / NVSwitch P2P)
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b) {
                if (devices[a] == devices[b]) continue;
                int can = 0;
                CK(cudaDeviceCanAccessPeer(&can, devices[a], devices[b]));
                if (!can) continue;
                CK(cudaSetDevice(devices[a]));
                const cudaError_t rc = cudaDeviceEnablePeerAccess(devices[b], 0);
                if (rc == cudaErrorPeerAccessAlreadyEnabled)
                    cudaGetLastError();
                else
                    CK(rc);
            }
        CK(cudaSetDevice(devices[0]));
        *out = e.release();
    });
}

void dg_engine_destroy(dg_engine* e) { delete e; }

int dg_engine_descriptor(const dg_engine* e, char* name, size_t nl, char* kind, size_t kl,
                         unsigned* workers) {
    return guard([&] {
        if (!e) raise(DG_EINVAL, "null engine");
        if (name && nl) std::snprintf(name, nl, "%s", "b200");
        if (kind && kl) std::snprintf(kind, kl, "%s", "parallel-batched");
        if (workers) *workers = (unsigned)e->n_devices();
    });
}

// ---- sessions --------------------------------------------------------------
int dg_stage(dg_engine* eng, const double* y1, int64_t n1, double fs1, const double* y2, int64_t n2,
             double fs2, dg_session** out) {
    return guard([&] {
        auto s = make_session(eng, n1, fs1, n2, fs2);
        auto* y64 = static_cast<double2*>(s->y64->p) + kCapturePad;
        auto* y32 = static_cast<float2*>(s->y32->p) + kCapturePad;
        CK(cudaMemcpyAsync(y64, y1, n1 * sizeof(double2), cudaMemcpyHostToDevice, s->st));
        CK(cudaMemcpyAsync(y64 + s->stride, y2, n1 * sizeof(double2), cudaMemcpyHostToDevice, s->st));
        launch_f64_to_f32(y64, y32, n1, s->st);
        launch_f64_to_f32(y64 + s->stride, y32 + s->stride, n1, s->st);
        s->e64 = std::make_unique<DevMem>(2 * (n1 + 1) * sizeof(double));
        launch_energy_prefix(y64, s->stride, 2, n1, static_cast<double*>(s->e64->p), s->st);
        CK(cudaStreamSynchronize(s->st));
        *out = s.release();
    });
}

int dg_stage_f32(dg_engine* eng, const float* y1, int64_t n1, double fs1, const float* y2,
                 int64_t n2, double fs2, dg_session** out) {
    return guard([&] {
        auto s = make_session(eng, n1, fs1, n2, fs2);
        auto* y64 = static_cast<double2*>(s->y64->p) + kCapturePad;
        auto* y32 = static_cast<float2*>(s->y32->p) + kCapturePad;
        CK(cudaMemcpyAsync(y32, y1, n1 * sizeof(float2), cudaMemcpyHostToDevice, s->st));
        CK(cudaMemcpyAsync(y32 + s->stride, y2, n1 * sizeof(float2), cudaMemcpyHostToDevice, s->st));
        launch_f32_to_f64(y32, y64, n1, s->st);
        launch_f32_to_f64(y32 + s->stride, y64 + s->stride, n1, s->st);
        s->e64 = std::make_unique<DevMem>(2 * (n1 + 1) * sizeof(double));
        launch_energy_prefix(y64, s->stride, 2, n1, static_cast<double*>(s->e64->p), s->st);
        CK(cudaStreamSynchronize(s->st));
        *out = s.release();
    });
}

void dg_session_destroy(dg_session* s) { delete s; }

int dg_correlate_batch(dg_session* s, const dg_pair_offsets* batch, int64_t n, double* out,
                       int64_t n_out) {
    return guard([&] {
        if (!s) raise(DG_EINVAL, "null session");
        // SerialSession::correlate_batch (backend.hpp:235-242)
        if (n <= 0 || !batch) raise(DG_EINVAL, "correlate_batch: empty batch");
        if (n_out != n) raise(DG_EINVAL, "correlate_batch: output size mismatch");
        set_device(s->eng);
        Scratch sc(s->st);
        Pipeline pl;
        pl.init(sc, s->eng, n, s->N, 1);
        pl.init_lanes(sc);
        auto* off = sc.alloc<dg_pair_offsets>(n);
        auto* vals = sc.alloc<double>(n);
        const int64_t n_words = (n + 31) / 32;
        auto* bits = sc.alloc<uint32_t>(n_words);
        CK(cudaMemsetAsync(bits, 0, n_words * sizeof(uint32_t), s->st));
        CK(cudaMemcpyAsync(off, batch, n * sizeof(dg_pair_offsets), cudaMemcpyHostToDevice, s->st));
        pl.reset_ranges(sc, 1);
        launch_offsets_hist(off, n, pl.N, pl.d_slot(0), pl.rank_slot(0), pl.fdoa_slot(0),
                            pl.hist_slot(0), vals,
                            pl.overlap, pl.range, s->st);
        pl.plan_window(sc, 1, s->fs);
        const auto* y32 = static_cast<const float2*>(s->y32->p) + kCapturePad;
        const auto* y64 = static_cast<const double2*>(s->y64->p) + kCapturePad;
        const double* e64 = static_cast<const double*>(s->e64->p);
        pl.correlate(0, y64, y32, y32 + s->stride, e64, e64 + (s->N + 1), s->fs, vals, bits, 0,
                     nullptr, nullptr,
                     nullptr);
        RefineCtx ctx{};
        ctx.P = n;
        ctx.offsets = off;
        ctx.y64 = static_cast<const double2*>(s->y64->p) + kCapturePad;
        ctx.stride = s->stride;
        ctx.N = (int)s->N;
        ctx.fs = s->fs;
        ctx.raw = vals;
        int64_t launches = 0;
        run_refine(sc, bits, n, ctx, &launches);
        CK(cudaMemcpyAsync(out, vals, n * sizeof(double), cudaMemcpyDeviceToHost, s->st));
        CK(cudaStreamSynchronize(s->st));
    });
}

// ---- grids -----------------------------------------------------------------
}  // extern "C"
namespace {
// The eager ECEF lattice of GridAxis pairs (geodesy.hpp:151-168, lla_to_ecef
// :82-92 per lattice_coord): per-row / per-column libm trig on the host, the
// products on the device (launch_grid_ecef), then the FP32 planning copy.
std::unique_ptr<dg_grid> make_lattice(dg_engine* eng, double lat_start, double lat_step,
                                      int64_t n_lat, double lon_start, double lon_step,
                                      int64_t n_lon, double alt) {
    const int64_t n = n_lat * n_lon;
    std::vector<double> ra(n_lat), rz(n_lat), cc(n_lon), cs(n_lon);
    for (int64_t i = 0; i < n_lat; ++i) {
        const double lat = deg2rad(lat_start + static_cast<double>(i) * lat_step);
        const double slat = std::sin(lat), clat = std::cos(lat);
        const double nn = kA / std::sqrt(1.0 - kE2 * slat * slat);
        ra[i] = (nn + alt) * clat;
        rz[i] = (nn * (1.0 - kE2) + alt) * slat;
    }
    for (int64_t j = 0; j < n_lon; ++j) {
        const double lon = deg2rad(lon_start + static_cast<double>(j) * lon_step);
        cc[j] = std::cos(lon);
        cs[j] = std::sin(lon);
    }
    set_device(eng);
    auto g = std::make_unique<dg_grid>();
    g->eng = eng;
    g->lat_start = lat_start;
    g->lon_start = lon_start;
    g->lat_step = lat_step;
    g->lon_step = lon_step;
    g->alt = alt;
    g->n_lat = n_lat;
    g->n_lon = n_lon;
    g->mem = std::make_shared<DevMem>(3 * n * sizeof(double));
    double* base = static_cast<double*>(g->mem->p);
    g->x = base;
    g->y = base + n;
    g->z = base + 2 * n;
    StreamGuard sg(nullptr, eng->stream);
    Scratch sc(sg.st);
    double* t = sc.alloc<double>(2 * n_lat + 2 * n_lon);
    CK(cudaMemcpyAsync(t, ra.data(), n_lat * 8, cudaMemcpyHostToDevice, sg.st));
    CK(cudaMemcpyAsync(t + n_lat, rz.data(), n_lat * 8, cudaMemcpyHostToDevice, sg.st));
    CK(cudaMemcpyAsync(t + 2 * n_lat, cc.data(), n_lon * 8, cudaMemcpyHostToDevice, sg.st));
    CK(cudaMemcpyAsync(t + 2 * n_lat + n_lon, cs.data(), n_lon * 8, cudaMemcpyHostToDevice, sg.st));
    launch_grid_ecef(t, t + n_lat, t + 2 * n_lat, t + 2 * n_lat + n_lon, n_lat, n_lon, base,
                     base + n, base + 2 * n, sg.st);
    CK(cudaGetLastError());
    finish_lattice(g.get(), sg.st);
    return g;
}

}  // namespace
extern "C" {

int dg_build_candidate_grid(dg_engine* eng, const dg_latlon_bounds* b, double spacing, double alt,
                            uint64_t cap, dg_grid** out) {
    return guard([&] {
        if (!eng || !b) raise(DG_EINVAL, "null argument");
        if (cap == 0) cap = 20'000'000;  // default_grid_point_cap (geodesy.hpp:170)
        // LatLonBounds::validate (geodesy.hpp:132-137) — lon_max is not range-checked there
        validate_geodetic(b->lat_min_deg, b->lon_min_deg, 0.0);
        validate_geodetic(b->lat_max_deg, b->lon_min_deg, 0.0);
        if (b->lat_max_deg < b->lat_min_deg || b->lon_max_deg < b->lon_min_deg)
            raise(DG_EINVAL, "LatLonBounds: max < min");
        if (!(spacing > 0.0)) raise(DG_EINVAL, "build_candidate_grid: spacing_deg <= 0");
        if (!std::isfinite(alt)) raise(DG_EINVAL, "build_candidate_grid: altitude_m not finite");
        auto axis_count = [](double span, double step) {  // geodesy.hpp:175-177
            return static_cast<int64_t>(std::floor(span / step + 1e-6)) + 1;
        };
        const int64_t n_lat = axis_count(b->lat_max_deg - b->lat_min_deg, spacing);
        const int64_t n_lon = axis_count(b->lon_max_deg - b->lon_min_deg, spacing);
        const int64_t n = n_lat * n_lon;
        if ((uint64_t)n > cap)
            raise(DG_EINVAL, "build_candidate_grid: " + std::to_string(n) +
                                 " points exceed cap of " + std::to_string(cap));
        // validated in the reference's loop order
        for (int64_t i = 0; i < n_lat; ++i) {
            const double lat_deg = b->lat_min_deg + static_cast<double>(i) * spacing;
            if (!(lat_deg >= -90.0 && lat_deg <= 90.0))
                raise(DG_EINVAL, "GeodeticCoord: lat_deg out of [-90, 90]: " + fmt_double(lat_deg));
            if (i == 0)
                for (int64_t j = 0; j < n_lon; ++j) {
                    const double lon_deg = b->lon_min_deg + static_cast<double>(j) * spacing;
                    validate_geodetic(lat_deg, lon_deg, alt);
                }
        }
        auto g = make_lattice(eng, b->lat_min_deg, spacing, n_lat, b->lon_min_deg, spacing, n_lon,
                              alt);
        *out = g.release();
    });
}

int dg_grid_slab(const dg_grid* g, int64_t r0, int64_t r1, dg_grid** out) {
    return guard([&] {
        if (!g) raise(DG_EINVAL, "null grid");
        if (r0 < 0 || r1 > g->n_lat || r0 > r1) raise(DG_EINVAL, "dg_grid_slab: bad row range");
        auto s = std::make_unique<dg_grid>(*g);
        s->replicas = std::make_shared<Replicas<dg_grid>>();
        s->n_lat = r1 - r0;
        s->row_offset = g->row_offset + r0;
        s->x = g->x + r0 * g->n_lon;
        s->y = g->y + r0 * g->n_lon;
        s->z = g->z + r0 * g->n_lon;
        *out = s.release();
    });
}

int dg_grid_from_axes(dg_engine* eng, const dg_grid_axes* a, dg_grid** out) {
    return guard([&] {
        if (!eng || !a || !out) raise(DG_EINVAL, "null argument");
        if (a->lat_count <= 0 || a->lon_count <= 0) raise(DG_EINVAL, "dg_grid_from_axes: empty axis");
        *out = make_lattice(eng, a->lat_start_deg, a->lat_step_deg, a->lat_count,
                            a->lon_start_deg, a->lon_step_deg, a->lon_count, a->altitude_m)
                   .release();
    });
}

int dg_grid_from_points(dg_engine* eng, const dg_ecef* pts, int64_t n, double lat_start,
                        double lat_step, int64_t n_lat, double lon_start, double lon_step,
                        int64_t n_lon, double alt, dg_grid** out) {
    return guard([&] {
        if (!eng || !pts || n <= 0) raise(DG_EINVAL, "correlate_snapshot: empty grid");
        if (n_lat * n_lon != n) raise(DG_EINVAL, "dg_grid_from_points: n_lat*n_lon != n_points");
        set_device(eng);
        auto g = std::make_unique<dg_grid>();
        g->eng = eng;
        g->lat_start = lat_start;
        g->lat_step = lat_step;
        g->lon_start = lon_start;
        g->lon_step = lon_step;
        g->n_lat = n_lat;
        g->n_lon = n_lon;
        g->alt = alt;
        std::vector<double> soa(3 * n);
        for (int64_t i = 0; i < n; ++i) {
            soa[i] = pts[i].x;
            soa[n + i] = pts[i].y;
            soa[2 * n + i] = pts[i].z;
        }
        g->mem = std::make_shared<DevMem>(3 * n * sizeof(double));
        double* base = static_cast<double*>(g->mem->p);
        CK(cudaMemcpy(base, soa.data(), 3 * n * sizeof(double), cudaMemcpyHostToDevice));
        g->x = base;
        g->y = base + n;
        g->z = base + 2 * n;
        StreamGuard sg(nullptr, eng->stream);
        finish_lattice(g.get(), sg.st);
        *out = g.release();
    });
}

int dg_grid_info(const dg_grid* g, double* lat_start, double* lat_step, int64_t* n_lat,
                 double* lon_start, double* lon_step, int64_t* n_lon, double* alt,
                 int64_t* row_offset) {
    return guard([&] {
        if (!g) raise(DG_EINVAL, "null grid");
        if (lat_start) *lat_start = g->lat_start;
        if (lat_step) *lat_step = g->lat_step;
        if (n_lat) *n_lat = g->n_lat;
        if (lon_start) *lon_start = g->lon_start;
        if (lon_step) *lon_step = g->lon_step;
        if (n_lon) *n_lon = g->n_lon;
        if (alt) *alt = g->alt;
        if (row_offset) *row_offset = g->row_offset;
    });
}

int dg_grid_points(const dg_grid* g, dg_ecef* out) {
    return guard([&] {
        if (!g) raise(DG_EINVAL, "null grid");
        set_device(g->eng);
        const int64_t n = g->size();
        std::vector<double> soa(3 * n);
        CK(cudaMemcpy(soa.data(), g->x, n * 8, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(soa.data() + n, g->y, n * 8, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(soa.data() + 2 * n, g->z, n * 8, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < n; ++i) out[i] = dg_ecef{soa[i], soa[n + i], soa[2 * n + i]};
    });
}

void dg_grid_destroy(dg_grid* g) { delete g; }

int dg_predict_offsets(dg_engine* eng, const dg_grid* g, const dg_state* rx_i, const dg_state* rx_j,
                       double fs, double wl, dg_pair_offsets* out) {
    return guard([&] {
        if (!eng || !g || !rx_i || !rx_j || !out) raise(DG_EINVAL, "null argument");
        set_device(eng);
        StreamGuard sg(nullptr, eng->stream);
        Scratch sc(sg.st);
        const int64_t P = g->size();
        auto* pg = sc.alloc<PairGeom>(1);
        auto* err = sc.alloc<int>(1);
        auto* o = sc.alloc<dg_pair_offsets>(P);
        const PairGeom h{*rx_i, *rx_j};
        CK(cudaMemcpyAsync(pg, &h, sizeof h, cudaMemcpyHostToDevice, sg.st));
        CK(cudaMemsetAsync(err, 0, sizeof(int), sg.st));
        launch_predict_offsets(g->x, g->y, g->z, P, pg, fs, wl, o, err, sg.st);
        check_err_flag(sc, err);
        CK(cudaMemcpyAsync(out, o, P * sizeof(dg_pair_offsets), cudaMemcpyDeviceToHost, sg.st));
        CK(cudaStreamSynchronize(sg.st));
    });
}


int dg_correlate_snapshot(dg_session* s, const dg_grid* g, const dg_state* rx_i,
                          const dg_state* rx_j, double fc, double* out) {
    return guard([&] {
        if (!s || !g || !rx_i || !rx_j || !out) raise(DG_EINVAL, "null argument");
        if (g->size() == 0) raise(DG_EINVAL, "correlate_snapshot: empty grid");
        if (!(fc > 0.0)) raise(DG_EINVAL, "wavelength_m: center_freq_hz <= 0");
        const double wl = kC / fc;  // wavelength_m (geometry.hpp:36-39)
        set_device(s->eng);
        Scratch sc(s->st);
        const int64_t P = g->size();
        Pipeline pl;
        pl.init(sc, s->eng, P, s->N, 1);
        pl.init_lanes(sc);
        auto* pg = sc.alloc<PairGeom>(1);
        auto* vals = sc.alloc<double>(P);
        const int64_t n_words = (P + 31) / 32;
        auto* bits = sc.alloc<uint32_t>(n_words);
        const PairGeom h{*rx_i, *rx_j};
        CK(cudaMemcpyAsync(pg, &h, sizeof h, cudaMemcpyHostToDevice, s->st));
        CK(cudaMemsetAsync(bits, 0, n_words * sizeof(uint32_t), s->st));
        pl.reset_ranges(sc, 1);
        launch_geometry_hist(g->x, g->y, g->z, P, pg, s->fs, wl, pl.N, pl.d_slot(0),
                             pl.rank_slot(0), pl.fdoa_slot(0), pl.hist_slot(0), vals, pl.overlap, pl.err, pl.range,
                             s->st);
        const StepRange* approx = pl.lattice_ranges(sc, g, &h, 1, s->fs, wl);
        pl.plan_window(sc, 1, s->fs, approx, fp32_fdoa_margin(&h, 1, wl), g->full_size);
        const auto* y32 = static_cast<const float2*>(s->y32->p) + kCapturePad;
        const auto* y64 = static_cast<const double2*>(s->y64->p) + kCapturePad;
        const double* e64 = static_cast<const double*>(s->e64->p);
        pl.correlate(0, y64, y32, y32 + s->stride, e64, e64 + (s->N + 1), s->fs, vals, bits, 0,
                     nullptr, nullptr,
                     nullptr);
        check_err_flag(sc, pl.err);
        static const int pair_rx[2] = {0, 1};
        auto* prx = sc.alloc<int>(2);
        CK(cudaMemcpyAsync(prx, pair_rx, sizeof pair_rx, cudaMemcpyHostToDevice, s->st));
        RefineCtx ctx{};
        ctx.x = g->x;
        ctx.y = g->y;
        ctx.z = g->z;
        ctx.P = P;
        ctx.pg = pg;
        ctx.pair_rx = prx;
        ctx.pairs = 1;
        ctx.R = 2;
        ctx.y64 = static_cast<const double2*>(s->y64->p) + kCapturePad;
        ctx.stride = s->stride;
        ctx.N = (int)s->N;
        ctx.fs = s->fs;
        ctx.wl = wl;
        ctx.raw = vals;
        int64_t launches = 0;
        run_refine(sc, bits, P, ctx, &launches);
        CK(cudaMemcpyAsync(out, vals, P * sizeof(double), cudaMemcpyDeviceToHost, s->st));
        CK(cudaStreamSynchronize(s->st));
    });
}

// ---- staged snapshots --------------------------------------------------------
namespace {

void validate_snapshots(const dg_snapshots* sn) {
    if (!sn) raise(DG_EINVAL, "null snapshots");
    if (sn->n_snapshots < 1) raise(DG_EINVAL, "geolocate_snapshots: no snapshots");
    if (sn->n_receivers < 2) raise(DG_EINVAL, "correlate_snapshot_all_pairs: need >= 2 receivers");
    if (sn->n_samples < 1) raise(DG_EINVAL, "BasebandCapture: no samples");
    if (!(sn->sample_rate_hz > 0.0)) raise(DG_EINVAL, "BasebandCapture: sample_rate_hz <= 0");
    if (!(sn->center_freq_hz > 0.0)) raise(DG_EINVAL, "wavelength_m: center_freq_hz <= 0");
    if (!sn->states) raise(DG_EINVAL, "null receiver states");
    if (!sn->captures_iq && !sn->captures_f32) raise(DG_EINVAL, "null captures");
}

}  // namespace

// ---- DGIQ capture files (io.hpp:123-167) ------------------------------------
namespace {

// read_iq's header checks and messages (io.hpp:140-163, ByteReader io.hpp:75-84,
// read_file_bytes :112-117); leaves `f` positioned at the payload
struct IqReader {
    std::FILE* f = nullptr;
    dg_iq_header h{};
    explicit IqReader(const char* path) {
        if (!path) raise(DG_EINVAL, "null path");
        const std::string p(path);
        f = std::fopen(path, "rb");
        if (!f) raise(DG_ERUNTIME, "cannot open " + p);
        unsigned char hb[38];
        const size_t got = std::fread(hb, 1, sizeof hb, f);
        const std::string ctx = "read_iq(" + p + ")";
        if (got < 4) raise(DG_ERUNTIME, ctx + ": truncated file");
        if (std::memcmp(hb, "DGIQ", 4) != 0) raise(DG_ERUNTIME, "read_iq: bad magic in " + p);
        if (got < 6) raise(DG_ERUNTIME, ctx + ": truncated file");
        const unsigned version = hb[4] | (hb[5] << 8);
        if (version != 1)
            raise(DG_ERUNTIME, "read_iq: unsupported version " + std::to_string(version));
        if (got < 38) raise(DG_ERUNTIME, ctx + ": truncated file");
        uint64_t cnt = 0;
        std::memcpy(&h.sample_rate_hz, hb + 6, 8);  // little-endian host (x86-64 / aarch64)
        std::memcpy(&h.center_freq_hz, hb + 14, 8);
        std::memcpy(&h.start_time_s, hb + 22, 8);
        std::memcpy(&cnt, hb + 30, 8);
        if (std::fseek(f, 0, SEEK_END) != 0) raise(DG_ERUNTIME, "cannot open " + p);
        const long end = std::ftell(f);
        if (end < 38 || (uint64_t)(end - 38) != cnt * 8)
            raise(DG_ERUNTIME, "read_iq: payload length does not match sample_count in " + p);
        std::fseek(f, 38, SEEK_SET);
        h.sample_count = (int64_t)cnt;
        // BasebandCapture::validate (capture.hpp:42-46)
        if (cnt == 0) raise(DG_EINVAL, "BasebandCapture: no samples");
        if (!(h.sample_rate_hz > 0.0)) raise(DG_EINVAL, "BasebandCapture: sample_rate_hz <= 0");
    }
    void read_payload(float* dst) {
        const size_t n = (size_t)h.sample_count * 2;
        if (std::fread(dst, sizeof(float), n, f) != n)
            raise(DG_ERUNTIME, "read_iq: short read");
    }
    ~IqReader() {
        if (f) std::fclose(f);
    }
};

}  // namespace

int dg_read_iq_header(const char* path, dg_iq_header* out) {
    return guard([&] {
        if (!out) raise(DG_EINVAL, "null argument");
        IqReader r(path);
        *out = r.h;
    });
}

int dg_read_iq(const char* path, dg_iq_header* out, float* iq, int64_t capacity) {
    return guard([&] {
        if (!out) raise(DG_EINVAL, "null argument");
        IqReader r(path);
        *out = r.h;
        if (iq) {
            if (capacity < r.h.sample_count) raise(DG_EINVAL, "dg_read_iq: buffer too small");
            r.read_payload(iq);
        }
    });
}

int dg_stage_snapshots_iq(dg_engine* eng, const char* const* paths, int64_t S, int64_t R,
                          const dg_state* states, dg_staged** out) {
    return guard([&] {
        if (!eng || !paths || !states || !out) raise(DG_EINVAL, "null argument");
        if (S < 1) raise(DG_EINVAL, "geolocate_snapshots: no snapshots");
        if (R < 2) raise(DG_EINVAL, "correlate_snapshot_all_pairs: need >= 2 receivers");
        const int64_t n_caps = S * R;
        std::vector<dg_iq_header> hdr(n_caps);
        for (int64_t c = 0; c < n_caps; ++c) hdr[c] = IqReader(paths[c]).h;
        for (int64_t c = 1; c < n_caps; ++c) {  // check_pair (backend.hpp:221-228)
            if (hdr[c].sample_rate_hz != hdr[0].sample_rate_hz)
                raise(DG_EINVAL, "backend stage: sample rates differ");
            if (hdr[c].sample_count != hdr[0].sample_count)
                raise(DG_EINVAL, "backend stage: sample counts differ");
            if (hdr[c].center_freq_hz != hdr[0].center_freq_hz)
                raise(DG_EINVAL, "dg_stage_snapshots_iq: center frequencies differ");
        }
        if (!(hdr[0].center_freq_hz > 0.0)) raise(DG_EINVAL, "wavelength_m: center_freq_hz <= 0");
        set_device(eng);
        auto s = std::make_unique<dg_staged>();
        s->eng = eng;
        s->S = S;
        s->R = R;
        s->N = hdr[0].sample_count;
        s->stride = capture_stride(s->N);
        s->fs = hdr[0].sample_rate_hz;
        s->fc = hdr[0].center_freq_hz;
        s->states.assign(states, states + n_caps);
        s->y32 = std::make_unique<DevMem>(n_caps * s->stride * sizeof(float2));
        s->y64 = std::make_unique<DevMem>(n_caps * s->stride * sizeof(double2));
        auto* y32 = static_cast<float2*>(s->y32->p) + kCapturePad;
        auto* y64 = static_cast<double2*>(s->y64->p) + kCapturePad;
        StreamGuard sg(nullptr, eng->stream);
        CK(cudaMemsetAsync(s->y32->p, 0, s->y32->bytes, sg.st));
        CK(cudaMemsetAsync(s->y64->p, 0, s->y64->bytes, sg.st));
        // payloads go from disk straight into two pinned buffers (float32 I/Q is
        // the device layout), each copy to HBM overlapping the next file's read
        const size_t bytes = (size_t)s->N * sizeof(float2);
        void* pin[2] = {nullptr, nullptr};
        cudaEvent_t ev[2] = {nullptr, nullptr};
        struct PinFree {
            void** p;
            cudaEvent_t* e;
            ~PinFree() {
                for (int i = 0; i < 2; ++i) {
                    if (e[i]) {
                        cudaEventSynchronize(e[i]);
                        cudaEventDestroy(e[i]);
                    }
                    if (p[i]) cudaFreeHost(p[i]);
                }
            }
        } pin_free{pin, ev};
        for (int i = 0; i < 2; ++i) {
            CK(cudaHostAlloc(&pin[i], bytes, cudaHostAllocDefault));
            CK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        }
        for (int64_t c = 0; c < n_caps; ++c) {
            const int b = (int)(c & 1);
            if (c >= 2) CK(cudaEventSynchronize(ev[b]));  // its previous copy is done
            IqReader r(paths[c]);
            r.read_payload(static_cast<float*>(pin[b]));
            CK(cudaMemcpyAsync(y32 + c * s->stride, pin[b], bytes, cudaMemcpyHostToDevice,
                               sg.st));
            CK(cudaEventRecord(ev[b], sg.st));
            launch_f32_to_f64(y32 + c * s->stride, y64 + c * s->stride, s->N, sg.st);
        }
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(sg.st));
        *out = s.release();
    });
}

}  // extern "C"

namespace {

// H2D staging of a run's captures (complex double or float I/Q). Contiguous
// [S][R][N] host captures go up in one 2-D copy and one conversion kernel.
// async: on the engine's upload stream, completion recorded in s->ready and
// not waited for here (dg_geolocate_snapshots overlaps it with the geometry
// and planning phase; the correlator lanes wait for the event).
std::unique_ptr<dg_staged> stage_impl(dg_engine* eng, const dg_snapshots* sn, bool async) {
    if (!eng) raise(DG_EINVAL, "null engine");
    validate_snapshots(sn);
    set_device(eng);
    auto s = std::make_unique<dg_staged>();
    s->eng = eng;
    s->S = sn->n_snapshots;
    s->R = sn->n_receivers;
    s->N = sn->n_samples;
    s->stride = capture_stride(s->N);
    s->fs = sn->sample_rate_hz;
    s->fc = sn->center_freq_hz;
    s->states.assign(sn->states, sn->states + s->S * s->R);
    const int64_t n_caps = s->S * s->R;
    s->y32 = std::make_unique<DevMem>(n_caps * s->stride * sizeof(float2));
    s->y64 = std::make_unique<DevMem>(n_caps * s->stride * sizeof(double2));
    auto* y32 = static_cast<float2*>(s->y32->p);
    auto* y64 = static_cast<double2*>(s->y64->p);
    cudaStream_t st = async ? eng->upload : eng->stream;
    const bool f64 = sn->captures_iq != nullptr;
    bool contiguous = true;
    for (int64_t c = 0; c < n_caps; ++c) {
        const void* p = f64 ? (const void*)sn->captures_iq[c] : (const void*)sn->captures_f32[c];
        if (!p) raise(DG_EINVAL, "null capture pointer");
        const char* base = f64 ? (const char*)sn->captures_iq[0] : (const char*)sn->captures_f32[0];
        const size_t el = f64 ? sizeof(double2) : sizeof(float2);
        contiguous = contiguous && (const char*)p == base + c * s->N * el;
    }
    // one contiguous upload (a pitched 2-D copy of ~100 rows stalled the host
    // for ~0.3 ms in the driver), then one kernel fills both padded copies
    const size_t el = f64 ? sizeof(double2) : sizeof(float2);
    void* tmp = nullptr;
    CK(cudaMallocAsync(&tmp, (size_t)n_caps * s->N * el, st));
    if (contiguous) {
        const void* src = f64 ? (const void*)sn->captures_iq[0] : (const void*)sn->captures_f32[0];
        CK(cudaMemcpyAsync(tmp, src, (size_t)n_caps * s->N * el, cudaMemcpyHostToDevice, st));
    } else {
        for (int64_t c = 0; c < n_caps; ++c) {
            const void* src = f64 ? (const void*)sn->captures_iq[c] : (const void*)sn->captures_f32[c];
            CK(cudaMemcpyAsync((char*)tmp + c * s->N * el, src, s->N * el, cudaMemcpyHostToDevice,
                               st));
        }
    }
    launch_stage_captures(tmp, f64, n_caps, s->N, s->stride, kCapturePad, y64, y32, st);
    CK(cudaFreeAsync(tmp, st));
    CK(cudaGetLastError());
    if (async) {
        CK(cudaEventCreateWithFlags(&s->ready, cudaEventDisableTiming));
        CK(cudaEventRecord(s->ready, st));
    } else {
        CK(cudaStreamSynchronize(st));
    }
    return s;
}

}  // namespace

extern "C" {

int dg_stage_snapshots(dg_engine* eng, const dg_snapshots* sn, dg_staged** out) {
    return guard([&] { *out = stage_impl(eng, sn, false).release(); });
}

void dg_staged_destroy(dg_staged* s) { delete s; }

}  // extern "C"

// ---- the driver --------------------------------------------------------------
namespace {

constexpr int kDetCap = 8192;
// k_greedy holds the sorted list, statuses and 16-bit kept indices in shared memory
// (24 + 1 + 2 bytes per entry: 216 KiB at 8,192)
static_assert(kDetCap <= 8192, "k_greedy's shared-memory layout");

// detect_emitters (correlate.hpp:127-201). Mean / sigma, the threshold and the
// 3x3 local-maximum test run on the device; up to kDetCap local maxima are
// sorted and greedily excluded by one CTA (k_greedy). Past that (low k_sigma
// on large grids) every local maximum is listed on the device and the sort +
// Chebyshev exclusion run on the host over a bucket grid of side radius + 1
// (at most 4 accepted peaks per bucket), so the list is never truncated.
void lattice_fill(const dg_grid* g, dg_emitter_estimate* out, int64_t m) {
    for (int64_t i = 0; i < m; ++i) {
        // lattice_coord (geodesy.hpp:160-162) with GridAxis::value (:145)
        const int64_t ilat = (int64_t)out[i].lat_deg + g->row_offset;
        const int64_t ilon = (int64_t)out[i].lon_deg;
        out[i].lat_deg = g->lat_start + static_cast<double>(ilat) * g->lat_step;
        out[i].lon_deg = g->lon_start + static_cast<double>(ilon) * g->lon_step;
        out[i].alt_m = g->alt;
        out[i].grid_index = ilat * g->n_lon + ilon;
    }
}

void greedy_host(std::vector<DetCand>& c, int radius, double mean, double sigma, int64_t n_lon,
                 std::vector<dg_emitter_estimate>& out) {
    std::sort(c.begin(), c.end(), [](const DetCand& a, const DetCand& b) {
        if (a.score != b.score) return a.score > b.score;
        return a.key < b.key;  // correlate.hpp:172-175
    });
    const int64_t side = (int64_t)radius + 1;
    std::unordered_map<uint64_t, std::vector<int>> buckets;  // accepted (ilat, ilon) by bucket
    std::vector<DetCand> acc;
    auto bkey = [](int64_t a, int64_t b) { return ((uint64_t)(uint32_t)a << 32) | (uint32_t)b; };
    for (const DetCand& d : c) {
        const int64_t bi = d.ilat / side, bj = d.ilon / side;
        bool excluded = false;
        for (int64_t a = bi - 1; a <= bi + 1 && !excluded; ++a)
            for (int64_t b = bj - 1; b <= bj + 1 && !excluded; ++b) {
                auto it = buckets.find(bkey(a, b));
                if (it == buckets.end()) continue;
                for (int k : it->second)
                    if (std::max(std::abs(d.ilat - acc[k].ilat), std::abs(d.ilon - acc[k].ilon)) <=
                        radius) {
                        excluded = true;
                        break;
                    }
            }
        if (excluded) continue;
        buckets[bkey(bi, bj)].push_back((int)acc.size());
        acc.push_back(d);
        dg_emitter_estimate e;
        e.lat_deg = (double)d.ilat;  // lattice coordinates filled in by lattice_fill
        e.lon_deg = (double)d.ilon;
        e.alt_m = 0.0;
        e.grid_index = (int64_t)d.ilat * n_lon + d.ilon;
        e.score = d.score;
        e.score_zsigma = (d.score - mean) / sigma;
        out.push_back(e);
    }
}

void run_detect(const dg_grid* g, const double* v_dev, double k_sigma, int radius,
                dg_emitter_estimate* out, int64_t capacity, int64_t* n_out, Scratch& sc,
                int64_t* launches) {
    if (radius < 0) raise(DG_EINVAL, "detect_emitters: negative exclusion radius");
    const int64_t P = g->size();
    const int n_part = 148 * 4;
    auto* part = sc.alloc<double>(n_part);
    auto* stats = sc.alloc<double>(3);
    auto* cands = sc.alloc<DetCand>(kDetCap);
    auto* n_c = sc.alloc<int>(2);
    auto* dets = sc.alloc<dg_emitter_estimate>(kDetCap);
    CK(cudaMemsetAsync(n_c, 0, 2 * sizeof(int), sc.st));
    launch_mean_var(v_dev, P, part, n_part, stats, sc.st);
    launch_local_max(v_dev, g->n_lat, g->n_lon, stats, k_sigma, cands, n_c, kDetCap, sc.st);
    int hc = 0;
    CK(cudaMemcpyAsync(&hc, n_c, sizeof hc, cudaMemcpyDeviceToHost, sc.st));
    CK(cudaStreamSynchronize(sc.st));
    *launches += 6;
    *n_out = 0;
    if (hc == 0) return;
    if (hc > kDetCap) {  // every local maximum, host sort + exclusion
        auto* all = sc.alloc<DetCand>(hc);
        CK(cudaMemsetAsync(n_c, 0, sizeof(int), sc.st));
        launch_local_max(v_dev, g->n_lat, g->n_lon, stats, k_sigma, all, n_c, hc, sc.st);
        *launches += 1;
        std::vector<DetCand> h(hc);
        double hs[3];
        CK(cudaMemcpyAsync(h.data(), all, hc * sizeof(DetCand), cudaMemcpyDeviceToHost, sc.st));
        CK(cudaMemcpyAsync(hs, stats, sizeof hs, cudaMemcpyDeviceToHost, sc.st));
        CK(cudaStreamSynchronize(sc.st));
        std::vector<dg_emitter_estimate> d;
        greedy_host(h, radius, hs[0], hs[2], g->n_lon, d);
        *n_out = (int64_t)d.size();
        if (out && capacity > 0) {
            const int64_t m = std::min<int64_t>((int64_t)d.size(), capacity);
            std::copy(d.begin(), d.begin() + m, out);
            lattice_fill(g, out, m);
        }
        return;
    }
    launch_greedy(cands, n_c, kDetCap, radius, stats, g->n_lon, dets, n_c + 1, sc.st);
    CK(cudaGetLastError());
    *launches += 1;
    int nd = 0;
    CK(cudaMemcpyAsync(&nd, n_c + 1, sizeof nd, cudaMemcpyDeviceToHost, sc.st));
    CK(cudaStreamSynchronize(sc.st));
    *n_out = nd;
    if (out && capacity > 0) {
        const int64_t m = std::min<int64_t>(nd, capacity);
        CK(cudaMemcpyAsync(out, dets, m * sizeof(dg_emitter_estimate), cudaMemcpyDeviceToHost,
                           sc.st));
        CK(cudaStreamSynchronize(sc.st));
        lattice_fill(g, out, m);
    }
}

// Everything a run shares: pairs, per-(snapshot, pair) receiver states.
struct RunGeo {
    int S = 0, R = 0, pairs = 0, SP = 0;
    double fs = 0, wl = 0;
    std::vector<int> prx;
    std::vector<PairGeom> hpg;
    PairGeom* pg = nullptr;  // device [SP]
    int* d_prx = nullptr;    // device [2 * pairs]
};

RunGeo make_geo(Scratch& sc, const dg_staged* sn) {
    RunGeo r;
    r.S = (int)sn->S;
    r.R = (int)sn->R;
    r.pairs = r.R * (r.R - 1) / 2;
    r.SP = r.S * r.pairs;
    r.fs = sn->fs;
    r.wl = kC / sn->fc;
    for (int i = 0; i < r.R; ++i)
        for (int j = i + 1; j < r.R; ++j) {
            r.prx.push_back(i);
            r.prx.push_back(j);
        }
    r.hpg.resize(r.SP);
    for (int s = 0; s < r.S; ++s)
        for (int q = 0; q < r.pairs; ++q)
            r.hpg[s * r.pairs + q] = PairGeom{sn->states[s * r.R + r.prx[2 * q]],
                                              sn->states[s * r.R + r.prx[2 * q + 1]]};
    r.pg = sc.alloc<PairGeom>(r.SP);
    r.d_prx = sc.alloc<int>(r.prx.size());
    CK(cudaMemcpyAsync(r.pg, r.hpg.data(), r.SP * sizeof(PairGeom), cudaMemcpyHostToDevice, sc.st));
    CK(cudaMemcpyAsync(r.d_prx, r.prx.data(), r.prx.size() * sizeof(int), cudaMemcpyHostToDevice,
                       sc.st));
    // pageable sources: cudaMemcpyAsync has staged them when it returns
    return r;
}

RefineCtx refine_ctx(const dg_grid* g, const dg_staged* sn, const RunGeo& geo, double* raw) {
    RefineCtx ctx{};
    ctx.x = g->x;
    ctx.y = g->y;
    ctx.z = g->z;
    ctx.P = g->size();
    ctx.pg = geo.pg;
    ctx.pair_rx = geo.d_prx;
    ctx.pairs = geo.pairs;
    ctx.R = geo.R;
    ctx.y64 = static_cast<const double2*>(sn->y64->p) + kCapturePad;
    ctx.stride = sn->stride;
    ctx.N = (int)sn->N;
    ctx.fs = geo.fs;
    ctx.wl = geo.wl;
    ctx.raw = raw;
    return ctx;
}

// the per-call counters of a dg_result (the correlate phases add to them)
void reset_stats(dg_result* r) {
    r->n_refined = 0;
    r->n_reranked = 0;
    r->sum_overlap_samples = 0.0;
    r->correlate_ms = 0.0;
    r->correlate_launches = 0;
    r->total_ms = 0.0;
    r->kernel_launches = 0;
    r->moments_ms = 0.0;
    r->evaluate_ms = 0.0;
    r->moment_ffma2 = 0.0;
    r->evaluate_ffma2 = 0.0;
    r->direct_steps = 0;
    r->evaluate_tc_flop = 0.0;
    r->moment_fft_flop = 0.0;
}

dg_options options_or_default(const dg_options* o) {
    dg_options opt;
    if (o) {
        opt = *o;
    } else {
        dg_options_default(&opt);
    }
    return opt;
}

// the run's per-capture |y|^2 prefix sums, made on first use: behind the
// capture upload on the engine's upload stream when staging is still in flight
// (the correlator lanes wait for it with the captures), else on st; st (and so
// everything ordered after it) waits for them
const double* energy_prefix(const dg_staged* sn, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(sn->e_mu);
    if (!sn->e64) {
        cudaStream_t es = sn->ready ? sn->eng->upload : st;
        auto e = std::make_unique<DevMem>(sn->S * sn->R * (sn->N + 1) * sizeof(double));
        launch_energy_prefix(static_cast<const double2*>(sn->y64->p) + kCapturePad, sn->stride,
                             sn->S * sn->R, sn->N, static_cast<double*>(e->p), es);
        CK(cudaEventCreateWithFlags(&sn->e_ready, cudaEventDisableTiming));
        CK(cudaEventRecord(sn->e_ready, es));
        sn->e64 = std::move(e);
    }
    return static_cast<const double*>(sn->e64->p);
}

// Units over the whole grid g: geometry, correlation, exact refinement -> raw
// surfaces [n_units][P] (device). The step-sharded half of geolocate_snapshots
// and, with every step of a snapshot range, the
// single-GPU path.
void correlate_units_impl(dg_engine* eng, const dg_grid* g, const dg_staged* sn,
                          const RunGeo& geo, const std::vector<StepUnit>& units,
                          const dg_options& opt, double* raw, Scratch& sc, dg_result* res) {
    const int64_t P = g->size();
    const int pairs = geo.pairs, R = geo.R;
    const int SPl = (int)units.size();
    const double fs = geo.fs, wl = geo.wl;
    cudaStream_t st = sc.st;
    int64_t launches = 0;
    if (SPl <= 0) return;

    std::vector<cudaEvent_t> evs;
    if (opt.profile) {
        evs.resize(3 * SPl);
        for (auto& e : evs) CK(cudaEventCreate(&e));
    }
    struct EvFree {
        std::vector<cudaEvent_t>* v;
        ~EvFree() {
            for (auto e : *v) cudaEventDestroy(e);
        }
    } ev_free{&evs};

    // the units' receiver pairs and global step indices (refinement maps a
    // unit row back to its snapshot / pair)
    std::vector<PairGeom> hpg(SPl);
    std::vector<int> hstep(SPl);
    for (int u = 0; u < SPl; ++u) {
        if (units[u].sp < 0 || units[u].sp >= geo.SP || units[u].parts < 1 ||
            units[u].part < 0 || units[u].part >= units[u].parts)
            raise(DG_EINVAL, "dg_correlate_units: bad work unit");
        hpg[u] = geo.hpg[units[u].sp];
        hstep[u] = units[u].sp;
    }
    auto* ustep = sc.alloc<int>(SPl);
    CK(cudaMemcpyAsync(ustep, hstep.data(), SPl * sizeof(int), cudaMemcpyHostToDevice, st));

    Pipeline pl;
    pl.init(sc, eng, P, sn->N, SPl, opt.profile ? 1 : 2, eng->lane);
    const double* e64 = energy_prefix(sn, st);
    // the geometry pass's receiver-group tables, one per 64 units of a window
    std::vector<GeoScratch> geo_ws((pl.slots + 63) / 64);
    for (auto& w : geo_ws) {
        w.d_rx = sc.alloc<dg_state>(128);
        w.d_groups = sc.alloc<GeoGroup>(64);
        w.d_upair = sc.alloc<int2>(64);
    }
    // refine flags: one bitmap row of whole words per unit (bit p of unit i at
    // i * P32 + p), so batches of units are refined on a side stream while the
    // lanes correlate later units (FP64 refinement next to FP32 correlation)
    const int64_t P32 = (P + 31) & ~int64_t(31);
    const int64_t n_words = SPl * (P32 / 32);
    const auto* y32 = static_cast<const float2*>(sn->y32->p) + kCapturePad;
    const auto* y64 = static_cast<const double2*>(sn->y64->p) + kCapturePad;
    RefineCtx ctx = refine_ctx(g, sn, geo, raw);  // element = unit row * P + p
    ctx.unit_step = ustep;
    for (int u = 0; u < SPl; ++u)  // parts: candidates of the other parts stay 0
        if (units[u].parts > 1)
            CK(cudaMemsetAsync(raw + (int64_t)u * P, 0, P * sizeof(double), st));
    uint32_t* bits = nullptr;
    std::unique_ptr<SideRefine> rfp;

    for (int w0 = 0; w0 < SPl; w0 += pl.slots) {
        const int nw = std::min(pl.slots, SPl - w0);
        // phase A: geometry of the whole window in one pass; bins from the
        // histograms, B / R / centre frequency from the FP32 lattice ranges
        if (w0 > 0) CK(cudaMemsetAsync(pl.hist, 0, sizeof(int) * pl.nbins * nw, st));
        launch_geometry_units(g->x, g->y, g->z, P, hpg.data() + w0, nw, fs, wl, pl.N,
                              pl.d_slot(0), pl.rank_slot(0), pl.fdoa_slot(0), pl.hist_slot(0),
                              pl.nbins, raw + (int64_t)w0 * P, pl.overlap, pl.err, geo_ws.data(),
                              st);
        launch_hist_range(pl.hist_slot(0), pl.nbins, nw, pl.N, pl.range, st);
        launches += (nw + 63) / 64 + 2;
        if (w0 == 0) {  // the rest of the run's state, while the first geometry pass runs
            pl.init_lanes(sc);
            bits = sc.alloc<uint32_t>(n_words);
            CK(cudaMemsetAsync(bits, 0, n_words * sizeof(uint32_t), st));
            rfp = std::make_unique<SideRefine>(sc, SPl, P, P32, opt.profile ? 0 : 10, eng->refine);
        }
        SideRefine& rf = *rfp;
        const PairGeom* hw = hpg.data() + w0;
        const StepRange* approx = pl.lattice_ranges(sc, g, hw, nw, fs, wl);
        std::vector<StepUnit> wunits(units.begin() + w0, units.begin() + w0 + nw);
        pl.plan_window(sc, nw, fs, approx, fp32_fdoa_margin(hw, nw, wl), g->full_size,
                       /*exact_ranges=*/false, &wunits);
        if (w0 == 0) {  // captures still uploading / their energy sums
            if (sn->ready) pl.wait_event(sn->ready);
            pl.wait_event(sn->e_ready);
        }
        for (int i = 0; i < nw; ++i) {  // phase B: bucket + correlate each unit
            const int lsp = w0 + i, sp = units[lsp].sp;
            const int s = sp / pairs, q = sp - s * pairs;
            const int64_t c1 = ((int64_t)s * R + geo.prx[2 * q]) * sn->stride;
            const int64_t c2 = ((int64_t)s * R + geo.prx[2 * q + 1]) * sn->stride;
            const int64_t r1 = (int64_t)s * R + geo.prx[2 * q], r2 = (int64_t)s * R + geo.prx[2 * q + 1];
            pl.correlate(i, y64 + c1, y32 + c1, y32 + c2, e64 + r1 * (sn->N + 1),
                         e64 + r2 * (sn->N + 1), fs, raw + (int64_t)lsp * P, bits,
                         (int64_t)lsp * P32, opt.profile ? evs[3 * lsp] : nullptr,
                         opt.profile ? evs[3 * lsp + 1] : nullptr,
                         opt.profile ? evs[3 * lsp + 2] : nullptr);
            rf.step_done(lsp, pl.lane_stream(i), bits, ctx);
        }
        pl.join(sc);  // the next window reuses the d / fdoa / histogram slots
    }
    launches += pl.launches;
    CK(cudaGetLastError());

    SideRefine& rf = *rfp;
    rf.finish(bits, ctx);  // remaining units; the main stream joins the side stream
    launches += rf.launches;

    // the run's counters in one read-back (no host round trip before the last
    // refinement batch is queued): error flag, overlap, work per lane, refined
    // elements per batch
    std::vector<unsigned long long> hc(2 + 3 * pl.n_lanes + std::max(rf.batches, 1), 0ull);
    int herr = 0;
    CK(cudaMemcpyAsync(&herr, pl.err, sizeof herr, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hc.data(), pl.overlap, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       st));
    for (int l = 0; l < pl.n_lanes; ++l)
        CK(cudaMemcpyAsync(hc.data() + 2 + 3 * l, pl.lanes[l].work, 3 * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, st));
    const size_t c0 = 2 + 3 * (size_t)pl.n_lanes;
    CK(cudaMemcpyAsync(hc.data() + c0, rf.counts, (hc.size() - c0) * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (herr) raise(DG_EINVAL, "predict_geometry: candidate coincides with receiver");
    unsigned long long work[3] = {0, 0, 0}, refined = 0;
    for (int l = 0; l < pl.n_lanes; ++l)
        for (int k = 0; k < 3; ++k) work[k] += hc[2 + 3 * l + k];
    for (size_t i = c0; i < hc.size(); ++i) refined += hc[i];
    res->n_refined += (int64_t)refined;
    res->sum_overlap_samples += (double)hc[0];
    res->kernel_launches += launches;
    res->correlate_launches += SPl;
    res->moment_ffma2 += (double)work[0];
    res->evaluate_ffma2 += (double)work[1];
    res->evaluate_tc_flop += (double)work[2];
    res->direct_steps += pl.direct_steps;
    res->moment_fft_flop += pl.fft_flop;
    if (opt.profile) {
        double tm = 0.0, te = 0.0;
        for (int i = 0; i < SPl; ++i) {
            float a = 0.f, b = 0.f;
            CK(cudaEventElapsedTime(&a, evs[3 * i], evs[3 * i + 1]));
            CK(cudaEventElapsedTime(&b, evs[3 * i + 1], evs[3 * i + 2]));
            tm += a;
            te += b;
        }
        res->moments_ms += tm;
        res->evaluate_ms += te;
        res->correlate_ms += tm + te;
    }
}

// Snapshots [s0, s1) over the whole grid g: every pair of each (the units of
// the snapshot range), pair sums (correlate_snapshot_all_pairs) and the
// optional median scaling -> grids [(s1-s0)][P] (device), medians [s1-s0].
void correlate_steps_impl(dg_engine* eng, const dg_grid* g, const dg_staged* sn,
                          const RunGeo& geo, int s0, int s1, const dg_options& opt, double* grids,
                          double* medians, Scratch& sc, dg_result* res) {
    const int64_t P = g->size();
    const int pairs = geo.pairs;
    const int ns = s1 - s0;
    cudaStream_t st = sc.st;
    if (ns <= 0) return;
    std::vector<StepUnit> units(ns * pairs);
    for (int i = 0; i < ns * pairs; ++i) units[i].sp = s0 * pairs + i;
    double* raw = pairs == 1 ? grids : sc.alloc<double>((int64_t)ns * pairs * P);
    correlate_units_impl(eng, g, sn, geo, units, opt, raw, sc, res);
    int64_t launches = 0;
    if (pairs > 1) {
        launch_combine_pairs(raw, ns, pairs, P, grids, st);
        launches += 1;
    }
    if (opt.normalize_per_snapshot) {
        auto* hist = sc.alloc<unsigned>(256);
        auto* state = sc.alloc<unsigned long long>(2 * ns);
        std::vector<unsigned long long> init(2 * ns);
        for (int s = 0; s < ns; ++s) {
            init[2 * s] = 0ull;
            init[2 * s + 1] = (unsigned long long)(P / 2);
        }
        CK(cudaMemcpyAsync(state, init.data(), init.size() * sizeof(unsigned long long),
                           cudaMemcpyHostToDevice, st));
        CK(cudaMemsetAsync(hist, 0, 256 * sizeof(unsigned), st));
        for (int s = 0; s < ns; ++s) {
            launch_median(grids + (int64_t)s * P, P, hist, state + 2 * s, medians + s, st);
            launch_scale(grids + (int64_t)s * P, P, medians + s, st);
            launches += 17;
        }
        CK(cudaStreamSynchronize(st));  // `init` is host memory of this frame
    }
    res->kernel_launches += launches;
}

// dg_shard_plan (b200geo.h): whole steps in contiguous blocks, the remainder
// steps split into `world` bucket-range parts, one per rank.
std::vector<dg_work_unit> shard_plan(int64_t S, int64_t pairs, int world, bool whole) {
    std::vector<dg_work_unit> u;
    if (whole) {
        for (int r = 0; r < world; ++r)
            for (int64_t s = r * S / world; s < (r + 1) * S / world; ++s)
                u.push_back(dg_work_unit{s, 0, 1, r, 0});
        return u;
    }
    const int64_t steps = S * pairs, q = steps / world;
    for (int r = 0; r < world; ++r) {
        for (int64_t sp = r * q; sp < (r + 1) * q; ++sp) u.push_back(dg_work_unit{sp, 0, 1, r, 0});
        for (int64_t sp = world * q; sp < steps; ++sp)
            u.push_back(dg_work_unit{sp, r, world, r, 0});
    }
    return u;
}

// Accumulation over ALL S snapshots of grid g (a slab or the full lattice)
// from per-snapshot grids [S][P] (device), then the exact peak (near-peak
// cells re-evaluated in FP64 for every (snapshot, pair)), detection and the
// host copies — the other half of geolocate_snapshots.

// stream `st` waits for the work queued so far on two side streams
struct SideJoin {
    cudaStream_t st, side[2];
    cudaEvent_t e[2] = {nullptr, nullptr};
    SideJoin(cudaStream_t s, cudaStream_t a, cudaStream_t b) : st(s), side{a, b} {
        for (auto& x : e) CK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    }
    void join() {
        for (int i = 0; i < 2; ++i) {
            CK(cudaEventRecord(e[i], side[i]));
            CK(cudaStreamWaitEvent(st, e[i], 0));
        }
    }
    ~SideJoin() {
        for (int i = 0; i < 2; ++i) {
            if (cudaEventRecord(e[i], side[i]) == cudaSuccess) cudaStreamWaitEvent(st, e[i], 0);
            cudaEventDestroy(e[i]);
        }
    }
};

// The exact peak. Every unrefined element meets |fast - exact| <= eps exact
// (eps = 1e-4, the per-element contract; refined elements are FP64), so with
// all terms non-negative every accumulated value does too, and the true argmax
// c* satisfies fast(c*) >= exact(c*)(1 - eps) >= M (1 - eps) / (1 + eps), M the
// fast maximum. Every cell at or above that threshold is re-evaluated with the
// reference's FP64 recurrence for all (snapshot, pair) steps and recombined in
// the reference's order; the exact maximum (lowest flat index on ties, as
// std::max_element) over them is the reference's argmax. Past kRerankRound
// cells they are re-ranked in rounds in descending fast order, stopping once
// the best exact value exceeds fast(next) / (1 - eps) >= exact(any later cell).
constexpr double kPeakEps = 1e-4;
// per-snapshot surfaces held at once when the caller does not want them: past
// this the run is solved in chunks of snapshots (C5: 16M cells x 100 snapshots
// would be 12.8 GB)
constexpr int64_t kSurfaceBudget = 4ll << 30;
constexpr int kRerankRound = 4096;

struct PeakCells {
    int n = 0;                   // re-ranked cells
    int* cells = nullptr;        // [n] device, in re-rank order
    double* acc_ex = nullptr;    // [n] exact accumulated values
    double* grid_ex = nullptr;   // [n][S] exact per-snapshot values
    long long best_i = -1;
    double best_v = 0.0;
};

PeakCells exact_peak(const dg_grid* g, const dg_staged* sn, const RunGeo& geo, const double* acc,
                     const double* medians, double M, Scratch& sc, int64_t* launches) {
    const int64_t P = g->size();
    const int S = geo.S, SP = geo.SP, pairs = geo.pairs;
    cudaStream_t st = sc.st;
    PeakCells pk;
    const double thr = M * (1.0 - kPeakEps) / (1.0 + kPeakEps);
    auto* cnt = sc.alloc<unsigned long long>(1);
    CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st));
    launch_count_ge(acc, P, thr, cnt, st);
    unsigned long long hc = 0;
    CK(cudaMemcpyAsync(&hc, cnt, sizeof hc, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *launches += 1;
    if (hc == 0) return pk;
    const int n = (int)hc;
    const size_t tb = select_ge_temp_bytes(P, n);
    void* temp = sc.alloc<unsigned char>(tb);
    int* sel = sc.alloc<int>(n);
    auto* n_sel = sc.alloc<int>(1);
    launch_select_ge(acc, P, thr, sel, n_sel, temp, tb, st);
    *launches += 1;
    int* order = sel;
    if (n > kRerankRound) {  // rounds in descending fast value
        auto* keys = sc.alloc<unsigned long long>(2 * (size_t)n);
        order = sc.alloc<int>(n);
        launch_sort_by_value(acc, sel, n, keys, keys + n, order, temp, tb, st);
        *launches += 2;
    }
    RefineCtx ctx = refine_ctx(g, sn, geo, nullptr);
    auto* ex = sc.alloc<double>((int64_t)std::min(n, kRerankRound) * SP);
    pk.acc_ex = sc.alloc<double>(n);
    pk.grid_ex = sc.alloc<double>((int64_t)n * S);
    auto* n_batch = sc.alloc<int>(1);
    auto* best_i = sc.alloc<long long>(1);
    auto* best_v = sc.alloc<double>(1);
    std::vector<double> next_fast(1);
    // each chain's phasor start and step from the host's libm, as the reference
    // computes them (correlate.hpp:51-54), so the FP64 chains are bit-identical
    const int chains_max = std::min(n, kRerankRound) * SP;
    auto* offs = sc.alloc<dg_pair_offsets>(chains_max);
    auto* trig = sc.alloc<double>(4 * (size_t)chains_max);
    std::vector<dg_pair_offsets> h_offs(chains_max);
    std::vector<double> h_trig(4 * (size_t)chains_max);
    ctx.trig = trig;
    for (int r0 = 0; r0 < n; r0 += kRerankRound) {
        const int m = std::min(kRerankRound, n - r0);
        launch_chain_offsets(order + r0, m, SP, ctx, offs, st);
        CK(cudaMemcpyAsync(h_offs.data(), offs, (size_t)m * SP * sizeof(dg_pair_offsets),
                           cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int64_t i = 0; i < (int64_t)m * SP; ++i) {
            const int64_t d = h_offs[i].tdoa_samples;
            const int64_t kb = std::max<int64_t>(0, -d);
            const double step = 2.0 * std::numbers::pi * h_offs[i].fdoa_hz / geo.fs;
            const double phase0 = step * static_cast<double>(kb);
            double* t = h_trig.data() + 4 * i;
            t[0] = std::cos(step);
            t[1] = std::sin(step);
            t[2] = std::cos(phase0);
            t[3] = std::sin(phase0);
        }
        CK(cudaMemcpyAsync(trig, h_trig.data(), 4 * (size_t)m * SP * sizeof(double),
                           cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(n_batch, &m, sizeof m, cudaMemcpyHostToDevice, st));
        launch_rerank(order + r0, n_batch, m, m, SP, ctx, ex, st);
        launch_recombine_cells(n_batch, m, ex, S, pairs, medians, pk.acc_ex + r0,
                               pk.grid_ex + (int64_t)r0 * S, st);
        launch_argmax_cells(order + r0, n_batch, m, pk.acc_ex + r0, best_i, best_v, st);
        *launches += 3;
        long long bi = 0;
        double bv = 0.0;
        CK(cudaMemcpyAsync(&bi, best_i, sizeof bi, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&bv, best_v, sizeof bv, cudaMemcpyDeviceToHost, st));
        const bool more = r0 + m < n;
        int next_cell = 0;
        if (more)
            CK(cudaMemcpyAsync(&next_cell, order + r0 + m, sizeof next_cell,
                               cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));  // m is host memory of this frame
        if (pk.best_i < 0 || bv > pk.best_v || (bv == pk.best_v && bi < pk.best_i)) {
            pk.best_i = bi;
            pk.best_v = bv;
        }
        pk.n = r0 + m;
        if (!more) break;
        CK(cudaMemcpyAsync(next_fast.data(), acc + next_cell, sizeof(double),
                           cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (pk.best_v > next_fast[0] / (1.0 - kPeakEps)) break;  // no later cell can reach it
    }
    pk.cells = order;
    return pk;
}

// per_pitch: elements between snapshot rows of the host per_snapshot buffer
// (0: P; a slab of a multi-GPU run writes its columns of the full rows)
// acc_in (nullable): the surface already accumulated (chunked runs), else
// accumulate `grids`
void peak_impl(dg_engine* eng, const dg_grid* g, const dg_staged* sn, const RunGeo& geo,
               const double* grids, const double* medians, const dg_options& opt,
               bool acc_dev_allowed, dg_result* res, Scratch& sc, int64_t per_pitch = 0,
               double* acc_in = nullptr) {
    const int64_t P = g->size();
    if (per_pitch == 0) per_pitch = P;
    const int S = geo.S;
    cudaStream_t st = sc.st;
    int64_t launches = 0;
    if (opt.peak_stage < 0 || opt.peak_stage > 2) raise(DG_EINVAL, "dg_options: bad peak_stage");
    if (opt.peak_stage == 2 && !res->accumulated_device)
        raise(DG_EINVAL, "dg_options: peak_stage 2 needs the surface in accumulated_device");
    if (!(opt.peak_max >= 0.0)) raise(DG_EINVAL, "dg_options: peak_max < 0");
    double* acc = acc_in ? acc_in
                  : acc_dev_allowed && res->accumulated_device ? res->accumulated_device
                                                               : sc.alloc<double>(P);
    if (opt.peak_stage != 2 && !acc_in) {
        launch_accumulate(grids, S, P, acc, st);
        launches += 1;
    }
    const int64_t base = g->row_offset * g->n_lon;  // flat index of this grid's first cell
    const bool patch = opt.patch_peak && opt.peak_stage != 1;
    // the fast surfaces' device->host copies (engine refine stream) run beside
    // the latency-bound exact re-rank; the re-ranked values are patched into
    // the host copies afterwards and into the device surface before detection
    cudaEvent_t acc_done, patched;
    CK(cudaEventCreateWithFlags(&acc_done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&patched, cudaEventDisableTiming));
    struct EvGuard {
        cudaEvent_t a, b;
        ~EvGuard() {
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
    } ev_guard{acc_done, patched};
    CK(cudaEventRecord(acc_done, st));
    cudaStream_t d2h = eng->refine, det = eng->lane;
    CK(cudaStreamWaitEvent(d2h, acc_done, 0));
    if (res->accumulated)
        CK(cudaMemcpyAsync(res->accumulated, acc, P * sizeof(double), cudaMemcpyDeviceToHost,
                           d2h));
    if (res->per_snapshot && grids)
        CK(cudaMemcpy2DAsync(res->per_snapshot, per_pitch * sizeof(double), grids,
                             P * sizeof(double), P * sizeof(double), S, cudaMemcpyDeviceToHost,
                             d2h));
    // `acc` / `grids` are freed on st when the caller's scratch goes: st waits
    // for these readers before returning (also when an error unwinds)
    SideJoin sj(st, d2h, det);

    const int n_part = 148 * 4;
    auto* part = sc.alloc<double>(n_part);
    auto* vmax = sc.alloc<double>(1);
    launch_max(acc, P, part, n_part, vmax, st);
    launches += 2;
    double hmax = 0.0;
    CK(cudaMemcpyAsync(&hmax, vmax, sizeof hmax, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    PeakCells pk;
    if (opt.peak_stage == 1) {  // fast maximum only (sharded runs, before peak_max is known)
        auto* fi = sc.alloc<unsigned long long>(1);
        CK(cudaMemsetAsync(fi, 0xff, sizeof(unsigned long long), st));
        launch_first_max(acc, P, vmax, fi, st);
        launches += 1;
        unsigned long long hi = 0;
        CK(cudaMemcpyAsync(&hi, fi, sizeof hi, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        res->argmax_index = (int64_t)hi + base;
        res->argmax_value = hmax;
    } else {
        const double M = opt.peak_max > 0.0 ? opt.peak_max : hmax;
        if (opt.peak_max > 0.0 && hmax > opt.peak_max)
            raise(DG_EINVAL, "dg_options: peak_max below this surface's maximum");
        if (M > 0.0) {
            pk = exact_peak(g, sn, geo, acc, medians, M, sc, &launches);
            res->argmax_index = pk.best_i >= 0 ? pk.best_i + base : -1;
            res->argmax_value = pk.best_i >= 0 ? pk.best_v : 0.0;
        } else {
            // all-zero surface (no overlap / silent captures): first index wins
            res->argmax_index = base;
            res->argmax_value = hmax;
        }
        if (patch && pk.n > 0) {
            launch_patch_cells(pk.cells, pk.n, pk.acc_ex, acc, st);
            launches += 1;
        }
    }
    res->n_reranked = pk.n;
    CK(cudaEventRecord(patched, st));
    CK(cudaStreamWaitEvent(det, patched, 0));
    res->n_detections = 0;
    if (opt.detect && opt.peak_stage != 1) {
        Scratch sd(det);
        run_detect(g, acc, opt.k_sigma, opt.exclusion_radius_cells, res->detections,
                   res->detections_capacity, &res->n_detections, sd, &launches);
    }

    sj.join();
    CK(cudaStreamSynchronize(st));
    if (patch && pk.n > 0 && (res->accumulated || res->per_snapshot)) {
        // exact FP64 values of the re-ranked cells into the host copies
        const int n = pk.n;
        std::vector<int> hc(n);
        std::vector<double> ha(n), hg((size_t)n * S);
        CK(cudaMemcpyAsync(hc.data(), pk.cells, n * sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(ha.data(), pk.acc_ex, n * sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hg.data(), pk.grid_ex, (size_t)n * S * sizeof(double),
                           cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int i = 0; i < n; ++i) {
            if (res->accumulated) res->accumulated[hc[i]] = ha[i];
            if (res->per_snapshot && grids)
                for (int s = 0; s < S; ++s)
                    res->per_snapshot[(int64_t)s * per_pitch + hc[i]] = hg[(size_t)i * S + s];
        }
    }
    res->kernel_launches += launches;
}

void check_run(const dg_engine* eng, const dg_grid* g, const dg_staged* sn, const dg_options& opt,
               const void* res) {
    if (!eng || !g || !sn || !res) raise(DG_EINVAL, "null argument");
    if (g->size() == 0) raise(DG_EINVAL, "correlate_snapshot: empty grid");
    if (opt.exclusion_radius_cells < 0)
        raise(DG_EINVAL, "detect_emitters: negative exclusion radius");
}

void geolocate_impl(dg_engine* eng, const dg_grid* g, const dg_staged* sn, const dg_options* opt_in,
                    dg_result* res) {
    const dg_options opt = options_or_default(opt_in);
    check_run(eng, g, sn, opt, res);
    set_device(eng);
    StreamGuard sg(opt.stream, eng->stream);
    Scratch sc(sg.st, &eng->arena);
    reset_stats(res);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (opt.profile) {
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, sc.st));
    }
    const RunGeo geo = make_geo(sc, sn);
    const int64_t P = g->size();
    double* medians = opt.normalize_per_snapshot ? sc.alloc<double>(geo.S) : nullptr;
    int64_t budget = kSurfaceBudget;
    {
        std::lock_guard<std::mutex> lk(eng->tables_mu);
        if (eng->tuning.surface_budget_bytes > 0) budget = eng->tuning.surface_budget_bytes;
    }
    const int64_t chunk = std::max<int64_t>(1, budget / (P * (int64_t)sizeof(double)));
    if (res->per_snapshot || chunk >= geo.S) {
        auto* grids = sc.alloc<double>((int64_t)geo.S * P);
        correlate_steps_impl(eng, g, sn, geo, 0, geo.S, opt, grids, medians, sc, res);
        peak_impl(eng, g, sn, geo, grids, medians, opt, opt_in != nullptr, res, sc);
    } else {
        // per-snapshot surfaces not wanted and over budget: snapshots in chunks,
        // each added to the running accumulated surface in snapshot order
        // (bit-identical to accumulating them all at once)
        double* acc = opt_in != nullptr && res->accumulated_device ? res->accumulated_device
                                                                   : sc.alloc<double>(P);
        auto* grids = sc.alloc<double>(chunk * P);
        dg_result part{};
        for (int s0 = 0; s0 < geo.S; s0 += (int)chunk) {
            const int s1 = std::min<int>(geo.S, s0 + (int)chunk);
            reset_stats(&part);
            correlate_steps_impl(eng, g, sn, geo, s0, s1, opt, grids,
                                 medians ? medians + s0 : nullptr, sc, &part);
            launch_accumulate(grids, s1 - s0, P, acc, sc.st, s0 == 0);
            res->n_refined += part.n_refined;
            res->sum_overlap_samples += part.sum_overlap_samples;
            res->kernel_launches += part.kernel_launches + 1;
            res->correlate_launches += part.correlate_launches;
            res->moment_ffma2 += part.moment_ffma2;
            res->evaluate_ffma2 += part.evaluate_ffma2;
            res->evaluate_tc_flop += part.evaluate_tc_flop;
            res->direct_steps += part.direct_steps;
            res->moment_fft_flop += part.moment_fft_flop;
            res->moments_ms += part.moments_ms;
            res->evaluate_ms += part.evaluate_ms;
            res->correlate_ms += part.correlate_ms;
        }
        peak_impl(eng, g, sn, geo, nullptr, medians, opt, opt_in != nullptr, res, sc, 0, acc);
    }
    if (opt.profile) {
        CK(cudaEventRecord(e1, sc.st));
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        res->total_ms = ms;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
}

// ---- multi-GPU engine (dg_engine_create_multi) --------------------------------
// The rows [r0, r1) of a grid as a grid of its own (flat indices stay global).
dg_grid slab_view(const dg_grid& g, int64_t r0, int64_t r1) {
    dg_grid s = g;
    s.replicas = std::make_shared<Replicas<dg_grid>>();
    s.n_lat = r1 - r0;
    s.row_offset = g.row_offset + r0;
    s.x = g.x + r0 * g.n_lon;
    s.y = g.y + r0 * g.n_lon;
    s.z = g.z + r0 * g.n_lon;
    return s;
}

// g's cells (and its full FP32 planning lattice) on engine e's device
const dg_grid* grid_on(const dg_grid* g, const dg_engine* e) {
    if (g->eng == e) return g;
    std::lock_guard<std::mutex> lk(g->replicas->mu);
    for (auto& [k, v] : g->replicas->v)
        if (k == e) return v.get();
    set_device(e);
    auto r = std::make_unique<dg_grid>(slab_view(*g, 0, g->n_lat));
    r->eng = const_cast<dg_engine*>(e);
    r->row_offset = g->row_offset;
    const int64_t P = g->size();
    r->mem = std::make_shared<DevMem>(3 * P * sizeof(double));
    double* base = static_cast<double*>(r->mem->p);
    CK(cudaMemcpyPeer(base, e->device, g->x, g->eng->device, P * sizeof(double)));
    CK(cudaMemcpyPeer(base + P, e->device, g->y, g->eng->device, P * sizeof(double)));
    CK(cudaMemcpyPeer(base + 2 * P, e->device, g->z, g->eng->device, P * sizeof(double)));
    r->x = base;
    r->y = base + P;
    r->z = base + 2 * P;
    r->rel = std::make_shared<DevMem>(g->rel->bytes);
    CK(cudaMemcpyPeer(r->rel->p, e->device, g->rel->p, g->eng->device, g->rel->bytes));
    const dg_grid* out = r.get();
    g->replicas->v.emplace_back(e, std::move(r));
    return out;
}

const dg_staged* staged_on(const dg_staged* s, const dg_engine* e) {
    if (s->eng == e) return s;
    std::lock_guard<std::mutex> lk(s->replicas->mu);
    for (auto& [k, v] : s->replicas->v)
        if (k == e) return v.get();
    if (s->ready) CK(cudaEventSynchronize(s->ready));
    set_device(e);
    auto r = std::make_unique<dg_staged>();
    r->eng = const_cast<dg_engine*>(e);
    r->S = s->S;
    r->R = s->R;
    r->N = s->N;
    r->stride = s->stride;
    r->fs = s->fs;
    r->fc = s->fc;
    r->states = s->states;
    r->y32 = std::make_unique<DevMem>(s->y32->bytes);
    r->y64 = std::make_unique<DevMem>(s->y64->bytes);
    CK(cudaMemcpyPeer(r->y32->p, e->device, s->y32->p, s->eng->device, s->y32->bytes));
    CK(cudaMemcpyPeer(r->y64->p, e->device, s->y64->p, s->eng->device, s->y64->bytes));
    const dg_staged* out = r.get();
    s->replicas->v.emplace_back(e, std::move(r));
    return out;
}

// run f(k) on one host thread per device; the first exception is rethrown
template <class F>
void on_devices(int G, F&& f) {
    std::vector<std::exception_ptr> err(G);
    std::vector<std::thread> th;
    for (int k = 0; k < G; ++k)
        th.emplace_back([&, k] {
            try {
                f(k);
            } catch (...) {
                err[k] = std::current_exception();
            }
        });
    for (auto& t : th) t.join();
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}

// geolocate_snapshots over every device of a multi-GPU engine (DESIGN.md
// section 7): the run's work units (dg_shard_plan) are correlated on their
// devices (no communication), every unit's slab columns go by peer copy
// (NVLink) to the device owning that latitude slab, which sums the parts of a
// step (exact: disjoint candidates), adds the pairs and accumulates its slab
// over all snapshots in the reference's order — every accumulated value is
// bit-identical to the one-GPU solve. The exact peak re-ranks the cells above
// the band of the global fast maximum on every slab (two-stage peak), and
// detection runs on device 0 over the gathered surface.
void geolocate_multi(dg_engine* eng, const dg_grid* g, const dg_staged* sn,
                     const dg_options* opt_in, dg_result* res) {
    const dg_options opt = options_or_default(opt_in);
    check_run(eng, g, sn, opt, res);
    if (opt.profile) raise(DG_EINVAL, "b200: profiled runs use one device");
    reset_stats(res);
    const int G = eng->n_devices();
    const int64_t P = g->size(), n_lon = g->n_lon, n_lat = g->n_lat;
    const int S = (int)sn->S, R = (int)sn->R, pairs = R * (R - 1) / 2;
    const bool whole = opt.normalize_per_snapshot != 0;
    const auto plan = shard_plan(S, pairs, G, whole);
    const int U = (int)plan.size();
    std::vector<std::vector<int>> mine(G);  // plan indices of each device's units
    for (int u = 0; u < U; ++u) mine[plan[u].rank].push_back(u);
    std::vector<int64_t> r0(G), r1(G);
    for (int k = 0; k < G; ++k) {
        r0[k] = k * n_lat / G;
        r1[k] = (k + 1) * n_lat / G;
    }
    std::vector<std::unique_ptr<Scratch>> scr(G);
    std::vector<RunGeo> geo(G);
    std::vector<const dg_grid*> gk(G);
    std::vector<const dg_staged*> sk(G);
    std::vector<double*> out(G, nullptr), med(G, nullptr);
    std::vector<dg_result> part(G);
    // phase 1: each device correlates its units over the whole grid
    on_devices(G, [&](int k) {
        dg_engine* e = eng->dev(k);
        set_device(e);
        gk[k] = grid_on(g, e);
        sk[k] = staged_on(sn, e);
        scr[k] = std::make_unique<Scratch>(e->stream, &e->arena);
        Scratch& sc = *scr[k];
        geo[k] = make_geo(sc, sk[k]);
        std::memset(&part[k], 0, sizeof(dg_result));
        const int n = (int)mine[k].size();
        out[k] = sc.alloc<double>((int64_t)std::max(n, 1) * P);
        if (whole) {  // contiguous snapshots, pair sums and median scaling on the device
            med[k] = sc.alloc<double>(std::max(n, 1));
            if (n > 0)
                correlate_steps_impl(e, gk[k], sk[k], geo[k], (int)plan[mine[k][0]].step,
                                     (int)plan[mine[k][0]].step + n, opt, out[k], med[k], sc,
                                     &part[k]);
        } else if (n > 0) {
            std::vector<StepUnit> u(n);
            for (int i = 0; i < n; ++i) {
                const dg_work_unit& w = plan[mine[k][i]];
                u[i] = StepUnit{(int)w.step, w.part, w.parts};
            }
            correlate_units_impl(e, gk[k], sk[k], geo[k], u, opt, out[k], sc, &part[k]);
        }
        CK(cudaStreamSynchronize(sc.st));
    });
    // phase 2: slab j gathers its columns of every unit (peer copies), then the
    // per-snapshot slab surfaces [S][slab] in the reference's pair / step order
    std::vector<double*> grids(G, nullptr), meds(G, nullptr);
    std::vector<int> local_idx(U);
    for (int k = 0; k < G; ++k)
        for (int i = 0; i < (int)mine[k].size(); ++i) local_idx[mine[k][i]] = i;
    on_devices(G, [&](int j) {
        dg_engine* e = eng->dev(j);
        set_device(e);
        Scratch& sc = *scr[j];
        const int64_t slab = (r1[j] - r0[j]) * n_lon, c0 = r0[j] * n_lon;
        if (slab == 0) return;
        const int rows = whole ? S : U;
        double* recv = sc.alloc<double>((int64_t)rows * slab);
        for (int u = 0; u < U; ++u) {
            const int k = plan[u].rank;
            const int dst_row = whole ? (int)plan[u].step : u;
            CK(cudaMemcpyPeerAsync(recv + (int64_t)dst_row * slab, e->device,
                                   out[k] + (int64_t)local_idx[u] * P + c0, eng->dev(k)->device,
                                   slab * sizeof(double), sc.st));
        }
        if (whole) {
            grids[j] = recv;
            meds[j] = sc.alloc<double>(S);
            for (int u = 0; u < U; ++u)
                CK(cudaMemcpyPeerAsync(meds[j] + plan[u].step, e->device,
                                       med[plan[u].rank] + local_idx[u],
                                       eng->dev(plan[u].rank)->device, sizeof(double), sc.st));
            return;
        }
        // the parts of a step hold disjoint candidates: their sum is exact in
        // any order; then the pairs in the reference's order
        std::vector<int> hstep(U);
        for (int u = 0; u < U; ++u) hstep[u] = (int)plan[u].step;
        int* ustep = sc.alloc<int>(U);
        CK(cudaMemcpyAsync(ustep, hstep.data(), U * sizeof(int), cudaMemcpyHostToDevice, sc.st));
        double* steps = sc.alloc<double>((int64_t)S * pairs * slab);
        CK(cudaMemsetAsync(steps, 0, (int64_t)S * pairs * slab * sizeof(double), sc.st));
        launch_sum_units(recv, U, slab, ustep, steps, sc.st);
        if (pairs == 1) {
            grids[j] = steps;
        } else {
            grids[j] = sc.alloc<double>((int64_t)S * slab);
            launch_combine_pairs(steps, S, pairs, slab, grids[j], sc.st);
        }
        CK(cudaStreamSynchronize(sc.st));  // hstep is host memory of this frame
    });
    // phase 3: accumulation and the fast maximum of every slab
    std::vector<dg_grid> slabs;
    for (int k = 0; k < G; ++k) slabs.push_back(slab_view(*gk[k], r0[k], r1[k]));
    std::vector<double*> acc(G, nullptr);
    std::vector<dg_result> pr(G);
    dg_options o1 = opt;
    o1.stream = nullptr;
    o1.detect = 0;
    o1.peak_stage = 1;
    on_devices(G, [&](int j) {
        if (slabs[j].size() == 0) return;
        dg_engine* e = eng->dev(j);
        set_device(e);
        Scratch& sc = *scr[j];
        acc[j] = sc.alloc<double>(slabs[j].size());
        std::memset(&pr[j], 0, sizeof(dg_result));
        pr[j].accumulated_device = acc[j];
        peak_impl(e, &slabs[j], sk[j], geo[j], grids[j], whole ? meds[j] : nullptr, o1, true,
                  &pr[j], sc);
    });
    double M = 0.0;
    for (int j = 0; j < G; ++j)
        if (slabs[j].size() > 0) M = std::max(M, pr[j].argmax_value);
    // phase 4: exact peak of every slab against the global band, host copies
    dg_options o2 = o1;
    o2.peak_stage = 2;
    o2.peak_max = M;
    on_devices(G, [&](int j) {
        if (slabs[j].size() == 0) return;
        dg_engine* e = eng->dev(j);
        set_device(e);
        Scratch& sc = *scr[j];
        dg_result& r = pr[j];
        const int64_t c0 = r0[j] * n_lon;
        r.accumulated = res->accumulated ? res->accumulated + c0 : nullptr;
        r.per_snapshot = res->per_snapshot ? res->per_snapshot + c0 : nullptr;
        peak_impl(e, &slabs[j], sk[j], geo[j], grids[j], whole ? meds[j] : nullptr, o2, true, &r,
                  sc, P);
    });
    if (M > 0.0) {
        res->argmax_index = -1;
        for (int j = 0; j < G; ++j) {
            const dg_result& r = pr[j];
            if (slabs[j].size() == 0 || r.argmax_index < 0) continue;
            if (res->argmax_index < 0 || r.argmax_value > res->argmax_value ||
                (r.argmax_value == res->argmax_value && r.argmax_index < res->argmax_index)) {
                res->argmax_index = r.argmax_index;
                res->argmax_value = r.argmax_value;
            }
        }
    } else {  // all-zero surface: first index wins
        res->argmax_index = g->row_offset * n_lon;
        res->argmax_value = 0.0;
    }
    // the full surface on device 0 (caller's buffer or scratch) and detection
    set_device(eng);
    Scratch& s0 = *scr[0];
    double* full = res->accumulated_device ? res->accumulated_device : nullptr;
    if (!full && opt.detect) full = s0.alloc<double>(P);
    if (full) {
        for (int j = 0; j < G; ++j)
            if (slabs[j].size() > 0)
                CK(cudaMemcpyPeerAsync(full + r0[j] * n_lon, eng->device, acc[j],
                                       eng->dev(j)->device, slabs[j].size() * sizeof(double),
                                       s0.st));
    }
    res->n_detections = 0;
    int64_t launches = 0;
    if (opt.detect)
        run_detect(g, full, opt.k_sigma, opt.exclusion_radius_cells, res->detections,
                   res->detections_capacity, &res->n_detections, s0, &launches);
    CK(cudaStreamSynchronize(s0.st));
    for (int k = 0; k < G; ++k) {
        const dg_result& a = part[k];
        res->n_refined += a.n_refined;
        res->sum_overlap_samples += a.sum_overlap_samples;
        res->correlate_launches += a.correlate_launches;
        res->moment_ffma2 += a.moment_ffma2;
        res->evaluate_ffma2 += a.evaluate_ffma2;
        res->evaluate_tc_flop += a.evaluate_tc_flop;
        res->direct_steps += a.direct_steps;
        res->moment_fft_flop += a.moment_fft_flop;
        res->kernel_launches += a.kernel_launches + pr[k].kernel_launches;
        res->n_reranked += pr[k].n_reranked;
    }
    res->kernel_launches += launches;
    // scratch of each device freed on its own device
    for (int k = G - 1; k >= 0; --k) {
        set_device(eng->dev(k));
        CK(cudaStreamSynchronize(scr[k]->st));
        scr[k].reset();
    }
    set_device(eng);
}

}  // namespace

extern "C" {

int dg_correlate_steps(dg_engine* eng, const dg_grid* g, const dg_staged* sn, int64_t s_begin,
                       int64_t s_end, const dg_options* opt_in, double* grids_device,
                       double* medians_device, dg_result* res) {
    return guard([&] {
        const dg_options opt = options_or_default(opt_in);
        check_run(eng, g, sn, opt, res);
        if (s_begin < 0 || s_end > sn->S || s_begin > s_end)
            raise(DG_EINVAL, "dg_correlate_steps: bad snapshot range");
        if (!grids_device) raise(DG_EINVAL, "dg_correlate_steps: null grids");
        if (opt.normalize_per_snapshot && !medians_device)
            raise(DG_EINVAL, "dg_correlate_steps: normalisation needs a medians buffer");
        set_device(eng);
        StreamGuard sg(opt.stream, eng->stream);
        Scratch sc(sg.st, &eng->arena);
        reset_stats(res);
        const RunGeo geo = make_geo(sc, sn);
        correlate_steps_impl(eng, g, sn, geo, (int)s_begin, (int)s_end, opt, grids_device,
                             medians_device, sc, res);
    });
}

int dg_shard_plan(int64_t S, int64_t R, int world, int whole, dg_work_unit* out, int64_t cap,
                  int64_t* n_out) {
    return guard([&] {
        if (S < 1) raise(DG_EINVAL, "geolocate_snapshots: no snapshots");
        if (R < 2) raise(DG_EINVAL, "correlate_snapshot_all_pairs: need >= 2 receivers");
        if (world < 1) raise(DG_EINVAL, "dg_shard_plan: world < 1");
        const auto units = shard_plan(S, R * (R - 1) / 2, world, whole != 0);
        if (n_out) *n_out = (int64_t)units.size();
        if (out)
            for (int64_t i = 0; i < std::min<int64_t>(cap, (int64_t)units.size()); ++i)
                out[i] = units[i];
    });
}

int dg_correlate_units(dg_engine* eng, const dg_grid* g, const dg_staged* sn,
                       const dg_work_unit* units, int64_t n_units, const dg_options* opt_in,
                       double* raw, dg_result* res) {
    return guard([&] {
        const dg_options opt = options_or_default(opt_in);
        check_run(eng, g, sn, opt, res);
        if (n_units < 0 || (n_units > 0 && (!units || !raw)))
            raise(DG_EINVAL, "dg_correlate_units: null units / surfaces");
        set_device(eng);
        StreamGuard sg(opt.stream, eng->stream);
        Scratch sc(sg.st, &eng->arena);
        reset_stats(res);
        const RunGeo geo = make_geo(sc, sn);
        std::vector<StepUnit> u(n_units);
        for (int64_t i = 0; i < n_units; ++i)
            u[i] = StepUnit{(int)units[i].step, units[i].part, units[i].parts};
        correlate_units_impl(eng, g, sn, geo, u, opt, raw, sc, res);
    });
}

int dg_accumulate_peak(dg_engine* eng, const dg_grid* g, const dg_staged* sn,
                       const double* grids_device, const double* medians_device,
                       const dg_options* opt_in, dg_result* res) {
    return guard([&] {
        const dg_options opt = options_or_default(opt_in);
        check_run(eng, g, sn, opt, res);
        if (!grids_device && opt.peak_stage != 2)
            raise(DG_EINVAL, "dg_accumulate_peak: null grids");
        set_device(eng);
        StreamGuard sg(opt.stream, eng->stream);
        Scratch sc(sg.st, &eng->arena);
        reset_stats(res);
        const RunGeo geo = make_geo(sc, sn);
        peak_impl(eng, g, sn, geo, grids_device,
                  opt.normalize_per_snapshot ? medians_device : nullptr, opt, opt_in != nullptr,
                  res, sc);
    });
}

int dg_geolocate_staged(dg_engine* eng, const dg_grid* g, const dg_staged* sn, const dg_options* opt,
                        dg_result* res) {
    return guard([&] {
        if (eng && eng->n_devices() > 1)
            geolocate_multi(eng, g, sn, opt, res);
        else
            geolocate_impl(eng, g, sn, opt, res);
    });
}

int dg_geolocate_snapshots(dg_engine* eng, const dg_grid* g, const dg_snapshots* sn,
                           const dg_options* opt, dg_result* res) {
    return guard([&] {
        // the capture upload overlaps the geometry / planning phase
        std::unique_ptr<dg_staged> staged = stage_impl(eng, sn, true);
        if (eng->n_devices() > 1)
            geolocate_multi(eng, g, staged.get(), opt, res);
        else
            geolocate_impl(eng, g, staged.get(), opt, res);
        CK(cudaStreamSynchronize(eng->upload));  // before the host captures may change
    });
}

int dg_detect_emitters(dg_engine* eng, const dg_grid* g, const double* values, int is_device,
                       double k_sigma, int radius, dg_emitter_estimate* out, int64_t capacity,
                       int64_t* n_out) {
    return guard([&] {
        if (!eng || !g || !values || !n_out) raise(DG_EINVAL, "null argument");
        if (radius < 0) raise(DG_EINVAL, "detect_emitters: negative exclusion radius");
        set_device(eng);
        StreamGuard sg(nullptr, eng->stream);
        Scratch sc(sg.st);
        const int64_t P = g->size();
        const double* v = values;
        if (!is_device) {
            double* dv = sc.alloc<double>(P);
            CK(cudaMemcpyAsync(dv, values, P * sizeof(double), cudaMemcpyHostToDevice, sg.st));
            v = dv;
        }
        int64_t launches = 0;
        run_detect(g, v, k_sigma, radius, out, capacity, n_out, sc, &launches);
    });
}

int dg_plan_batches(uint64_t n_points, uint64_t batch_size, uint64_t budget, uint64_t capture_bytes,
                    uint64_t* batch_count) {
    // plan_batches (backend.hpp:77-93), messages verbatim
    return guard([&] {
        if (budget == 0) budget = 512ull << 20;
        if (n_points < 1) raise(DG_EINVAL, "plan_batches: n_points < 1");
        if (batch_size < 1) raise(DG_EINVAL, "plan_batches: batch_size < 1");
        if (capture_bytes > budget)
            raise(DG_EINVAL, "plan_batches: staged captures (" + std::to_string(capture_bytes) +
                                 " bytes) exceed the memory budget of " + std::to_string(budget));
        const uint64_t ws = batch_size * 24ull + capture_bytes;  // sizeof(PairOffsets)+sizeof(double)
        if (ws > budget)
            raise(DG_EINVAL, "plan_batches: batch working set (" + std::to_string(ws) +
                                 " bytes at batch_size " + std::to_string(batch_size) +
                                 ") exceeds the memory budget of " + std::to_string(budget));
        if (batch_count) *batch_count = (n_points + batch_size - 1) / batch_size;
    });
}

}  // extern "C"
