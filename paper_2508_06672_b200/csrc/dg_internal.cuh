// Internal declarations shared by the kernels (dg_kernels.cu) and the C ABI
// layer (dg_capi.cu). Not installed; the public boundary is include/b200geo.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "b200geo.h"

namespace dg {

// One warp-task of the correlator: up to correlate_task_size() candidates (32 per
// lane-slot) that share one integer
// TDOA d (so one z_d[k] = y1[k] conj(y2[k+d]) stream and one overlap range).
struct Task {
    int d;      // tdoa_samples
    int start;  // offset into the d-sorted candidate list
    int count;  // 1..correlate_task_size() candidates live
    int pad;    // index of the task's d-bucket (block-moment correlator)
};

// One d-bucket: every candidate with this integer TDOA (block-moment correlator).
struct Bucket {
    int d;      // tdoa_samples
    int start;  // offset into the d-sorted candidate list
    int count;  // candidates
    int nb;     // blocks of B samples covering the overlap [max(0,-d), min(N, N-d))
};

// Per-(snapshot, pair) ranges reduced by the geometry kernel: FDOA as
// order-preserving keys of the doubles, TDOA as ints (overlapping candidates only).
struct StepRange {
    unsigned long long fmin, fmax;
    int dmin, dmax;
};
inline void step_range_init(StepRange* r) {
    r->fmin = ~0ull;
    r->fmax = 0ull;
    r->dmin = 0x7fffffff;
    r->dmax = -0x7fffffff - 1;
}
__host__ __device__ inline unsigned long long f64_key(double v) {
    unsigned long long b;
#ifdef __CUDA_ARCH__
    b = (unsigned long long)__double_as_longlong(v);
#else
    __builtin_memcpy(&b, &v, 8);
#endif
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
inline double f64_from_key(unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double v;
    __builtin_memcpy(&v, &b, 8);
    return v;
}

// receiver pair of one step in FP32, positions relative to the lattice centre
struct RxPairF32 {
    float pi[3], vi[3], pj[3], vj[3];
};

constexpr int kMaxMoments = 16;  // Chebyshev table width (moments per block <= 16)
constexpr int kEvalG = 8;  // blocks per exact-phase group in k_evaluate (moment rows padded to it)
__host__ __device__ constexpr int pad_blocks(int nb) { return (nb + kEvalG - 1) / kEvalG * kEvalG; }

// Geometry of one (snapshot, pair): receiver states for predict_pair_offsets.
struct PairGeom {
    dg_state rx_i, rx_j;
};

// Per-element flag: FP32 result too close to zero for the relative tolerance;
// re-evaluated in FP64 in the reference's exact operation order.
constexpr int kChunk = 256;  // samples per z-chunk (per warp, TMA-staged in smem)

// Device capture layout: every capture sits in a zero-filled slot of `stride`
// elements starting kCapturePad elements in, with >= kCaptureTail zeros after
// it, so the correlator's chunked bulk copies never leave the allocation.
constexpr int64_t kCapturePad = 32;
constexpr int64_t kCaptureTail = 512;
inline int64_t capture_stride(int64_t n) {
    return (kCapturePad + n + kCaptureTail + 31) & ~int64_t(31);
}
constexpr int kL = 16;       // phasor table length (samples per inner block)

// Threshold on S / sqrt(max(sum_chunks |chunk sum|^2, sum_blocks |block sum|^2,
// ||z||_2^2)) below which a direct-correlator FP32 value is re-evaluated exactly
// (dg_correlate.cu); see DESIGN.md "Parity" for the error model behind it. The
// +40 dB chirp scenes, whose product tones alias onto the 16-sample blocks,
// showed ~1e-6 ||z||_2 errors (tests/gpu_error_diag.py): 0.04 -> 2.5e-5, 0.06
// keeps them near 1.7e-5 (tests/test_gpu_error_model.py).
constexpr float kRefineTau = 0.06f;
// block-moment correlator (refine_moment in dg_device.cuh): a
// value is re-evaluated in FP64 when S is small next to the bucket's noise floor
// ||z||_2 (tau_noise for incoherent buckets rising to tau for coherent ones) or
// next to the coherent part of its error scales (tau). Worst unrefined relative
// error on the stress scenes of tests/test_gpu_error_model.py vs the reference
// (tests/gpu_tau_sweep.py): tau 0.015 -> 2.5e-5, 0.02 -> 1.8e-5 (coherent scenes);
// tau_noise 0.005 / 0.01 / 0.02 -> 5.1e-5 / 3.7e-5 / 2.0e-5 on a +40 dB chirp with
// the moments forced (its aliased product tones read as incoherent) and 2.3e-5 /
// 1.5e-5 / 1.2e-5 on the C3 scene at 1 km, at 7k / 20k / 78k refined elements per C3
// solve (52.0 / 52.0 / 55.7 ms). 0.014 keeps >= 5x margin on every scene.
constexpr float kMomentRefineTau = 0.02f;
constexpr float kNoiseRefineTau = 0.014f;

// --------------------------------------------------------------------------
// launchers (dg_kernels.cu). All asynchronous on `st`.
void launch_grid_ecef(const double* row_a, const double* row_z, const double* col_c,
                      const double* col_s, int64_t n_lat, int64_t n_lon, double* x, double* y,
                      double* z, cudaStream_t st);

// geometry + histogram over grid points (geometry.hpp:51-83, bit-exact)
void launch_geometry_hist(const double* x, const double* y, const double* z, int64_t P,
                          const PairGeom* pg_dev, double fs, double wl, int N, int* d_out,
                          int* rank_out, double* fdoa_out, int* hist, double* s_out,
                          unsigned long long* overlap, int* err, StepRange* range,
                          cudaStream_t st);
// every unit of a window in one pass, receivers shared within groups (the pairs
// of a snapshot): d/rank/fdoa/surface slices of stride P, histograms of stride
// nbins. `pg` is HOST memory; the grouping tables go through `ws` (one per 64
// units of the window: pinned-free staging, device tables allocated by the caller).
struct GeoGroup {
    int rx0, nrx, u0, nu;  // receiver table slice, unit range
};
struct GeoScratch {
    dg_state rx[128];
    GeoGroup groups[64];
    int2 upair[64];
    int nrx = 0, ng = 0;
    dg_state* d_rx = nullptr;
    GeoGroup* d_groups = nullptr;
    int2* d_upair = nullptr;
};
void launch_geometry_units(const double* x, const double* y, const double* z, int64_t P,
                           const PairGeom* pg_host, int n, double fs, double wl, int N, int* d_out,
                           int* rank_out, double* fdoa_out, int* hist, int nbins, double* s_out,
                           unsigned long long* overlap, int* err, GeoScratch* ws,
                           cudaStream_t st);
// per capture (n_caps rows of `stride` elements) the exclusive prefix sums of
// |y|^2 in FP64: out[c][k], k <= N
void launch_energy_prefix(const double2* y, int64_t stride, int64_t n_caps, int64_t N,
                          double* out, cudaStream_t st);
// exact TDOA range (first / last non-empty bin) of each of n_steps histograms
void launch_hist_range(const int* hist, int nbins, int n_steps, int N, StepRange* out,
                       cudaStream_t st);
void launch_predict_offsets(const double* x, const double* y, const double* z, int64_t P,
                            const PairGeom* pg_dev, double fs, double wl, dg_pair_offsets* out,
                            int* err, cudaStream_t st);
// the same from caller offsets (correlate_batch path)
void launch_offsets_hist(const dg_pair_offsets* off, int64_t P, int N, int* d_out,
                         int* rank_out, double* fdoa_out, int* hist, double* s_out,
                         unsigned long long* overlap, StepRange* range, cudaStream_t st);
// planning ranges over a whole lattice (FP32, partition-independent)
void launch_lattice_rel(const double* x, const double* y, const double* z, int64_t P, double cx,
                        double cy, double cz, float4* out, cudaStream_t st);
void launch_range_fp32(const float4* rel, int64_t P, const RxPairF32* rx, int n_steps, double fs,
                       double wl, StepRange* out, cudaStream_t st);
// bins [bin0, bin0 + nb) of the TDOA histogram (bin = d + N - 1) -> d-sorted
// candidate ids, warp tasks of <= correlate_task_size() candidates and one
// Bucket per non-empty bin (blocks of length B; B = 0 skips buckets)
// rank: each candidate's rank in its bin (the geometry pass's histogram atomic)
void launch_bucket(int* hist, int bin0, int nb, int N, int* off, int* toff, int* boff,
                   int* cursor, int* n_tasks, int* n_buckets, const int* d, const int* rank,
                   int64_t P, int* sorted, Task* tasks, Bucket* buckets, int* ubin, int B,
                   cudaStream_t st, const double* fdoa = nullptr, double* sfdoa = nullptr);
// candidates per warp task of the active correlator variant (32 x candidates/lane)
int correlate_task_size();
void launch_correlate(const Task* tasks, const int* n_tasks, int max_tasks, const int* sorted,
                      const double* fdoa, const float2* y1, const float2* y2, int N, double fs,
                      double* s_out, uint32_t* flag_bits, int64_t flag_base, float tau,
                      cudaStream_t st);

// block-moment correlator (dg_moments.cu)
void launch_center(const double2* y, const float2* y2, int N, const double* nu_c, float2* y1c,
                   float2* y2p, int padf, cudaStream_t st);
void launch_work_count(const Bucket* buckets, const int* n_buckets, int B, int R, int tc,
                       unsigned long long* work, cudaStream_t st);
// moments of every bucket of a step (blocks aligned to absolute sample index);
// ubin[bin - bin0] = bucket of a TDOA bin or -1
void launch_moments(int B, int R, const Bucket* buckets, const int* ubin, int bin0, int nbins,
                    int N, const float* tcheb, const float2* y1c, const float2* y2p, int padf,
                    float2* mom, int nbmax, int sm_count, cudaStream_t st);
// the same moments as FFT cross-correlations (dg_moments_fft.cu), for 256 <= B <= 768:
// af = moments_fft_af_bytes of scratch, queue = N / 256 + 2 ints of scratch; fe receives per
// (window, block, moment) the mean square of the window's correlation, the scale of
// the FFT's rounding (moments_fft_fe_floats of scratch)
constexpr int kFftLen = 1024;
// weight of the FFT rounding's window excess in the refinement scale (calibrated
// on the error-model scenes)
constexpr float kFftRefineKappa = 4.0f;
bool moments_fft_supported(int B);
size_t moments_fft_af_bytes(int N, int B, int R);
size_t moments_fft_fe_floats(int N, int B, int R);
void launch_moments_fft(int B, int R, const int* ubin, int bin0, int nbins, int N,
                        const float* tchebT, const float2* y1c, const float2* y2p, int padf,
                        float2* mom, int nbmax, float2* af, float* fe, int* queue, int sm_count,
                        cudaStream_t st);
// what k_evaluate_tc needs of an FFT-moment step (qf = nullptr: direct moments):
// qf[bucket * kMaxMoments + m] = sum over the bucket's blocks of fe of its lag window
struct FftErr {
    const float* qf;
    float kappa;  // weight of the window's excess over the bucket's own moment energy
};
// qf of every bucket of a step (fe: launch_moments_fft's, window of a bin = bin / G -
// bin0 / G, fe[(window * R + m) * nblk + block])
void launch_fft_bucket_energy(const Bucket* buckets, const int* n_buckets, int max_buckets,
                              const float* fe, int bin0, int G, int nblk, int N, int B, int R,
                              float* qf, cudaStream_t st);
// per-bucket candidate evaluation; `queue` is a zeroed int (dynamic bucket queue);
// sfdoa = the candidates' FDOA in bucket order (launch_bucket's sfdoa)
size_t evaluate_smem_bytes(int nbmax, int R);
// e1 / e2: the two captures' |y|^2 prefix sums (launch_energy_prefix), N samples
void launch_evaluate(int R, const Bucket* buckets, const int* n_buckets, int* queue,
                     int max_buckets, const int* sorted, const double* fdoa, double fs,
                     const double* nu_c, int B, const float2* mom, int nbmax, double* s_out,
                     uint32_t* flag_bits, int64_t flag_base, float tau, float tau_noise,
                     const double* e1, const double* e2, int N, int sm_count, cudaStream_t st);

// surface writers (dg_writers.cu): "%.17g" text in kFmtSlot-byte slots, CSV rows
// at scanned offsets, P5 pixels
constexpr int kFmtSlot = 32;
// axis text of values start + (first + i) * step, i < count (GridAxis::value)
void launch_format_axis(double start, double step, int64_t first, int64_t count, char* slots,
                        uint8_t* len, cudaStream_t st);
void launch_format_values(const double* v, int64_t n, char* slots, uint8_t* len, cudaStream_t st);
size_t csv_scan_temp_bytes(int64_t n);
// row_end = inclusive scan of the row lengths (the CSV body is row_end[n-1] bytes)
void launch_csv_offsets(const uint8_t* lat_len, const uint8_t* lon_len, const uint8_t* val_len,
                        int64_t n_lat, int64_t n_lon, int64_t* row_len, int64_t* row_end,
                        void* temp, size_t temp_bytes, cudaStream_t st);
void launch_csv_emit(const char* lat_s, const uint8_t* lat_len, const char* lon_s,
                     const uint8_t* lon_len, const char* val_s, const uint8_t* val_len,
                     const int64_t* row_end, int64_t n_lat, int64_t n_lon, char* out,
                     cudaStream_t st);
void launch_minmax(const double* v, int64_t n, double2* part, double2* out, cudaStream_t st);
void launch_heatmap(const double* v, int64_t n_lat, int64_t n_lon, double lo, double scale,
                    uint8_t* out, cudaStream_t st);

// capture synthesis (dg_scene.cu): waveforms, the FFT fractional advance, the
// receive channel and MT19937-64 noise (reference scene.hpp / waveform.hpp)
constexpr int kWaveSpoofer = 0, kWaveTone = 1, kWaveChirp = 2, kWaveSawtooth = 3;
struct WaveParams {
    int kind;
    uint64_t seed;  // spoofer nav-bit seed
    double a, b;    // tone: offset; chirp: bandwidth, period; sawtooth: bandwidth, chirp period
};
void launch_waveform(const WaveParams& w, double start, double ts, int64_t n, const int8_t* chips,
                     double2* out, cudaStream_t st);
int fft_log2_max();
// forward spectrum of the tapered record padded to 2^l (four-step layout)
void launch_fractional_fwd(const double2* tx, int64_t n_tx, int guard, int l, double2* spec,
                           cudaStream_t st);
// advance by frac, inverse, and received[k] = amplitude * delayed[shift + k] * phasor[k]
void launch_fractional_inv(const double2* spec, int l, double frac, int64_t shift, int64_t n_out,
                           double amplitude, const double2* phasor, double2* work, double2* recv,
                           cudaStream_t st);
void launch_receive_direct(const double2* tx, int64_t shift, int64_t n_out, double amplitude,
                           const double2* phasor, double2* recv, cudaStream_t st);
void launch_phasors(const double2* rotation, int n_rec, int64_t n_out, double2* phasor,
                    cudaStream_t st);
// recv [S][E][R][n] -> caps (stride cap_stride per (s, r)) + sigma * noise
void launch_noise_combine(const uint64_t* seeds, int n_snap, int n_rx, int n_em,
                          const double2* recv, int64_t n, double sigma, int add_noise,
                          double2* caps, int64_t cap_stride, cudaStream_t st);

// the same evaluation with the block sums C_b on the tensor cores (dg_evaluate_tc.cu,
// tcgen05 kind::tf32, split hi/lo operands); needs 2 nbmax <= 512 TMEM columns
bool evaluate_tc_supported(int nbmax, int R);
void launch_evaluate_tc(FftErr fx, int R, const Bucket* buckets, const int* n_buckets, int* queue,
                        int max_buckets, const int* sorted, const double* fdoa, double fs,
                        const double* nu_c, int B, const float2* mom, int nbmax, double* s_out,
                        uint32_t* flag_bits, int64_t flag_base, float tau, float tau_noise,
                        const double* e1, const double* e2, int N, int sm_count,
                        cudaStream_t st);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for the current device, once
// per (call site, device, larger size): function attributes are per device and one
// process may drive engines on several GPUs
template <class K>
inline void ensure_smem(K kern, size_t smem, size_t (&done)[64]) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 64 || smem > done[dev]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (dev < 64) done[dev] = smem;
    }
}

// exact FP64 reference-order re-evaluation of flagged elements
// elem = s*pairs*P + pair*P + p ; (geolocate path recomputes geometry)
void launch_count_flags(const uint32_t* bits, int64_t n_words, unsigned long long* count,
                        cudaStream_t st);
void launch_compact_flags(const uint32_t* bits, int64_t n_words, int64_t* list,
                          unsigned long long* cursor, cudaStream_t st);
struct RefineCtx {
    // geolocate path (grid != nullptr) or batch path (offsets != nullptr)
    const double *x, *y, *z;
    int64_t P;
    const PairGeom* pg;       // [S*pairs]
    const int* pair_rx;       // [pairs*2] receiver indices
    int pairs, R;
    const dg_pair_offsets* offsets;  // batch path
    const double2* y64;       // geolocate: [S][R][stride]; batch: [2][stride]
    int64_t stride;           // elements between captures (>= N, multiple of 32)
    int N;
    double fs, wl;
    double* raw;              // [S*pairs*P] (batch: [P])
    const double* trig;       // re-rank only (nullable): [chain][4] host-libm phasors
    const int* unit_step;     // refine rows (nullable): global step of each row
};
void launch_refine(const int64_t* list, int64_t n, RefineCtx ctx, cudaStream_t st);
// refine steps [row0, row1) of a bitmap with one P32-element row per step
// (count of flagged elements left in *count); ctx.raw is dense [step][P]
void launch_refine_rows(const uint32_t* bits, int64_t row0, int64_t row1, int64_t P32,
                        int64_t* list, unsigned long long* count, RefineCtx ctx, cudaStream_t st);

void launch_combine_pairs(const double* raw, int S, int pairs, int64_t P, double* grids,
                          cudaStream_t st);
void launch_scale(double* v, int64_t P, const double* median, cudaStream_t st);
// steps[step[u]][i] += units[u][i], u in order (parts of split steps: exact)
void launch_sum_units(const double* units, int U, int64_t n, const int* step, double* steps,
                      cudaStream_t st);
// acc = [acc +] sum_s grids[s] in snapshot order (first: no running sum)
void launch_accumulate(const double* grids, int S, int64_t P, double* acc, cudaStream_t st,
                       bool first = true);
void launch_max(const double* v, int64_t P, double* partial, int n_partial, double* out,
                cudaStream_t st);
// near-peak selection for the exact re-rank: count of cells >= thr; the cells
// >= thr in ascending index (CUB select; temp sized by select_ge_temp_bytes for
// P cells and n_sel selected); a stable descending sort of selected cells by
// value (ties keep ascending index); exact values written into a surface
void launch_count_ge(const double* v, int64_t P, double thr, unsigned long long* count,
                     cudaStream_t st);
size_t select_ge_temp_bytes(int64_t P, int n_sel);
void launch_select_ge(const double* v, int64_t P, double thr, int* cells, int* n_out, void* temp,
                      size_t temp_bytes, cudaStream_t st);
void launch_sort_by_value(const double* v, const int* cells, int n, unsigned long long* keys,
                          unsigned long long* keys_out, int* cells_out, void* temp,
                          size_t temp_bytes, cudaStream_t st);
void launch_patch_cells(const int* cells, int n, const double* val, double* surf, cudaStream_t st);
void launch_first_max(const double* v, int64_t P, const double* vmax, unsigned long long* idx,
                      cudaStream_t st);
// n_items_hint: host-side count of near-peak cells (sizes the launch)
void launch_rerank(const int* cells, const int* n_cells, int cap, int n_items_hint, int SP,
                   RefineCtx ctx, double* ex, cudaStream_t st);
// exact offsets of every re-rank chain (cells[ci], step sp) -> out[ci * SP + sp]
void launch_chain_offsets(const int* cells, int n, int SP, RefineCtx ctx, dg_pair_offsets* out,
                          cudaStream_t st);
void launch_recombine_cells(const int* n_cells, int cap, const double* ex, int S, int pairs,
                            const double* medians, double* acc_ex, double* grid_ex /* [cap][S] */,
                            cudaStream_t st);
void launch_argmax_cells(const int* cells, const int* n_cells, int cap, const double* acc_ex,
                         long long* best_idx, double* best_val, cudaStream_t st);
// median (nth_element rank P/2) of nonnegative doubles by 4-pass radix select
void launch_median(const double* v, int64_t P, unsigned* hist, unsigned long long* state,
                   double* out, cudaStream_t st);

// detect_emitters (correlate.hpp:127-201)
struct DetCand {
    double score;
    long long key;  // ilat*1e6 + ilon (reference tie order)
    int ilat, ilon;
};
void launch_mean_var(const double* v, int64_t P, double* partial, int n_partial,
                     double* stats /* [mean, var, sigma] */, cudaStream_t st);
void launch_local_max(const double* v, int64_t n_lat, int64_t n_lon, const double* stats,
                      double k_sigma, DetCand* cands, int* n_cands, int cap, cudaStream_t st);
void launch_greedy(const DetCand* cands, const int* n_cands, int cap, int radius,
                   const double* stats, int64_t n_lon, dg_emitter_estimate* out, int* n_out,
                   cudaStream_t st);

void launch_f64_to_f32(const double2* in, float2* out, int64_t n, cudaStream_t st);
void launch_f32_to_f64(const float2* in, double2* out, int64_t n, cudaStream_t st);
// contiguous uploaded captures [n_caps][N] (double2 if f64, else float2) ->
// padded resident slots of stride elements (data at `pad`), FP64 and FP32
void launch_stage_captures(const void* in, bool f64, int64_t n_caps, int64_t N, int64_t stride,
                           int64_t pad, double2* y64, float2* y32, cudaStream_t st);

}  // namespace dg
