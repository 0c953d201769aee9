/*
 * b200geo — C ABI of the B200-native direct-geolocation engine.
 *
 * This is the drop-in boundary for the hot path of the reference `digeo`
 * library (paths relative to /root/reference/proj/include/digeo): the
 * position-domain correlation (Eq. 11) over every (candidate grid point,
 * time step), with the geometry that feeds it and the accumulation / peak
 * search after it. Every entry point below names the reference interface it
 * replaces. Plain pointers and sizes only; no C++ or torch types.
 *
 * Errors: every int-returning function returns DG_OK (0) or a DG_E* code and
 * leaves a thread-local message in dg_last_error(). Code 1 corresponds to the
 * reference's std::invalid_argument, 2 to std::runtime_error (CUDA, NCCL,
 * I/O), 3 to out-of-memory. The C++ shim (include/b200geo/digeo_plugin.hpp)
 * rethrows them as those exception types.
 *
 * Threading: one dg_engine per GPU (one process per GPU). A dg_engine may be
 * used from several host threads; every session / call owns its own stream
 * and device buffers (backend.hpp:196-209 "sessions are independent").
 */
#ifndef B200GEO_H
#define B200GEO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DG_ABI_VERSION 7

enum {
    DG_OK = 0,
    DG_EINVAL = 1,   /* std::invalid_argument */
    DG_ERUNTIME = 2, /* std::runtime_error / CUDA failure */
    DG_ENOMEM = 3
};

/* == digeo::PairOffsets (geometry.hpp:68-71): {int64 tdoa_samples; double fdoa_hz} */
typedef struct {
    int64_t tdoa_samples;
    double fdoa_hz;
} dg_pair_offsets;

/* == digeo::EcefVector (geodesy.hpp:43-50) */
typedef struct {
    double x, y, z;
} dg_ecef;

/* == digeo::EcefStateVector (state.hpp:27-39) */
typedef struct {
    dg_ecef position, velocity;
} dg_state;

/* == digeo::LatLonBounds (geodesy.hpp:126-138) */
typedef struct {
    double lat_min_deg, lat_max_deg, lon_min_deg, lon_max_deg;
} dg_latlon_bounds;

/* == digeo::EmitterEstimate (correlate.hpp:117-122), location flattened */
typedef struct {
    double lat_deg, lon_deg, alt_m;
    int64_t grid_index;
    double score;
    double score_zsigma;
} dg_emitter_estimate;

typedef struct dg_engine dg_engine;
typedef struct dg_session dg_session;
typedef struct dg_grid dg_grid;
typedef struct dg_staged dg_staged;

const char* dg_last_error(void);
int dg_abi_version(void);

/* ---- engine == digeo::CorrelationBackend (backend.hpp:211-217) ----------
 * Bound to one CUDA device (or several: dg_engine_create_multi). Descriptor is
 * {"b200", "parallel-batched", workers = number of GPUs} — never "gpu", which
 * the reference's tests require to be rejected by its own registry
 * (test_backend.cpp:181). */
int dg_device_count(int* n); /* visible CUDA devices */
int dg_engine_create(int device, dg_engine** out);
/* One engine over several GPUs of this process (devices[0] drives the calls
 * that use one device: sessions, grids, detection): dg_geolocate_snapshots /
 * dg_geolocate_staged on it shard the run across all of them (DESIGN.md
 * section 7), with peer copies over NVLink for the exchange. The descriptor's
 * workers = n_devices, as ParallelBatchedBackend(workers) (backend.hpp:292-317).
 * A device may repeat (tests run the sharded path on one GPU). */
int dg_engine_create_multi(const int* devices, int n_devices, dg_engine** out);
void dg_engine_destroy(dg_engine* engine);
int dg_engine_descriptor(const dg_engine* engine, char* name, size_t name_len, char* kind,
                         size_t kind_len, unsigned* workers);

/* ---- correlator tuning (tests / benchmarks; defaults are the product path) --
 * Replaces no reference interface: the reference's CPU kernel has no
 * variants. The settings live on the engine and are validated here, so no
 * caller environment can silently change a result: a forced moment count is
 * still used only where it meets the truncation bound (otherwise the planner
 * picks the next admissible choice), and a refinement threshold below the
 * default (which would weaken the 1e-4 relative contract) is rejected unless
 * allow_weaker_refine is set explicitly. */
#define DG_CORRELATOR_AUTO 0    /* block moments where cheaper, else the direct correlator */
#define DG_CORRELATOR_DIRECT 1  /* direct FP32 correlator only */
#define DG_CORRELATOR_MOMENTS 2 /* block moments wherever the truncation bound admits them */
typedef struct {
    int correlator;          /* DG_CORRELATOR_* */
    int moment_block;        /* 0 = planner's choice, else 64/128/256/512/640/768 */
    int moment_count;        /* 0 = planner's choice, else 8/10/12/14/16 */
    int evaluate_tensor;     /* 1: block sums on tcgen05 where they fit; 0: FFMA2 block loop */
    double refine_tau;       /* FP64 re-evaluation threshold of the moment path (0 = default) */
    int allow_weaker_refine; /* permit thresholds below the defaults (error-model studies only) */
    double direct_refine_tau; /* the same for the direct correlator (0 = default) */
    double noise_refine_tau;  /* moment path: threshold on the bucket's noise floor ||z||_2
                                 (0 = default); refine_tau applies to the coherent excess */
    int64_t surface_budget_bytes; /* per-snapshot surfaces held at once when the caller does not
                                     want them back; past it a run is solved in snapshot chunks
                                     (0 = default, 4 GiB) */
    int moment_fft;          /* 1: block moments as FFT cross-correlations (B >= 256);
                                0: direct FP32x2 sums */
    double fft_refine_kappa; /* FFT moments: weight of a lag window's excess energy in the
                                refinement scale (0 = default) */
} dg_tuning;
void dg_tuning_default(dg_tuning* t);
int dg_engine_set_tuning(dg_engine* engine, const dg_tuning* t);
int dg_engine_get_tuning(const dg_engine* engine, dg_tuning* t);

/* ---- session == CorrelationBackend::stage + CorrelationSession ---------
 * dg_stage replaces backend.hpp:214-215 (+ check_pair :221-228): copies both
 * captures (interleaved complex double, std::complex<double> layout) to the
 * device. n1/n2 and fs1/fs2 are validated like the reference (mismatch ->
 * DG_EINVAL). dg_stage_f32 takes float I/Q (the DGIQ on-disk format,
 * io.hpp:123-167). */
int dg_stage(dg_engine* engine, const double* y1_iq, int64_t n1, double fs1, const double* y2_iq,
             int64_t n2, double fs2, dg_session** out);
int dg_stage_f32(dg_engine* engine, const float* y1_iq, int64_t n1, double fs1,
                 const float* y2_iq, int64_t n2, double fs2, dg_session** out);
void dg_session_destroy(dg_session* session);

/* CorrelationSession::correlate_batch (backend.hpp:204-205): out[i] = S for
 * batch[i]; host spans, out fully written on return. Empty batch or
 * n_out != n -> DG_EINVAL (backend.hpp:236-238). */
int dg_correlate_batch(dg_session* session, const dg_pair_offsets* batch, int64_t n, double* out,
                       int64_t n_out);

/* ---- candidate grid == digeo::CandidateGrid / build_candidate_grid -----
 * geodesy.hpp:182-207: validation and axis counts exactly as the reference;
 * the lat-major ECEF lattice is formed on the GPU (bit-identical doubles to
 * lla_to_ecef). point_cap 0 means the reference default (20,000,000). */
int dg_build_candidate_grid(dg_engine* engine, const dg_latlon_bounds* bounds, double spacing_deg,
                            double altitude_m, uint64_t point_cap, dg_grid** out);
/* Sub-grid of lattice rows [row_begin, row_end): the slab one rank owns when
 * the grid is sharded across GPUs. Flat indices stay global via row offset. */
int dg_grid_slab(const dg_grid* grid, int64_t row_begin, int64_t row_end, dg_grid** out);
/* Arbitrary host ECEF points (e.g. CandidateGrid::points of a reference grid),
 * lattice shape n_lat x n_lon for detection (n_lat*n_lon == n_points). */
int dg_grid_from_points(dg_engine* engine, const dg_ecef* points, int64_t n_points, double lat_start,
                        double lat_step, int64_t n_lat, double lon_start, double lon_step,
                        int64_t n_lon, double altitude_m, dg_grid** out);
/* GridAxis fields + row offset of this slab in the full lattice */
int dg_grid_info(const dg_grid* grid, double* lat_start, double* lat_step, int64_t* n_lat,
                 double* lon_start, double* lon_step, int64_t* n_lon, double* altitude_m,
                 int64_t* row_offset);
int dg_grid_points(const dg_grid* grid, dg_ecef* out_host); /* D2H of the eager lattice */
void dg_grid_destroy(dg_grid* grid);

/* predict_pair_offsets (geometry.hpp:73-83) for every grid point, on the GPU,
 * bit-identical to the reference. */
int dg_predict_offsets(dg_engine* engine, const dg_grid* grid, const dg_state* rx_i,
                       const dg_state* rx_j, double sample_rate_hz, double wavelength_m,
                       dg_pair_offsets* out_host);

/* correlate_snapshot (geolocate.hpp:41-75): one snapshot, one pair, the whole
 * grid, offsets computed on the GPU; out_host has grid-size doubles. */
int dg_correlate_snapshot(dg_session* session, const dg_grid* grid, const dg_state* rx_i,
                          const dg_state* rx_j, double center_freq_hz, double* out_host);

/* ---- whole-run driver == geolocate_snapshots (geolocate.hpp:96-146) ---- */
typedef struct {
    int64_t n_snapshots;
    int64_t n_receivers;
    int64_t n_samples;
    double sample_rate_hz;
    double center_freq_hz;
    const dg_state* states;            /* [n_snapshots][n_receivers] */
    const double* const* captures_iq;  /* n_snapshots*n_receivers pointers, complex double */
    const float* const* captures_f32;  /* alternative (DGIQ float I/Q); used if captures_iq NULL */
} dg_snapshots;

typedef struct {
    double k_sigma;             /* GeolocateOptions::k_sigma (default 5) */
    int exclusion_radius_cells; /* default 5 */
    int normalize_per_snapshot; /* median normalisation (geolocate.hpp:115-122) */
    int detect;                 /* run detect_emitters on the accumulated surface */
    void* stream;               /* cudaStream_t to launch on; NULL = private stream */
    int profile;                /* record per-kernel CUDA events into dg_result stats
                                   (steps then run serialised on one stream, so each
                                   kernel's event time is its own) */
    int patch_peak;             /* write the exact FP64 values of the re-ranked near-peak
                                   cells into the returned surfaces, host and device, before
                                   detection (default 1), so max_element on them is the exact
                                   argmax and detection scores equal the surface; 0 keeps every
                                   cell the FP32-path value */
    /* Exact peak: every cell whose fast accumulated value
     * is >= M (1 - 1e-4) / (1 + 1e-4), M the fast maximum, is re-evaluated in the
     * reference's FP64 order (the 1e-4 per-element contract bounds where the true
     * argmax can lie); past 4096 such cells they are re-ranked in rounds by
     * descending fast value until no remaining cell can reach the best exact one. */
    int peak_stage;             /* 0: accumulate + exact peak (default); 1: accumulate only
                                   (argmax_* = the fast maximum, lowest index); 2: exact peak of
                                   the surface given in accumulated_device (no accumulation) */
    double peak_max;            /* > 0: M for the band instead of this call's own maximum (the
                                   maximum over all slabs of a sharded run, so every partition
                                   re-ranks the same cells); a slab with no cell in the band
                                   returns argmax_index -1 */
} dg_options;

typedef struct {
    /* outputs (all nullable) */
    double* accumulated;        /* host [P] */
    double* accumulated_device; /* device [P] (caller-owned, e.g. a torch tensor) */
    double* per_snapshot;       /* host [n_snapshots][P] */
    dg_emitter_estimate* detections; /* the first detections_capacity of n_detections are
                                        written; the whole list (never truncated by the
                                        engine) comes from dg_detect_emitters on the returned
                                        surface with a buffer of n_detections entries */
    int64_t detections_capacity;
    /* filled by the call */
    int64_t n_detections;
    int64_t argmax_index;       /* flat index in the FULL lattice (slab row offset applied) */
    double argmax_value;        /* exact FP64 accumulated value at argmax */
    int64_t n_refined;          /* elements re-evaluated in FP64 (small |S|) */
    int64_t n_reranked;         /* near-peak cells re-evaluated in FP64 for the argmax */
    double sum_overlap_samples; /* sum over (point, step, pair) of N_ov (algorithmic work) */
    double correlate_ms;        /* profile: summed CUDA-event time of the correlate kernel */
    int64_t correlate_launches;
    double total_ms;            /* profile: event time of the whole device pipeline */
    int64_t kernel_launches;    /* all kernels this call launched */
    /* block-moment correlator accounting */
    double moments_ms;          /* profile: event time of k_moments (+ k_center) */
    double evaluate_ms;         /* profile: event time of k_evaluate */
    double moment_ffma2;        /* k_moments FMA-pipe work in FP32x2 operations: per bucket-
                                   block B/2 (R + 6) (R moment MACs per folded sample pair,
                                   two complex products, one fold) */
    double evaluate_ffma2;      /* candidate-side FP32x2 operations: block loop count*nb*(R+3);
                                   tensor-core path count*nb*3 (group sums on CUDA cores) */
    int64_t direct_steps;       /* (snapshot, pair) steps run on the direct correlator */
    double evaluate_tc_flop;    /* tensor-core FLOPs k_evaluate_tc issued (BF16 MMAs, 0 if none) */
    double moment_fft_flop;     /* FFT moments (k_mfft_a + k_mfft): 5 L log2 L per 1024-point
                                   FFT + 6 L per spectrum product; moment_ffma2 then counts the
                                   direct sums the FFTs replaced */
} dg_result;

void dg_options_default(dg_options* opt);

/* Host snapshots in, host results out (H2D/D2H inside). */
int dg_geolocate_snapshots(dg_engine* engine, const dg_grid* grid, const dg_snapshots* snaps,
                           const dg_options* opt, dg_result* result);

/* Stage a run's captures/states on the device once (H2D + FP32 conversion) … */
int dg_stage_snapshots(dg_engine* engine, const dg_snapshots* snaps, dg_staged** out);
/* … and solve with inputs already resident in HBM. */
int dg_geolocate_staged(dg_engine* engine, const dg_grid* grid, const dg_staged* staged,
                        const dg_options* opt, dg_result* result);
void dg_staged_destroy(dg_staged* staged);

/* DGIQ capture files, the reference's on-disk capture format (io.hpp:45-52,
 * read_iq :140-167): 38-byte little-endian header + float32 I/Q payload. The
 * checks and messages are read_iq's; runtime_error -> DG_ERUNTIME. */
typedef struct {
    double sample_rate_hz;
    double center_freq_hz;
    double start_time_s;
    int64_t sample_count;
} dg_iq_header;
int dg_read_iq_header(const char* path, dg_iq_header* out);
/* header + payload (2 * sample_count floats into iq_out; nullable = header only) */
int dg_read_iq(const char* path, dg_iq_header* out, float* iq_out, int64_t capacity);
/* load_snapshots (tools/digeo_cli.cpp:64-85) + dg_stage_snapshots for files: paths
 * [n_snapshots][n_receivers], states likewise; each payload is read straight into a
 * pinned buffer and copied to HBM as float2 (exact) while the next file is read. */
int dg_stage_snapshots_iq(dg_engine* engine, const char* const* paths, int64_t n_snapshots,
                          int64_t n_receivers, const dg_state* states, dg_staged** out);

/* Surfaces and detections on disk (io.hpp:169-280), formatted on the device.
 * `values` = grid size doubles, lat-major, in device memory when values_on_device
 * (e.g. dg_result.accumulated_device), else host memory. Bytes are identical to
 * the reference writers': CSV "%.17g,%.17g,%.17g\n" rows after the
 * "lat_deg,lon_deg,value" header (write_grid csv, :174-183), DGGR binary
 * (:187-202), 16-bit big-endian P5 with min->0, max->65535 and north on top
 * (render_heatmap, :245-268). Errors: "cannot open <path> for writing",
 * "write failed: <path>" (DG_ERUNTIME), as write_file_bytes (:114-119). */
#define DG_GRID_CSV 0
#define DG_GRID_BINARY 1
int dg_write_grid(dg_engine* engine, const dg_grid* grid, const double* values,
                  int values_on_device, const char* path, int format);
int dg_render_heatmap(dg_engine* engine, const dg_grid* grid, const double* values,
                      int values_on_device, const char* path);
/* write_detections_csv (:270-280) */
int dg_write_detections_csv(const dg_emitter_estimate* detections, int64_t n, const char* path);
/* == GridAxis pair + altitude of a DGGR file / lattice (geodesy.hpp:140-168) */
typedef struct {
    double lat_start_deg, lat_step_deg;
    int64_t lat_count;
    double lon_start_deg, lon_step_deg;
    int64_t lon_count;
    double altitude_m;
} dg_grid_axes;
/* read_grid (:205-240): header checks and messages verbatim; `values` (nullable:
 * header only) receives lat_count*lon_count doubles if capacity allows. */
int dg_read_grid(const char* path, dg_grid_axes* axes, double* values, int64_t capacity);
/* the eager ECEF lattice of explicit axes (the lattice read_grid rebuilds) */
int dg_grid_from_axes(dg_engine* engine, const dg_grid_axes* axes, dg_grid** out);
/* "%.17g" of n host doubles by the device formatter the CSV writer uses: 32-byte
 * slots (not terminated) and lengths; for tests against the C library. */
int dg_format_g17(dg_engine* engine, const double* values, int64_t n, char* slots,
                  uint8_t* lengths);

/* Capture synthesis on the device: the reference's simulate_scenario
 * (scene.hpp:200-310) with its waveforms (waveform.hpp:124-204), FFT fractional
 * delay (scene.hpp:161-191) and seeded noise (scene.hpp:124-147). Scenario
 * arithmetic (epochs, orbits, geometry, delays, amplitudes, seeds) is the
 * reference's, bit for bit; per-sample values agree to FP64 rounding (device
 * cos/sin/log and FFT rounding; MT19937-64 integers exact). Captures land in HBM
 * as a dg_staged run ready for dg_geolocate_staged. */
#define DG_WAVE_SPOOFER 0
#define DG_WAVE_TONE 1
#define DG_WAVE_CHIRP 2
#define DG_WAVE_SAWTOOTH 3
/* == digeo::EmitterDef with its WaveformSpec (scene.hpp:46-60, waveform.hpp:58-97) */
typedef struct {
    double lat_deg, lon_deg, alt_m;
    int waveform;               /* DG_WAVE_* */
    int prn;                    /* spoofer: 1..32 */
    uint64_t data_seed;         /* spoofer nav bits */
    double tone_offset_hz;      /* tone */
    double bandwidth_hz;        /* chirp / sawtooth */
    double period_s;            /* chirp period / sawtooth chirp period */
    double ref_snr_db, ref_range_m;
} dg_emitter_def;
/* == digeo::ReceiverDef: a CircularOrbit (orbit.hpp:30-35) unless `states`
 * (snapshot_count explicit states) is non-null */
typedef struct {
    double alt_m, inclination_deg, raan_deg, phase_deg;
    const dg_state* states;
} dg_receiver_def;
/* == digeo::Scenario (scene.hpp:72-110) without the grid */
typedef struct {
    const dg_receiver_def* receivers;
    int64_t n_receivers;
    const dg_emitter_def* emitters;
    int64_t n_emitters;
    int64_t snapshot_count;
    double snapshot_spacing_s, capture_duration_s, sample_rate_hz, center_freq_hz, start_time_s;
    uint64_t noise_seed;
    double noise_power;
} dg_scenario;
/* samples per capture, llround(duration * fs) (scene.hpp:112-114) */
int dg_scenario_samples(const dg_scenario* scenario, int64_t* n_samples);
/* staged_out (nullable) receives the run in HBM; captures_host (nullable) the
 * [S][R][N] complex double captures, states_host [S][R] and epochs_host [S]
 * (nullable) the snapshot states and epochs. */
int dg_simulate_scenario(dg_engine* engine, const dg_scenario* scenario, dg_staged** staged_out,
                         double* captures_host, dg_state* states_host, double* epochs_host);

/* The two halves of geolocate_snapshots, for snapshot-sharded multi-GPU runs
 * (DESIGN.md section 7). dg_correlate_steps: snapshots [s_begin, s_end) over
 * the whole grid — correlate_snapshot_all_pairs (geolocate.hpp:79-94) and the
 * optional normalize_by_median (:115-122) — into grids_device
 * [(s_end-s_begin)][P] and medians_device [s_end-s_begin] (device, caller-
 * owned; medians only when opt->normalize_per_snapshot). Fills n_refined,
 * sum_overlap_samples, correlate/moments/evaluate stats of `result`.
 * dg_accumulate_peak: accumulate_grids (correlate.hpp:102-113) of
 * grids_device [S][P_grid] (all snapshots, this grid or slab) in snapshot
 * order, the exact argmax and detect_emitters; outputs as dg_geolocate_staged. */
int dg_correlate_steps(dg_engine* engine, const dg_grid* grid, const dg_staged* staged,
                       int64_t s_begin, int64_t s_end, const dg_options* opt,
                       double* grids_device, double* medians_device, dg_result* result);
int dg_accumulate_peak(dg_engine* engine, const dg_grid* grid, const dg_staged* staged,
                       const double* grids_device, const double* medians_device,
                       const dg_options* opt, dg_result* result);

/* Work units of a sharded run. A unit is one
 * (snapshot, pair) step s * pairs + q over the whole grid, or part `part` of
 * `parts` of it: the candidates of a contiguous, cost-balanced range of the
 * step's TDOA buckets, the other candidates 0, so the parts of a step sum to
 * the whole step exactly. dg_shard_plan gives rank r the whole steps
 * [r q, (r + 1) q), q = floor(steps / world), and part r of each of the last
 * steps mod world steps, so every rank holds q + (steps mod world) / world
 * steps of work (whole_snapshots: snapshot units [r S / world, (r + 1) S /
 * world) for median normalisation, which needs a whole snapshot surface). */
typedef struct {
    int64_t step;  /* s * pairs + q (whole_snapshots: the snapshot s) */
    int32_t part, parts;
    int32_t rank;  /* owner */
    int32_t reserved;
} dg_work_unit;
int dg_shard_plan(int64_t n_snapshots, int64_t n_receivers, int world, int whole_snapshots,
                  dg_work_unit* out, int64_t capacity, int64_t* n_out);
/* raw per-unit surfaces [n_units][P] (device, caller-owned) of the grid's
 * cells: correlation + exact refinement, no pair sums or normalisation. */
int dg_correlate_units(dg_engine* engine, const dg_grid* grid, const dg_staged* staged,
                       const dg_work_unit* units, int64_t n_units, const dg_options* opt,
                       double* raw_device, dg_result* result);

/* detect_emitters (correlate.hpp:127-201) on a caller-provided surface over a
 * grid lattice (host or device pointer; is_device selects). */
int dg_detect_emitters(dg_engine* engine, const dg_grid* grid, const double* values, int is_device,
                       double k_sigma, int exclusion_radius_cells, dg_emitter_estimate* out,
                       int64_t capacity, int64_t* n_out);

/* plan_batches (backend.hpp:77-93): same validation/messages; 0 budget means
 * the reference default (512 MiB). */
int dg_plan_batches(uint64_t n_points, uint64_t batch_size, uint64_t memory_budget_bytes,
                    uint64_t capture_bytes_total, uint64_t* batch_count);

/* Measured FP32 CUDA-core peak (FFMA, register operands, full occupancy) of
 * `device` in TFLOP/s: the roofline denominator bench.py reports against. */
int dg_fp32_peak_tflops(int device, double* tflops);
/* The same issued as packed FP32x2 FMAs (fma.rn.f32x2 / SASS FFMA2). */
int dg_fp32x2_peak_tflops(int device, double* tflops);
/* FP64 DFMA peak (geometry, refinement and re-rank run in FP64). */
int dg_fp64_peak_tflops(int device, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* B200GEO_H */
