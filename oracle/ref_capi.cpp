// ORACLE / TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// A thin extern "C" wrapper that exposes the *unmodified* reference library
// (`digeo`, header-only C++20 under /root/reference/proj/include) to the
// parity tests and to bench.py's CPU-baseline leg. It is compiled by
// oracle/Makefile into oracle/_ref/libdigeo_ref.so straight from the
// reference headers where they lie; no reference source is copied here.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load it.
//
// Every function forwards to the reference symbol cited beside it.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "digeo/backend.hpp"
#include "digeo/bench.hpp"
#include "digeo/config.hpp"
#include "digeo/correlate.hpp"
#include "digeo/geodesy.hpp"
#include "digeo/geolocate.hpp"
#include "digeo/geometry.hpp"
#include "digeo/io.hpp"
#include "digeo/scene.hpp"

using namespace digeo;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

#define REF_GUARD(...)                                             \
    try {                                                          \
        __VA_ARGS__;                                                    \
        return 0;                                                  \
    } catch (const std::invalid_argument& e) {                     \
        return fail(e, 1);                                         \
    } catch (const std::exception& e) {                            \
        return fail(e, 2);                                         \
    }

BasebandCapture make_cap(const double* iq, int64_t n, double fs, double fc) {
    BasebandCapture c;
    c.sample_rate_hz = fs;
    c.center_freq_hz = fc;
    c.samples.resize(static_cast<std::size_t>(n));
    if (n > 0) std::memcpy(c.samples.data(), iq, static_cast<std::size_t>(n) * sizeof(cplx));
    return c;
}

EcefStateVector make_state(const double* s6) {
    return EcefStateVector{{s6[0], s6[1], s6[2]}, {s6[3], s6[4], s6[5]}};
}

struct Scene {
    ScenarioConfig config;
    std::vector<Snapshot> snapshots;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// --- scenes (config.hpp:269-324, scene.hpp:253-310) ------------------------

int ref_scene_parse(const char* text, void** out) {
    REF_GUARD({
        std::istringstream in{std::string(text)};
        auto scene = std::make_unique<Scene>();
        scene->config = parse_scenario_stream(in, "<text>");
        *out = scene.release();
    })
}

void ref_scene_free(void* h) { delete static_cast<Scene*>(h); }

int ref_scene_simulate(void* h) {
    REF_GUARD({
        auto* s = static_cast<Scene*>(h);
        s->snapshots = simulate_scenario(s->config.scenario);
    })
}

// info: [n_snap, n_rx, n_samples] ints; [fs, fc, lat_min, lat_max, lon_min, lon_max,
// spacing, alt, k_sigma, exclusion_radius, normalize, batch_size] doubles
void ref_scene_info(void* h, int64_t* ints3, double* dbl12) {
    const auto* s = static_cast<Scene*>(h);
    const Scenario& sc = s->config.scenario;
    ints3[0] = static_cast<int64_t>(sc.snapshot_count);
    ints3[1] = static_cast<int64_t>(sc.receivers.size());
    ints3[2] = static_cast<int64_t>(sc.samples_per_capture());
    dbl12[0] = sc.sample_rate_hz;
    dbl12[1] = sc.center_freq_hz;
    dbl12[2] = sc.grid_bounds.lat_min_deg;
    dbl12[3] = sc.grid_bounds.lat_max_deg;
    dbl12[4] = sc.grid_bounds.lon_min_deg;
    dbl12[5] = sc.grid_bounds.lon_max_deg;
    dbl12[6] = sc.grid_spacing_deg;
    dbl12[7] = sc.grid_altitude_m;
    dbl12[8] = s->config.options.k_sigma;
    dbl12[9] = s->config.options.exclusion_radius_cells;
    dbl12[10] = s->config.options.normalize_per_snapshot ? 1.0 : 0.0;
    dbl12[11] = static_cast<double>(s->config.options.batch_size);
}

int ref_scene_capture(void* h, int64_t snap, int64_t rx, double* out_iq) {
    REF_GUARD({
        const auto* s = static_cast<Scene*>(h);
        const auto& cap = s->snapshots.at(static_cast<std::size_t>(snap))
                              .captures.at(static_cast<std::size_t>(rx));
        std::memcpy(out_iq, cap.samples.data(), cap.samples.size() * sizeof(cplx));
    })
}

int ref_scene_state(void* h, int64_t snap, int64_t rx, double* out6) {
    REF_GUARD({
        const auto* s = static_cast<Scene*>(h);
        const auto& st = s->snapshots.at(static_cast<std::size_t>(snap))
                             .states.at(static_cast<std::size_t>(rx));
        const double v[6] = {st.position.x, st.position.y, st.position.z,
                             st.velocity.x, st.velocity.y, st.velocity.z};
        std::memcpy(out6, v, sizeof v);
    })
}

// --- geodesy / geometry (geodesy.hpp:82-92,182-207; geometry.hpp:36-83) -----

int ref_lla_to_ecef(double lat, double lon, double alt, double* out3) {
    REF_GUARD({
        const EcefVector p = lla_to_ecef({lat, lon, alt});
        out3[0] = p.x;
        out3[1] = p.y;
        out3[2] = p.z;
    })
}

double ref_wavelength(double fc) { return wavelength_m(fc); }

int ref_build_grid(const double* bounds4, double spacing, double alt, uint64_t cap,
                   int64_t* n_lat, int64_t* n_lon, double* points_or_null) {
    REF_GUARD({
        const CandidateGrid g = build_candidate_grid(
            {bounds4[0], bounds4[1], bounds4[2], bounds4[3]}, spacing, alt, cap);
        *n_lat = static_cast<int64_t>(g.lat.count);
        *n_lon = static_cast<int64_t>(g.lon.count);
        if (points_or_null)
            std::memcpy(points_or_null, g.points.data(), g.points.size() * sizeof(EcefVector));
    })
}

int ref_predict_pair_offsets(const double* cand3, const double* rx_i6, const double* rx_j6,
                             double fs, double wl, int64_t* tdoa, double* fdoa) {
    REF_GUARD({
        const PairOffsets o = predict_pair_offsets({cand3[0], cand3[1], cand3[2]},
                                                   make_state(rx_i6), make_state(rx_j6), fs, wl);
        *tdoa = o.tdoa_samples;
        *fdoa = o.fdoa_hz;
    })
}

// --- correlation (correlate.hpp:44-86, backend.hpp:196-325) ----------------

int ref_correlate_point(const double* y1, const double* y2, int64_t n, double fs, int64_t tdoa,
                        double fdoa, double* out) {
    REF_GUARD({
        *out = correlate_point(make_cap(y1, n, fs, gps_l1_freq_hz), make_cap(y2, n, fs, gps_l1_freq_hz),
                               PairOffsets{tdoa, fdoa});
    })
}

// offsets: `count` records laid out exactly as digeo::PairOffsets {int64, double}
int ref_correlate_batch(const char* backend, unsigned workers, const double* y1, const double* y2,
                        int64_t n, double fs, const void* offsets, int64_t count,
                        int64_t batch_size, double* out) {
    static_assert(sizeof(PairOffsets) == 16, "PairOffsets layout");
    REF_GUARD({
        const auto be = make_backend(backend, workers);
        const auto session =
            be->stage(make_cap(y1, n, fs, gps_l1_freq_hz), make_cap(y2, n, fs, gps_l1_freq_hz));
        const auto* off = static_cast<const PairOffsets*>(offsets);
        const BatchPlan plan = plan_batches(static_cast<std::size_t>(count),
                                            static_cast<std::size_t>(batch_size));
        for (std::size_t b = 0; b < plan.batch_count(); ++b) {
            const auto [begin, end] = plan.batch_range(b);
            session->correlate_batch(std::span<const PairOffsets>(off + begin, end - begin),
                                     std::span<double>(out + begin, end - begin));
        }
    })
}

int ref_plan_batches(uint64_t n_points, uint64_t batch_size, uint64_t budget,
                     uint64_t capture_bytes, uint64_t* batch_count) {
    REF_GUARD({
        *batch_count = plan_batches(n_points, batch_size, budget, capture_bytes).batch_count();
    })
}

// --- driver (geolocate.hpp:41-146, correlate.hpp:102-201) -------------------
//
// states: [n_snap][n_rx][6]; captures: n_snap*n_rx pointers to n complex doubles.
// per_snapshot (nullable): [n_snap][P]. Detections written up to det_cap.
int ref_geolocate(int64_t n_snap, int64_t n_rx, int64_t n, double fs, double fc,
                  const double* states, const double* const* captures, const double* bounds4,
                  double spacing, double alt, const char* backend, unsigned workers,
                  uint64_t batch_size, double k_sigma, int radius, int normalize,
                  double* accumulated, double* per_snapshot, int64_t* n_det, int64_t det_cap,
                  int64_t* det_index, double* det_score, double* det_z, double* det_lat,
                  double* det_lon) {
    REF_GUARD({
        std::vector<Snapshot> snaps(static_cast<std::size_t>(n_snap));
        for (int64_t s = 0; s < n_snap; ++s) {
            for (int64_t r = 0; r < n_rx; ++r) {
                snaps[s].states.push_back(make_state(states + (s * n_rx + r) * 6));
                snaps[s].captures.push_back(make_cap(captures[s * n_rx + r], n, fs, fc));
            }
        }
        const auto grid = std::make_shared<const CandidateGrid>(build_candidate_grid(
            {bounds4[0], bounds4[1], bounds4[2], bounds4[3]}, spacing, alt));
        GeolocateOptions opt;
        opt.backend_name = backend;
        opt.workers = workers;
        opt.batch_size = batch_size;
        opt.k_sigma = k_sigma;
        opt.exclusion_radius_cells = radius;
        opt.normalize_per_snapshot = normalize != 0;
        const GeolocateResult res = geolocate_snapshots(snaps, grid, opt);
        const std::size_t P = grid->size();
        if (accumulated) std::memcpy(accumulated, res.accumulated.values.data(), P * sizeof(double));
        if (per_snapshot)
            for (std::size_t s = 0; s < res.per_snapshot.size(); ++s)
                std::memcpy(per_snapshot + s * P, res.per_snapshot[s].values.data(),
                            P * sizeof(double));
        *n_det = static_cast<int64_t>(res.detections.size());
        for (std::size_t i = 0; i < res.detections.size() && static_cast<int64_t>(i) < det_cap; ++i) {
            det_index[i] = static_cast<int64_t>(res.detections[i].grid_index);
            det_score[i] = res.detections[i].score;
            det_z[i] = res.detections[i].score_zsigma;
            det_lat[i] = res.detections[i].location.lat_deg;
            det_lon[i] = res.detections[i].location.lon_deg;
        }
    })
}

// One pair, one snapshot, through the reference's own correlate_snapshot with
// the named backend — the exact reference CPU path (host offsets included).
// Returns the wall time of the call in *seconds.
int ref_correlate_snapshot_timed(int64_t n, double fs, double fc, const double* state_i6,
                                 const double* state_j6, const double* y1, const double* y2,
                                 const double* bounds4, double spacing, double alt,
                                 const char* backend, unsigned workers, uint64_t batch_size,
                                 double* out_values, double* seconds) {
    REF_GUARD({
        Snapshot snap;
        snap.states = {make_state(state_i6), make_state(state_j6)};
        snap.captures = {make_cap(y1, n, fs, fc), make_cap(y2, n, fs, fc)};
        const auto grid = std::make_shared<const CandidateGrid>(build_candidate_grid(
            {bounds4[0], bounds4[1], bounds4[2], bounds4[3]}, spacing, alt));
        const auto be = make_backend(backend, workers);
        const auto t0 = std::chrono::steady_clock::now();
        const CorrelationGrid g = correlate_snapshot(grid, snap, {0, 1}, *be, batch_size);
        const auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
        if (out_values) std::memcpy(out_values, g.values.data(), g.values.size() * sizeof(double));
    })
}

int ref_detect_emitters(const double* bounds4, double spacing, double alt, const double* values,
                        double k_sigma, int radius, int64_t* n_det, int64_t det_cap,
                        int64_t* det_index, double* det_score, double* det_z) {
    REF_GUARD({
        auto g = std::make_shared<const CandidateGrid>(build_candidate_grid(
            {bounds4[0], bounds4[1], bounds4[2], bounds4[3]}, spacing, alt));
        CorrelationGrid cg{g, std::vector<double>(values, values + g->size())};
        const auto det = detect_emitters(cg, k_sigma, radius);
        *n_det = static_cast<int64_t>(det.size());
        for (std::size_t i = 0; i < det.size() && static_cast<int64_t>(i) < det_cap; ++i) {
            det_index[i] = static_cast<int64_t>(det[i].grid_index);
            det_score[i] = det[i].score;
            det_z[i] = det[i].score_zsigma;
        }
    })
}

// --- BenchWorkload (bench.hpp:41-88): the reference's plugin-path workload ---
// y1, y2: n_samples complex doubles each; offsets: n_points {int64, double}
int ref_build_workload(uint64_t n_points, uint64_t n_samples, double fs, uint64_t seed,
                       double* y1, double* y2, void* offsets, uint64_t* checksum) {
    REF_GUARD({
        BenchWorkload w;
        w.n_points = n_points;
        w.capture_samples = n_samples;
        w.sample_rate_hz = fs;
        w.seed = seed;
        const auto d = detail::build_workload(w);
        std::memcpy(y1, d.y1.samples.data(), n_samples * sizeof(cplx));
        std::memcpy(y2, d.y2.samples.data(), n_samples * sizeof(cplx));
        std::memcpy(offsets, d.offsets.data(), n_points * sizeof(PairOffsets));
        *checksum = detail::workload_checksum(d);
    })
}

// --- DGIQ files (io.hpp:123-167) -------------------------------------------

int ref_write_iq(const char* path, const double* iq, int64_t n, double fs, double fc, double t0) {
    REF_GUARD({
        BasebandCapture c = make_cap(iq, n, fs, fc);
        c.start_time_s = t0;
        write_iq(c, path);
    })
}

// info4 = {sample_rate_hz, center_freq_hz, start_time_s, sample_count}; iq (nullable) gets
// the widened complex<double> samples
int ref_read_iq(const char* path, double* info4, double* iq, int64_t capacity) {
    REF_GUARD({
        const BasebandCapture c = read_iq(path);
        info4[0] = c.sample_rate_hz;
        info4[1] = c.center_freq_hz;
        info4[2] = c.start_time_s;
        info4[3] = static_cast<double>(c.samples.size());
        if (iq && static_cast<int64_t>(c.samples.size()) <= capacity)
            std::memcpy(iq, c.samples.data(), c.samples.size() * sizeof(cplx));
    })
}

}  // extern "C"

// --- surface / detection writers (io.hpp:171-280) --------------------------

namespace {
// axes6 = {lat_start, lat_step, n_lat, lon_start, lon_step, n_lon}
CorrelationGrid make_surface(const double* axes6, double alt, const double* values) {
    auto g = std::make_shared<CandidateGrid>();
    g->lat = GridAxis{axes6[0], axes6[1], static_cast<std::size_t>(axes6[2])};
    g->lon = GridAxis{axes6[3], axes6[4], static_cast<std::size_t>(axes6[5])};
    g->altitude_m = alt;
    return CorrelationGrid{g, std::vector<double>(values, values + g->size())};
}
}  // namespace

extern "C" {

int ref_write_grid(const char* path, const double* axes6, double alt, const double* values,
                   int csv) {
    REF_GUARD({
        write_grid(make_surface(axes6, alt, values), path,
                   csv ? GridFileFormat::csv : GridFileFormat::binary);
    })
}

int ref_render_heatmap(const char* path, const double* axes6, double alt, const double* values) {
    REF_GUARD({ render_heatmap(make_surface(axes6, alt, values), path); })
}

// det7 per detection: lat, lon, alt, grid_index, score, zsigma (index as double)
int ref_write_detections_csv(const char* path, const double* det6, int64_t n) {
    REF_GUARD({
        std::vector<EmitterEstimate> d(static_cast<std::size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            const double* r = det6 + 6 * i;
            d[i].location = GeodeticCoord{r[0], r[1], r[2]};
            d[i].grid_index = static_cast<std::size_t>(r[3]);
            d[i].score = r[4];
            d[i].score_zsigma = r[5];
        }
        write_detections_csv(d, path);
    })
}

// read_grid: axes6/alt/count first (values nullable), then the values
int ref_read_grid(const char* path, double* axes6, double* alt, double* values, int64_t capacity) {
    REF_GUARD({
        const CorrelationGrid g = read_grid(path);
        axes6[0] = g.grid->lat.start_deg;
        axes6[1] = g.grid->lat.step_deg;
        axes6[2] = static_cast<double>(g.grid->lat.count);
        axes6[3] = g.grid->lon.start_deg;
        axes6[4] = g.grid->lon.step_deg;
        axes6[5] = static_cast<double>(g.grid->lon.count);
        *alt = g.grid->altitude_m;
        if (values && static_cast<int64_t>(g.values.size()) <= capacity)
            std::memcpy(values, g.values.data(), g.values.size() * sizeof(double));
    })
}

}  // extern "C"
