// b200geo/digeo_plugin.hpp — header-only C++ shim that plugs the B200 engine
// into the reference library `digeo` (paths relative to its include/ dir).
//
//   #include "digeo/digeo.hpp"            // the integrator's reference headers
//   #include "b200geo/digeo_plugin.hpp"   // this file (links libb200geo.so)
//
//   b200::B200Backend gpu;                            // a digeo::CorrelationBackend
//   auto g = digeo::correlate_snapshot(grid, snap, {0, 1}, gpu);   // reference driver
//   auto r = b200::geolocate_snapshots(snapshots, grid, options);  // whole path on GPU
//   b200::write_grid(r.accumulated, "acc.csv", digeo::GridFileFormat::csv);  // io.hpp writers
//
// B200Backend replaces digeo::CorrelationBackend (backend.hpp:211-217) and its
// sessions replace CorrelationSession::correlate_batch (backend.hpp:196-209);
// b200::geolocate_snapshots has the signature and result type of
// digeo::geolocate_snapshots (geolocate.hpp:127-146) but moves the offsets,
// correlation, accumulation, peak and detection onto the GPU. C ABI error
// codes are rethrown as the reference's exception types.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <new>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "b200geo.h"
#include "digeo/backend.hpp"
#include "digeo/geolocate.hpp"
#include "digeo/io.hpp"

namespace b200 {

inline void check(int rc) {
    if (rc == DG_OK) return;
    const std::string msg = dg_last_error();
    if (rc == DG_EINVAL) throw std::invalid_argument(msg);
    if (rc == DG_ENOMEM) throw std::runtime_error("out of device memory: " + msg);
    throw std::runtime_error(msg);
}

static_assert(sizeof(digeo::PairOffsets) == sizeof(dg_pair_offsets), "PairOffsets layout");
static_assert(sizeof(digeo::EcefStateVector) == sizeof(dg_state), "EcefStateVector layout");
static_assert(sizeof(digeo::EcefVector) == sizeof(dg_ecef), "EcefVector layout");
static_assert(sizeof(digeo::cplx) == 2 * sizeof(double), "complex<double> layout");

class Engine {
public:
    explicit Engine(int device = 0) { check(dg_engine_create(device, &h_)); }
    explicit Engine(const std::vector<int>& devices) {
        check(dg_engine_create_multi(devices.data(), static_cast<int>(devices.size()), &h_));
    }
    ~Engine() { dg_engine_destroy(h_); }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    dg_engine* get() const { return h_; }

private:
    dg_engine* h_ = nullptr;
};

class B200Session final : public digeo::CorrelationSession {
public:
    explicit B200Session(dg_session* s) : s_(s) {}
    ~B200Session() override { dg_session_destroy(s_); }

    void correlate_batch(std::span<const digeo::PairOffsets> batch,
                         std::span<double> out) override {
        check(dg_correlate_batch(s_, reinterpret_cast<const dg_pair_offsets*>(batch.data()),
                                 static_cast<int64_t>(batch.size()), out.data(),
                                 static_cast<int64_t>(out.size())));
    }
    using digeo::CorrelationSession::correlate_batch;

private:
    dg_session* s_;
};

class B200Backend final : public digeo::CorrelationBackend {
public:
    explicit B200Backend(int device = 0)
        : engine_(std::make_shared<Engine>(device)), descriptor_{"b200", "parallel-batched", 1} {}
    /// One engine over several GPUs: geolocate_snapshots shards each run across
    /// them (dg_engine_create_multi); sessions run on devices.front().
    explicit B200Backend(const std::vector<int>& devices)
        : engine_(std::make_shared<Engine>(devices)),
          descriptor_{"b200", "parallel-batched", static_cast<unsigned>(devices.size())} {}

    /// The GPUs for a worker count as GeolocateOptions::workers reads it
    /// (geolocate.hpp:98): 0 = every visible GPU, else min(workers, visible).
    static std::vector<int> devices_for(unsigned workers) {
        int n = 0;
        check(dg_device_count(&n));
        const int m = workers ? std::min<int>(static_cast<int>(workers), n) : n;
        std::vector<int> d(static_cast<std::size_t>(std::max(m, 1)));
        for (std::size_t i = 0; i < d.size(); ++i) d[i] = static_cast<int>(i);
        return d;
    }

    const digeo::BackendDescriptor& descriptor() const override { return descriptor_; }

    std::unique_ptr<digeo::CorrelationSession> stage(const digeo::BasebandCapture& y1,
                                                     const digeo::BasebandCapture& y2) const override {
        dg_session* s = nullptr;
        check(dg_stage(engine_->get(), reinterpret_cast<const double*>(y1.samples.data()),
                       static_cast<int64_t>(y1.samples.size()), y1.sample_rate_hz,
                       reinterpret_cast<const double*>(y2.samples.data()),
                       static_cast<int64_t>(y2.samples.size()), y2.sample_rate_hz, &s));
        return std::make_unique<B200Session>(s);
    }

    const std::shared_ptr<Engine>& engine() const { return engine_; }

private:
    std::shared_ptr<Engine> engine_;
    digeo::BackendDescriptor descriptor_;
};

/// The reference's registry (backend.hpp:311-317) for this engine: "b200"
/// with `workers` GPUs (0 = all visible).
inline std::unique_ptr<digeo::CorrelationBackend> make_backend(const std::string& name,
                                                               unsigned workers = 0) {
    if (name == "b200") return std::make_unique<B200Backend>(B200Backend::devices_for(workers));
    throw std::invalid_argument("make_backend: unknown backend '" + name + "' (expected b200)");
}

/// geolocate.hpp:127-146 with the same inputs and result. `options.backend_name`
/// is ignored (the engine is the backend); everything after the captures is on
/// the GPU. The grid's eager ECEF points are uploaded as-is.
inline digeo::GeolocateResult geolocate_snapshots(const std::vector<digeo::Snapshot>& snapshots,
                                                  std::shared_ptr<const digeo::CandidateGrid> grid,
                                                  const digeo::GeolocateOptions& options = {},
                                                  const B200Backend* backend = nullptr) {
    if (snapshots.empty()) throw std::invalid_argument("geolocate_snapshots: no snapshots");
    if (!grid || grid->size() == 0) throw std::invalid_argument("correlate_snapshot: empty grid");
    std::unique_ptr<B200Backend> own;
    if (!backend)
        backend =
            (own = std::make_unique<B200Backend>(B200Backend::devices_for(options.workers))).get();
    dg_engine* eng = backend->engine()->get();

    const std::size_t R = snapshots.front().captures.size();
    if (R < 2) throw std::invalid_argument("correlate_snapshot_all_pairs: need >= 2 receivers");
    const auto& c0 = snapshots.front().captures.front();
    std::vector<dg_state> states;
    std::vector<const double*> caps;
    for (const auto& snap : snapshots) {
        if (snap.captures.size() != R || snap.states.size() != R)
            throw std::invalid_argument("geolocate_snapshots: receiver count differs");
        for (std::size_t r = 0; r < R; ++r) {
            const auto& c = snap.captures[r];
            c.validate();
            if (c.sample_rate_hz != c0.sample_rate_hz)
                throw std::invalid_argument("backend stage: sample rates differ");
            if (c.size() != c0.size())
                throw std::invalid_argument("backend stage: sample counts differ");
            // the reference takes each pair's wavelength from its first capture
            // (geolocate.hpp:55); the engine runs one carrier per run
            if (c.center_freq_hz != c0.center_freq_hz)
                throw std::invalid_argument("geolocate_snapshots: center frequencies differ");
            states.push_back(*reinterpret_cast<const dg_state*>(&snap.states[r]));
            caps.push_back(reinterpret_cast<const double*>(c.samples.data()));
        }
    }
    digeo::plan_batches(grid->size(), options.batch_size, options.memory_budget_bytes,
                        2 * c0.size() * sizeof(digeo::cplx));

    dg_grid* g = nullptr;
    check(dg_grid_from_points(eng, reinterpret_cast<const dg_ecef*>(grid->points.data()),
                              static_cast<int64_t>(grid->size()), grid->lat.start_deg,
                              grid->lat.step_deg, static_cast<int64_t>(grid->lat.count),
                              grid->lon.start_deg, grid->lon.step_deg,
                              static_cast<int64_t>(grid->lon.count), grid->altitude_m, &g));
    std::unique_ptr<dg_grid, void (*)(dg_grid*)> hold(g, dg_grid_destroy);

    dg_snapshots sn{};
    sn.n_snapshots = static_cast<int64_t>(snapshots.size());
    sn.n_receivers = static_cast<int64_t>(R);
    sn.n_samples = static_cast<int64_t>(c0.size());
    sn.sample_rate_hz = c0.sample_rate_hz;
    sn.center_freq_hz = c0.center_freq_hz;
    sn.states = states.data();
    sn.captures_iq = caps.data();

    dg_options opt;
    dg_options_default(&opt);
    opt.k_sigma = options.k_sigma;
    opt.exclusion_radius_cells = options.exclusion_radius_cells;
    opt.normalize_per_snapshot = options.normalize_per_snapshot ? 1 : 0;

    const std::size_t P = grid->size();
    digeo::GeolocateResult result;
    result.grid = grid;
    std::vector<double> per(snapshots.size() * P);
    result.accumulated = digeo::CorrelationGrid{grid, std::vector<double>(P)};
    std::vector<dg_emitter_estimate> dets(4096);
    dg_result res{};
    res.accumulated = result.accumulated.values.data();
    res.per_snapshot = per.data();
    res.detections = dets.data();
    res.detections_capacity = static_cast<int64_t>(dets.size());
    check(dg_geolocate_snapshots(eng, g, &sn, &opt, &res));

    result.per_snapshot.reserve(snapshots.size());
    for (std::size_t s = 0; s < snapshots.size(); ++s)
        result.per_snapshot.push_back(digeo::CorrelationGrid{
            grid, std::vector<double>(per.begin() + s * P, per.begin() + (s + 1) * P)});
    if (res.n_detections > res.detections_capacity) {  // the whole list, same surface
        dets.resize(static_cast<std::size_t>(res.n_detections));
        int64_t n = 0;
        check(dg_detect_emitters(eng, g, result.accumulated.values.data(), 0, options.k_sigma,
                                 options.exclusion_radius_cells, dets.data(),
                                 static_cast<int64_t>(dets.size()), &n));
        res.n_detections = n;
        res.detections_capacity = static_cast<int64_t>(dets.size());
    }
    const auto n_det = std::min<int64_t>(res.n_detections, res.detections_capacity);
    for (int64_t i = 0; i < n_det; ++i) {
        digeo::EmitterEstimate e;
        e.location = {dets[i].lat_deg, dets[i].lon_deg, dets[i].alt_m};
        e.grid_index = static_cast<std::size_t>(dets[i].grid_index);
        e.score = dets[i].score;
        e.score_zsigma = dets[i].score_zsigma;
        result.detections.push_back(e);
    }
    return result;
}

namespace detail {
inline std::unique_ptr<dg_grid, void (*)(dg_grid*)> axes_grid(dg_engine* eng,
                                                             const digeo::CorrelationGrid& g) {
    g.validate();
    const dg_grid_axes a{g.grid->lat.start_deg, g.grid->lat.step_deg,
                         static_cast<int64_t>(g.grid->lat.count), g.grid->lon.start_deg,
                         g.grid->lon.step_deg, static_cast<int64_t>(g.grid->lon.count),
                         g.grid->altitude_m};
    dg_grid* h = nullptr;
    check(dg_grid_from_axes(eng, &a, &h));
    return {h, dg_grid_destroy};
}
}  // namespace detail

/// io.hpp:171-203 (write_grid) and :245-268 (render_heatmap): the same files,
/// byte for byte, with the text / pixels produced on the GPU.
inline void write_grid(const digeo::CorrelationGrid& grid, const std::filesystem::path& path,
                       digeo::GridFileFormat format, const B200Backend* backend = nullptr) {
    std::unique_ptr<B200Backend> own;
    if (!backend) backend = (own = std::make_unique<B200Backend>()).get();
    dg_engine* eng = backend->engine()->get();
    auto g = detail::axes_grid(eng, grid);
    check(dg_write_grid(eng, g.get(), grid.values.data(), 0, path.string().c_str(),
                        format == digeo::GridFileFormat::csv ? DG_GRID_CSV : DG_GRID_BINARY));
}

inline void render_heatmap(const digeo::CorrelationGrid& grid, const std::filesystem::path& path,
                           const B200Backend* backend = nullptr) {
    std::unique_ptr<B200Backend> own;
    if (!backend) backend = (own = std::make_unique<B200Backend>()).get();
    dg_engine* eng = backend->engine()->get();
    auto g = detail::axes_grid(eng, grid);
    check(dg_render_heatmap(eng, g.get(), grid.values.data(), 0, path.string().c_str()));
}

/// io.hpp:270-280
inline void write_detections_csv(std::span<const digeo::EmitterEstimate> detections,
                                 const std::filesystem::path& path) {
    std::vector<dg_emitter_estimate> d;
    for (const auto& e : detections)
        d.push_back({e.location.lat_deg, e.location.lon_deg, e.location.alt_m,
                     static_cast<int64_t>(e.grid_index), e.score, e.score_zsigma});
    check(dg_write_detections_csv(d.data(), static_cast<int64_t>(d.size()),
                                  path.string().c_str()));
}

}  // namespace b200
