// Drop-in check: the reference's OWN driver code runs with the B200 engine
// plugged in through include/b200geo/digeo_plugin.hpp, and its answers are
// compared with the reference's SerialBackend / ParallelBatchedBackend.
// Built against the unmodified reference headers by oracle/Makefile (target
// `dropin`) into oracle/_ref/drop_in; run by tests/test_gpu_dropin.py.
// Prints one [PASS]/[FAIL] line per check; the exit code is the failure count.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "b200geo/digeo_plugin.hpp"
#include "digeo/config.hpp"
#include "digeo/geolocate.hpp"
#include "digeo/io.hpp"
#include "digeo/scene.hpp"

using namespace digeo;

namespace {

int failures = 0;

void check(bool ok, const std::string& what) {
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++failures;
}

double worst_rel(const std::vector<double>& a, const std::vector<double>& b) {
    double w = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        const double d = std::max({std::abs(a[i]), std::abs(b[i]), 1e-300});
        w = std::max(w, std::abs(a[i] - b[i]) / d);
    }
    return w;
}

BasebandCapture gauss_capture(std::size_t n, double fs, std::mt19937_64& eng) {
    std::normal_distribution<double> g(0.0, 1.0);
    BasebandCapture c;
    c.sample_rate_hz = fs;
    c.center_freq_hz = gps_l1_freq_hz;
    for (std::size_t i = 0; i < n; ++i) c.samples.emplace_back(g(eng), g(eng));
    return c;
}

}  // namespace

int main(int argc, char** argv) {
    const std::string cfg_path = argc > 1 ? argv[1] : "";
    const b200::B200Backend gpu;
    check(gpu.descriptor().name == "b200" && gpu.descriptor().kind == "parallel-batched",
          "descriptor {b200, parallel-batched}");

    // acceptance.cpp criterion 4 style: batches through the plugin interface
    {
        std::mt19937_64 eng(0xBA7C);
        const auto y1 = gauss_capture(2048, 2.048e6, eng), y2 = gauss_capture(2048, 2.048e6, eng);
        std::vector<PairOffsets> off;
        for (int i = 0; i < 10000; ++i)
            off.push_back({static_cast<std::int64_t>(eng() % 4096) - 2048,
                           (static_cast<double>(eng() >> 11) * 0x1.0p-53 - 0.5) * 1e6});
        const SerialBackend serial;
        const auto want = correlate_batch(serial, off, y1, y2);
        for (const std::size_t bs : {1ul, 7ul, 64ul, 1000ul}) {
            const BatchPlan plan = plan_batches(off.size(), bs);
            std::vector<double> out(off.size());
            const auto session = gpu.stage(y1, y2);
            for (std::size_t b = 0; b < plan.batch_count(); ++b) {
                const auto [lo, hi] = plan.batch_range(b);
                session->correlate_batch(std::span<const PairOffsets>(off).subspan(lo, hi - lo),
                                         std::span<double>(out).subspan(lo, hi - lo));
            }
            std::ostringstream m;
            m << "criterion-4 batches of " << bs << ": worst rel " << worst_rel(out, want);
            check(worst_rel(out, want) <= 1e-4, m.str());
        }
        bool threw = false;
        try {
            BasebandCapture bad = y2;
            bad.sample_rate_hz = 1e6;
            gpu.stage(y1, bad);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        check(threw, "mismatched captures throw std::invalid_argument");
    }

    if (cfg_path.empty()) return failures;

    // the reference's own correlate_snapshot / geolocate_snapshots on a desk scene
    const ScenarioConfig cfg = parse_scenario(cfg_path);
    const auto snaps = simulate_scenario(cfg.scenario);
    const auto grid = std::make_shared<const CandidateGrid>(build_candidate_grid(
        cfg.scenario.grid_bounds, cfg.scenario.grid_spacing_deg, cfg.scenario.grid_altitude_m));
    const ParallelBatchedBackend cpu;
    const auto want = correlate_snapshot(grid, snaps[0], {0, 1}, cpu, 4096);
    const auto got = correlate_snapshot(grid, snaps[0], {0, 1}, gpu, 4096);
    {
        std::ostringstream m;
        m << "reference correlate_snapshot with B200Backend: worst rel "
          << worst_rel(got.values, want.values);
        check(worst_rel(got.values, want.values) <= 1e-4, m.str());
    }
    GeolocateOptions opt = cfg.options;
    opt.backend_name = "parallel";
    opt.batch_size = 4096;
    const GeolocateResult ref = geolocate_snapshots(snaps, grid, opt);
    const GeolocateResult b2 = b200::geolocate_snapshots(snaps, grid, opt, &gpu);
    const auto am = [](const std::vector<double>& v) {
        return static_cast<std::size_t>(std::max_element(v.begin(), v.end()) - v.begin());
    };
    check(am(b2.accumulated.values) == am(ref.accumulated.values),
          "b200::geolocate_snapshots argmax == reference (" +
              std::to_string(am(ref.accumulated.values)) + ")");
    bool same = b2.detections.size() == ref.detections.size();
    for (std::size_t i = 0; same && i < ref.detections.size(); ++i)
        same = b2.detections[i].grid_index == ref.detections[i].grid_index &&
               b2.detections[i].location.lat_deg == ref.detections[i].location.lat_deg &&
               b2.detections[i].location.lon_deg == ref.detections[i].location.lon_deg;
    check(same, "detections identical (" + std::to_string(ref.detections.size()) + ")");
    double w = 0.0;
    for (std::size_t s = 0; s < ref.per_snapshot.size(); ++s)
        w = std::max(w, worst_rel(b2.per_snapshot[s].values, ref.per_snapshot[s].values));
    check(w <= 1e-4, "per-snapshot grids within 1e-4 (worst " + std::to_string(w) + ")");

    // the multi-GPU engine behind the same driver (dg_engine_create_multi): three
    // device slots (the box's GPUs, repeated when fewer are visible) shard the
    // run; every value must equal the one-GPU solve's bit for bit
    {
        const auto devs = b200::B200Backend::devices_for(3);
        std::vector<int> slots(3);
        for (int i = 0; i < 3; ++i) slots[i] = devs[static_cast<std::size_t>(i) % devs.size()];
        const b200::B200Backend multi(slots);
        check(multi.descriptor().workers == 3, "B200Backend over 3 device slots: workers == 3");
        const GeolocateResult m3 = b200::geolocate_snapshots(snaps, grid, opt, &multi);
        bool bits = m3.accumulated.values == b2.accumulated.values &&
                    m3.detections.size() == b2.detections.size();
        for (std::size_t s = 0; bits && s < b2.per_snapshot.size(); ++s)
            bits = m3.per_snapshot[s].values == b2.per_snapshot[s].values;
        check(bits, "multi-GPU engine: surfaces and detections bit-identical to one GPU");
        const auto reg = b200::make_backend("b200", 0);
        check(reg->descriptor().name == "b200" && reg->descriptor().workers >= 1,
              "b200::make_backend(\"b200\", 0): every visible GPU");
        bool threw = false;
        try {
            b200::make_backend("gpu");
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        check(threw, "make_backend(\"gpu\") rejected (test_backend.cpp:181)");
    }

    // the reference's accumulated surface through both writer sets (io.hpp:171-280)
    const auto tmp = std::filesystem::temp_directory_path();
    const auto slurp = [](const std::filesystem::path& p) {
        std::ifstream in(p, std::ios::binary);
        return std::string((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    };
    write_grid(ref.accumulated, tmp / "dg_ref.csv", GridFileFormat::csv);
    b200::write_grid(ref.accumulated, tmp / "dg_b2.csv", GridFileFormat::csv, &gpu);
    check(slurp(tmp / "dg_ref.csv") == slurp(tmp / "dg_b2.csv"), "write_grid csv byte-identical");
    write_grid(ref.accumulated, tmp / "dg_ref.dggr", GridFileFormat::binary);
    b200::write_grid(ref.accumulated, tmp / "dg_b2.dggr", GridFileFormat::binary, &gpu);
    check(slurp(tmp / "dg_ref.dggr") == slurp(tmp / "dg_b2.dggr"),
          "write_grid binary byte-identical");
    render_heatmap(ref.accumulated, tmp / "dg_ref.pgm");
    b200::render_heatmap(ref.accumulated, tmp / "dg_b2.pgm", &gpu);
    check(slurp(tmp / "dg_ref.pgm") == slurp(tmp / "dg_b2.pgm"), "render_heatmap byte-identical");
    write_detections_csv(ref.detections, tmp / "dg_ref_det.csv");
    b200::write_detections_csv(ref.detections, tmp / "dg_b2_det.csv");
    check(slurp(tmp / "dg_ref_det.csv") == slurp(tmp / "dg_b2_det.csv"),
          "write_detections_csv byte-identical");
    return failures;
}
