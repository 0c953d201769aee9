// C ABI of the device capture synthesis (include/b200geo.h dg_simulate_scenario;
// reference scene.hpp:200-310). The scenario arithmetic that fixes WHAT is
// synthesised (epochs, circular orbits, emitter positions, geometry, pads,
// integer/fractional delays, amplitudes, Doppler rotations, noise seeds) is
// restated here on the host with the reference's operation order, validation
// and messages (g++ -O2 -ffp-contract=off, like the reference), so those values
// are bit-identical; the per-sample work runs in dg_scene.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <numbers>
#include <string>
#include <vector>

#include "b200geo.h"
#include "dg_host.hpp"
#include "dg_internal.cuh"

using namespace dg;

namespace {

// geodesy.hpp:31-38
constexpr double kA = 6378137.0;
constexpr double kF = 1.0 / 298.257223563;
constexpr double kB = kA * (1.0 - kF);
constexpr double kE2 = kF * (2.0 - kF);
constexpr double kC = 299792458.0;    // geometry.hpp:32
constexpr double kMu = 3.986004418e14;  // orbit.hpp:30
inline double deg2rad(double d) { return d * std::numbers::pi / 180.0; }

struct V3 {
    double x, y, z;
    double norm() const { return std::sqrt(x * x + y * y + z * z); }
};

void validate_geodetic(double lat, double lon, double alt) {  // geodesy.hpp:69-78
    if (!(lat >= -90.0 && lat <= 90.0))
        raise(DG_EINVAL, "GeodeticCoord: lat_deg out of [-90, 90]: " + std::to_string(lat));
    if (!(lon >= -180.0 && lon < 180.0))
        raise(DG_EINVAL, "GeodeticCoord: lon_deg out of [-180, 180): " + std::to_string(lon));
    if (!std::isfinite(alt)) raise(DG_EINVAL, "GeodeticCoord: alt_m not finite");
}

V3 lla_to_ecef(double lat_deg, double lon_deg, double alt) {  // geodesy.hpp:82-92
    validate_geodetic(lat_deg, lon_deg, alt);
    const double lat = deg2rad(lat_deg), lon = deg2rad(lon_deg);
    const double slat = std::sin(lat), clat = std::cos(lat);
    const double slon = std::sin(lon), clon = std::cos(lon);
    const double n = kA / std::sqrt(1.0 - kE2 * slat * slat);
    return {(n + alt) * clat * clon, (n + alt) * clat * slon, (n * (1.0 - kE2) + alt) * slat};
}

void validate_state(const dg_state& s) {  // state.hpp:31-38
    const V3 p{s.position.x, s.position.y, s.position.z};
    const V3 v{s.velocity.x, s.velocity.y, s.velocity.z};
    if (!(std::isfinite(p.x) && std::isfinite(p.y) && std::isfinite(p.z) && std::isfinite(v.x) &&
          std::isfinite(v.y) && std::isfinite(v.z)))
        raise(DG_EINVAL, "EcefStateVector: non-finite component");
    if (!(p.norm() > kB)) raise(DG_EINVAL, "EcefStateVector: position below Earth surface");
    if (!(v.norm() < 1e5)) raise(DG_EINVAL, "EcefStateVector: velocity above 1e5 m/s");
}

struct Geo {
    double range, delay, doppler;
};

Geo predict_geometry(const V3& c, const dg_state& rx, double wl) {  // geometry.hpp:51-64
    const V3 r{rx.position.x - c.x, rx.position.y - c.y, rx.position.z - c.z};
    const double rho = r.norm();
    if (!(rho > 0.0)) raise(DG_EINVAL, "predict_geometry: candidate coincides with receiver");
    const double inv = 1.0 / rho;
    const V3 u{inv * r.x, inv * r.y, inv * r.z};
    const double d = u.x * rx.velocity.x + u.y * rx.velocity.y + u.z * rx.velocity.z;
    return {rho, rho / kC, -d / wl};
}

// orbit.hpp:37-74
std::vector<dg_state> propagate_circular_orbit(const dg_receiver_def& o,
                                               const std::vector<double>& epochs) {
    if (!(o.alt_m >= 200e3 && o.alt_m <= 2000e3))
        raise(DG_EINVAL, "propagate_circular_orbit: altitude out of [200 km, 2000 km]");
    const double radius = kA + o.alt_m;
    const double mean_motion = std::sqrt(kMu / (radius * radius * radius));
    const double speed = radius * mean_motion;
    const double inc = deg2rad(o.inclination_deg), raan = deg2rad(o.raan_deg);
    const double ci = std::cos(inc), si = std::sin(inc);
    const double co = std::cos(raan), so = std::sin(raan);
    const auto rotate = [&](double px, double py, double pz) {
        const double x1 = px;
        const double y1 = ci * py - si * pz;
        const double z1 = si * py + ci * pz;
        return dg_ecef{co * x1 - so * y1, so * x1 + co * y1, z1};
    };
    std::vector<dg_state> out;
    for (const double t : epochs) {
        const double u = deg2rad(o.phase_deg) + mean_motion * t;
        const double cu = std::cos(u), su = std::sin(u);
        out.push_back({rotate(radius * cu, radius * su, 0.0), rotate(-speed * su, speed * cu, 0.0)});
    }
    return out;
}

// ca_code.hpp:43-74: G1 / G2 10-stage LFSRs, PRN-specific G2 phase taps
std::array<int8_t, 1023> ca_code(int prn) {
    static constexpr int taps[32][2] = {
        {2, 6}, {3, 7}, {4, 8},  {5, 9},  {1, 9}, {2, 10}, {1, 8}, {2, 9},  {3, 10}, {2, 3}, {3, 4},
        {5, 6}, {6, 7}, {7, 8},  {8, 9},  {9, 10}, {1, 4}, {2, 5}, {3, 6},  {4, 7},  {5, 8}, {6, 9},
        {1, 3}, {4, 6}, {5, 7},  {6, 8},  {7, 9}, {8, 10}, {1, 6}, {2, 7}, {3, 8},  {4, 9}};
    if (prn < 1 || prn > 32)
        raise(DG_EINVAL, "generate_ca_code: prn out of 1..32: " + std::to_string(prn));
    int g1[10], g2[10];
    for (int i = 0; i < 10; ++i) g1[i] = g2[i] = 1;
    const int ta = taps[prn - 1][0], tb = taps[prn - 1][1];
    std::array<int8_t, 1023> chips{};
    for (int i = 0; i < 1023; ++i) {
        const int bit = g1[9] ^ (g2[ta - 1] ^ g2[tb - 1]);
        chips[i] = bit ? -1 : 1;
        const int f1 = g1[2] ^ g1[9];
        const int f2 = g2[1] ^ g2[2] ^ g2[5] ^ g2[7] ^ g2[8] ^ g2[9];
        for (int k = 9; k > 0; --k) {
            g1[k] = g1[k - 1];
            g2[k] = g2[k - 1];
        }
        g1[0] = f1;
        g2[0] = f2;
    }
    return chips;
}

uint64_t splitmix64(uint64_t x) {  // waveform.hpp:38-43
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

uint64_t derive_seed(uint64_t seed, uint64_t si, uint64_t ri) {  // scene.hpp:115-121
    uint64_t s = splitmix64(seed);
    s = splitmix64(s ^ (0xA24BAED4963EE407ull + si));
    s = splitmix64(s ^ (0x9FB21C651E98DF25ull + ri));
    return s;
}

int64_t sample_count(double fs, double duration) {  // waveform.hpp:101-108
    if (!(fs > 0.0)) raise(DG_EINVAL, "waveform: sample_rate_hz <= 0");
    if (!(duration > 0.0)) raise(DG_EINVAL, "waveform: duration_s <= 0");
    const auto n = static_cast<int64_t>(std::llround(duration * fs));
    if (n == 0) raise(DG_EINVAL, "waveform: duration shorter than one sample");
    return n;
}

void validate_scenario(const dg_scenario* sc) {  // Scenario::validate (scene.hpp:86-104)
    if (sc->n_receivers < 2) raise(DG_EINVAL, "Scenario: need >= 2 receivers");
    if (sc->snapshot_count < 1) raise(DG_EINVAL, "Scenario: snapshot_count < 1");
    if (!(sc->capture_duration_s > 0.0 && sc->capture_duration_s <= 0.05))
        raise(DG_EINVAL, "Scenario: capture_duration_s must be in (0, 0.05] for snapshot constancy");
    if (!(sc->snapshot_spacing_s > 0.0)) raise(DG_EINVAL, "Scenario: snapshot_spacing_s <= 0");
    if (!(sc->sample_rate_hz > 0.0)) raise(DG_EINVAL, "Scenario: sample_rate_hz <= 0");
    if (!(sc->center_freq_hz > 0.0)) raise(DG_EINVAL, "Scenario: center_freq_hz <= 0");
    if (!(sc->noise_power >= 0.0)) raise(DG_EINVAL, "Scenario: noise_power < 0");
    for (int64_t e = 0; e < sc->n_emitters; ++e) {
        const dg_emitter_def& em = sc->emitters[e];
        validate_geodetic(em.lat_deg, em.lon_deg, em.alt_m);
        if (!(em.ref_range_m > 0.0)) raise(DG_EINVAL, "EmitterDef: ref_range_m <= 0");
    }
    // a receiver is an orbit or a state table of snapshot_count rows (the table's
    // length is the caller's array; nothing to check beyond the pointer)
}

// per-(snapshot, emitter) transmit record and per-receiver channel (scene.hpp:283-297)
struct TxPlan {
    WaveParams wave;
    double start = 0.0;
    int64_t n_tx = 0;
    int log2n = 0;
    int guard = 0;
    bool any_frac = false;
    std::vector<double> frac, amplitude;
    std::vector<int64_t> shift;
    std::vector<double2> rotation;
};

WaveParams wave_of(const dg_emitter_def& em, double fs) {  // generate_waveform + spec checks
    WaveParams w{};
    switch (em.waveform) {
        case DG_WAVE_SPOOFER:
            if (em.prn < 1 || em.prn > 32) raise(DG_EINVAL, "SpooferSpec: prn out of 1..32");
            w.kind = kWaveSpoofer;
            w.seed = em.data_seed;
            break;
        case DG_WAVE_TONE:
            if (!(std::abs(em.tone_offset_hz) < fs / 2.0))
                raise(DG_EINVAL, "generate_tone: offset beyond Nyquist");
            w.kind = kWaveTone;
            w.a = em.tone_offset_hz;
            break;
        case DG_WAVE_CHIRP:
            if (!(em.bandwidth_hz > 0.0)) raise(DG_EINVAL, "ChirpSpec: bandwidth_hz <= 0");
            if (!(em.period_s > 0.0)) raise(DG_EINVAL, "ChirpSpec: period_s <= 0");
            if (!(em.bandwidth_hz < fs))
                raise(DG_EINVAL, "generate_chirp: bandwidth must be below the sample rate");
            w.kind = kWaveChirp;
            w.a = em.bandwidth_hz;
            w.b = em.period_s;
            break;
        case DG_WAVE_SAWTOOTH:
            if (!(em.bandwidth_hz > 0.0)) raise(DG_EINVAL, "SawtoothSpec: bandwidth_hz <= 0");
            if (!(em.period_s > 0.0)) raise(DG_EINVAL, "SawtoothSpec: chirp_period_s <= 0");
            if (!(em.bandwidth_hz < fs))
                raise(DG_EINVAL, "generate_sawtooth: bandwidth must be below the sample rate");
            w.kind = kWaveSawtooth;
            w.a = em.bandwidth_hz;
            w.b = em.period_s;
            break;
        default:
            raise(DG_EINVAL, "unknown waveform kind " + std::to_string(em.waveform));
    }
    return w;
}

}  // namespace

extern "C" {

int dg_scenario_samples(const dg_scenario* sc, int64_t* n_samples) {
    return guard([&] {
        if (!sc || !n_samples) raise(DG_EINVAL, "null argument");
        *n_samples = static_cast<int64_t>(std::llround(sc->capture_duration_s * sc->sample_rate_hz));
    });
}

int dg_simulate_scenario(dg_engine* eng, const dg_scenario* sc, dg_staged** staged_out,
                         double* captures_host, dg_state* states_host, double* epochs_host) {
    return guard([&] {
        if (!eng || !sc) raise(DG_EINVAL, "null argument");
        if (sc->n_receivers > 0 && !sc->receivers) raise(DG_EINVAL, "null receivers");
        if (sc->n_emitters > 0 && !sc->emitters) raise(DG_EINVAL, "null emitters");
        validate_scenario(sc);
        const int64_t S = sc->snapshot_count, R = sc->n_receivers, E = sc->n_emitters;
        const double fs = sc->sample_rate_hz;
        if (!(sc->center_freq_hz > 0.0)) raise(DG_EINVAL, "wavelength_m: center_freq_hz <= 0");
        const double wl = kC / sc->center_freq_hz;
        const int64_t N = static_cast<int64_t>(std::llround(sc->capture_duration_s * fs));
        if (N <= 0) raise(DG_EINVAL, "synthesize_received: empty output");

        // epochs and receiver states (scene.hpp:106-110, 236-247)
        std::vector<double> epochs(S);
        for (int64_t i = 0; i < S; ++i)
            epochs[i] = sc->start_time_s + static_cast<double>(i) * sc->snapshot_spacing_s;
        std::vector<dg_state> states(S * R);  // [S][R]
        for (int64_t r = 0; r < R; ++r) {
            const dg_receiver_def& rd = sc->receivers[r];
            std::vector<dg_state> col;
            if (rd.states)
                col.assign(rd.states, rd.states + S);
            else
                col = propagate_circular_orbit(rd, epochs);
            for (int64_t s = 0; s < S; ++s) states[s * R + r] = col[s];
        }

        // the channel of every (snapshot, emitter, receiver), in the reference's order
        std::vector<std::array<int8_t, 1023>> chips(E);
        for (int64_t e = 0; e < E; ++e)
            if (sc->emitters[e].waveform == DG_WAVE_SPOOFER && sc->emitters[e].prn >= 1 &&
                sc->emitters[e].prn <= 32)
                chips[e] = ca_code(sc->emitters[e].prn);
        std::vector<V3> pos(E);
        std::vector<TxPlan> plan(S * E);
        std::vector<uint64_t> seeds(S * R);
        const double ts = 1.0 / fs;
        for (int64_t s = 0; s < S; ++s) {
            const double epoch = epochs[s];
            for (int64_t e = 0; e < E; ++e) {
                const dg_emitter_def& em = sc->emitters[e];
                pos[e] = lla_to_ecef(em.lat_deg, em.lon_deg, em.alt_m);
                double max_delay = 0.0;
                for (int64_t r = 0; r < R; ++r)
                    max_delay = std::max(max_delay, predict_geometry(pos[e], states[s * R + r], wl).delay);
                const double pad_s = max_delay + 512.0 / fs;
                TxPlan& tp = plan[s * E + e];
                tp.wave = wave_of(em, fs);
                tp.n_tx = sample_count(fs, sc->capture_duration_s + 2.0 * pad_s);
                tp.start = epoch - pad_s;
                tp.guard = (int)std::min<int64_t>(128, tp.n_tx / 2);
                int l = 0;
                while ((int64_t(1) << l) < tp.n_tx) ++l;
                tp.log2n = l;
                for (int64_t r = 0; r < R; ++r) {  // synthesize_received (scene.hpp:199-232)
                    const dg_state& st = states[s * R + r];
                    validate_state(st);
                    const Geo g = predict_geometry(pos[e], st, wl);
                    const double offset = (epoch - g.delay - tp.start) * fs;
                    const double base = std::floor(offset);
                    const double frac = offset - base;
                    const auto shift = static_cast<int64_t>(base);
                    const int64_t last = shift + (N - 1) + (frac > 0.0 ? 1 : 0);
                    if (shift < tp.guard || last >= tp.n_tx - tp.guard)
                        raise(DG_EINVAL,
                              "synthesize_received: applied delay plus the filter guard exceeds "
                              "the transmit buffer");
                    const double amp = std::pow(10.0, em.ref_snr_db / 20.0) * em.ref_range_m / g.range;
                    const double th = 2.0 * std::numbers::pi * g.doppler / fs;
                    tp.frac.push_back(frac);
                    tp.shift.push_back(shift);
                    tp.amplitude.push_back(amp);
                    tp.rotation.push_back(make_double2(std::cos(th), std::sin(th)));
                    tp.any_frac |= frac != 0.0;
                }
                if (tp.any_frac && tp.log2n > fft_log2_max())
                    raise(DG_EINVAL, "simulate_scenario: transmit record longer than 2^" +
                                         std::to_string(fft_log2_max()) + " samples");
                if (tp.any_frac && tp.log2n < 3) tp.log2n = 3;  // zero padding is exact
            }
            for (int64_t r = 0; r < R; ++r)
                seeds[s * R + r] = derive_seed(sc->noise_seed, (uint64_t)s, (uint64_t)r);
        }

        // ---- device: per snapshot waveform -> spectrum -> per receiver advance,
        // then the emitter sum plus noise straight into the staged captures
        set_device(eng);
        StreamGuard sg(nullptr, eng->stream);
        Scratch scr(sg.st);
        auto st = std::make_unique<dg_staged>();
        st->eng = eng;
        st->S = S;
        st->R = R;
        st->N = N;
        st->stride = capture_stride(N);
        st->fs = fs;
        st->fc = sc->center_freq_hz;
        st->states = states;
        st->y32 = std::make_unique<DevMem>(S * R * st->stride * sizeof(float2));
        st->y64 = std::make_unique<DevMem>(S * R * st->stride * sizeof(double2));
        CK(cudaMemsetAsync(st->y64->p, 0, st->y64->bytes, sg.st));
        double2* y64 = static_cast<double2*>(st->y64->p) + kCapturePad;

        int8_t* d_chips = scr.alloc<int8_t>(std::max<int64_t>(E, 1) * 1023);
        for (int64_t e = 0; e < E; ++e)
            CK(cudaMemcpyAsync(d_chips + e * 1023, chips[e].data(), 1023, cudaMemcpyHostToDevice,
                               sg.st));
        uint64_t* d_seeds = scr.alloc<uint64_t>(S * R);
        CK(cudaMemcpyAsync(d_seeds, seeds.data(), S * R * sizeof(uint64_t), cudaMemcpyHostToDevice,
                           sg.st));
        std::vector<double2> rot(S * E * R);
        int64_t max_tx = 1, max_n = 1;
        for (int64_t s = 0; s < S; ++s)
            for (int64_t e = 0; e < E; ++e) {
                const TxPlan& tp = plan[s * E + e];
                for (int64_t r = 0; r < R; ++r) rot[(s * E + e) * R + r] = tp.rotation[r];
                max_tx = std::max(max_tx, tp.n_tx);
                if (tp.any_frac) max_n = std::max<int64_t>(max_n, int64_t(1) << tp.log2n);
            }
        double2* d_rot = scr.alloc<double2>(std::max<int64_t>(S * E * R, 1));
        CK(cudaMemcpyAsync(d_rot, rot.data(), rot.size() * sizeof(double2), cudaMemcpyHostToDevice,
                           sg.st));
        double2* tx = scr.alloc<double2>(E * max_tx);
        double2* spec = scr.alloc<double2>(E * max_n);
        double2* work = scr.alloc<double2>(max_n);
        double2* phasor = scr.alloc<double2>(std::max<int64_t>(E * R, 1) * N);
        double2* recv = scr.alloc<double2>(std::max<int64_t>(E * R, 1) * N);
        const double sigma = std::sqrt(sc->noise_power);
        for (int64_t s = 0; s < S; ++s) {
            if (E > 0) launch_phasors(d_rot + s * E * R, (int)(E * R), N, phasor, sg.st);
            for (int64_t e = 0; e < E; ++e) {
                const TxPlan& tp = plan[s * E + e];
                double2* txe = tx + e * max_tx;
                launch_waveform(tp.wave, tp.start, ts, tp.n_tx, d_chips + e * 1023, txe, sg.st);
                double2* spe = spec + e * max_n;
                if (tp.any_frac) launch_fractional_fwd(txe, tp.n_tx, tp.guard, tp.log2n, spe, sg.st);
                for (int64_t r = 0; r < R; ++r) {
                    const double2* ph = phasor + (e * R + r) * N;
                    double2* out = recv + (e * R + r) * N;
                    if (tp.frac[r] == 0.0)
                        launch_receive_direct(txe, tp.shift[r], N, tp.amplitude[r], ph, out, sg.st);
                    else
                        launch_fractional_inv(spe, tp.log2n, tp.frac[r], tp.shift[r], N,
                                              tp.amplitude[r], ph, work, out, sg.st);
                }
            }
            launch_noise_combine(d_seeds + s * R, 1, (int)R, (int)E, recv, N, sigma,
                                 sc->noise_power > 0.0 ? 1 : 0, y64 + s * R * st->stride,
                                 st->stride, sg.st);
        }
        launch_f64_to_f32(static_cast<const double2*>(st->y64->p), static_cast<float2*>(st->y32->p),
                          S * R * st->stride, sg.st);
        CK(cudaGetLastError());
        if (captures_host)
            CK(cudaMemcpy2DAsync(captures_host, N * sizeof(double2), y64,
                                 st->stride * sizeof(double2), N * sizeof(double2), S * R,
                                 cudaMemcpyDeviceToHost, sg.st));
        CK(cudaStreamSynchronize(sg.st));
        if (states_host) std::memcpy(states_host, states.data(), states.size() * sizeof(dg_state));
        if (epochs_host) std::memcpy(epochs_host, epochs.data(), epochs.size() * sizeof(double));
        if (staged_out) *staged_out = st.release();
    });
}

}  // extern "C"
