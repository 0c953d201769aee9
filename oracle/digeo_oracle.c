/*
 * ORACLE — TEST INFRASTRUCTURE ONLY. NOT PART OF THE PRODUCT PATH.
 *
 * Plain-C restatement of the reference (`digeo`) algorithms on the hot path,
 * used by tests/ as the CPU checker and by bench.py's cpu_baseline leg as the
 * "port" baseline when oracle/_ref is unavailable. Each function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 *
 * Parity pinning: tests/test_oracle.py checks every function here against the
 * reference itself compiled into oracle/_ref/libdigeo_ref.so (bit-exact), and
 * against the committed golden vectors in tests/golden/.
 *
 * Floating-point contract: compiled with -O2 -ffp-contract=off (see
 * oracle/Makefile), i.e. plain IEEE double add/mul/div/sqrt in the reference's
 * evaluation order — the same code the reference gets from g++ -O2 on
 * x86-64 without FMA.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_PI 3.14159265358979323846264338327950288
#define WGS84_A 6378137.0
#define WGS84_F (1.0 / 298.257223563)
#define C_LIGHT 299792458.0

/* geodesy.hpp:34-35 — constexpr f*(2-f) */
static double wgs84_e2(void) { return WGS84_F * (2.0 - WGS84_F); }

/* geodesy.hpp:38 — deg * pi / 180 (left to right) */
static double deg2rad(double d) { return d * ORC_PI / 180.0; }

/* geodesy.hpp:82-92 (validation done by the caller) */
void orc_lla_to_ecef(double lat_deg, double lon_deg, double alt, double out[3]) {
    const double lat = deg2rad(lat_deg), lon = deg2rad(lon_deg);
    const double slat = sin(lat), clat = cos(lat), slon = sin(lon), clon = cos(lon);
    const double e2 = wgs84_e2();
    const double n = WGS84_A / sqrt(1.0 - e2 * slat * slat);
    out[0] = (n + alt) * clat * clon;
    out[1] = (n + alt) * clat * slon;
    out[2] = (n * (1.0 - e2) + alt) * slat;
}

/* geodesy.hpp:175-177 */
int64_t orc_axis_count(double span, double step) {
    return (int64_t)floor(span / step + 1e-6) + 1;
}

/* geodesy.hpp:182-207: lat-major ECEF lattice; returns point count or -1
 * (the reference's invalid_argument cases). points may be NULL. */
int64_t orc_build_grid(const double b[4], double spacing, double alt, uint64_t cap,
                       int64_t* n_lat, int64_t* n_lon, double* points) {
    /* LatLonBounds::validate (geodesy.hpp:132-137): lat_min, lat_max and
     * lon_min range-checked; lon_max is not (reference quirk). */
    if (!(b[0] >= -90.0 && b[0] <= 90.0) || !(b[1] >= -90.0 && b[1] <= 90.0)) return -1;
    if (!(b[2] >= -180.0 && b[2] < 180.0)) return -1;
    if (b[1] < b[0] || b[3] < b[2]) return -1;
    if (!(spacing > 0.0) || !isfinite(alt)) return -1;
    *n_lat = orc_axis_count(b[1] - b[0], spacing);
    *n_lon = orc_axis_count(b[3] - b[2], spacing);
    const int64_t n = *n_lat * *n_lon;
    if ((uint64_t)n > cap) return -1;
    if (points) {
        for (int64_t i = 0; i < *n_lat; ++i) {
            const double lat = b[0] + (double)i * spacing; /* GridAxis::value :145 */
            if (!(lat >= -90.0 && lat <= 90.0)) return -1;
            for (int64_t j = 0; j < *n_lon; ++j) {
                const double lon = b[2] + (double)j * spacing;
                if (!(lon >= -180.0 && lon < 180.0)) return -1; /* lla_to_ecef validate */
                orc_lla_to_ecef(lat, lon, alt, points + 3 * (i * *n_lon + j));
            }
        }
    }
    return n;
}

/* geometry.hpp:36-39 */
double orc_wavelength(double fc) { return C_LIGHT / fc; }

/* geometry.hpp:51-64; returns delay_s and doppler_hz. Norm per geodesy.hpp:48,
 * dot per geodesy.hpp:61-63, (1/rho)*r per :59. */
static void orc_predict_geometry(const double c[3], const double rx[6], double wl,
                                 double* delay_s, double* doppler_hz) {
    const double rx_ = rx[0] - c[0], ry = rx[1] - c[1], rz = rx[2] - c[2];
    const double rho = sqrt(rx_ * rx_ + ry * ry + rz * rz);
    *delay_s = rho / C_LIGHT;
    const double inv = 1.0 / rho;
    const double ux = inv * rx_, uy = inv * ry, uz = inv * rz;
    *doppler_hz = -(ux * rx[3] + uy * rx[4] + uz * rx[5]) / wl;
}

/* geometry.hpp:73-83 — llround: ties away from zero */
void orc_predict_pair_offsets(const double c[3], const double rx_i[6], const double rx_j[6],
                              double fs, double wl, int64_t* tdoa, double* fdoa) {
    double di, fi, dj, fj;
    orc_predict_geometry(c, rx_i, wl, &di, &fi);
    orc_predict_geometry(c, rx_j, wl, &dj, &fj);
    const double tdoa_s = dj - di;
    *tdoa = llround(tdoa_s * fs);
    *fdoa = fj - fi;
}

/* correlate.hpp:44-71 — single FP64 phasor recurrence over the overlap.
 * y1, y2: n interleaved complex doubles (std::complex<double> layout). */
double orc_correlate(const double* y1, const double* y2, int64_t n, int64_t tdoa, double fdoa,
                     double fs) {
    const int64_t k_begin = tdoa < 0 ? -tdoa : 0;
    const int64_t k_end = n - tdoa < n ? n - tdoa : n;
    if (k_begin >= k_end) return 0.0;
    const double step = 2.0 * ORC_PI * fdoa / fs;
    const double rot_re = cos(step), rot_im = sin(step);
    const double phase0 = step * (double)k_begin;
    double ph_re = cos(phase0), ph_im = sin(phase0);
    double acc_re = 0.0, acc_im = 0.0;
    const double* b = y2 + 2 * tdoa;
    for (int64_t k = k_begin; k < k_end; ++k) {
        const double a_re = y1[2 * k], a_im = y1[2 * k + 1];
        const double b_re = b[2 * k], b_im = -b[2 * k + 1];
        const double p_re = a_re * b_re - a_im * b_im;
        const double p_im = a_re * b_im + a_im * b_re;
        acc_re += p_re * ph_re - p_im * ph_im;
        acc_im += p_re * ph_im + p_im * ph_re;
        const double next_re = ph_re * rot_re - ph_im * rot_im;
        ph_im = ph_re * rot_im + ph_im * rot_re;
        ph_re = next_re;
    }
    return sqrt(acc_re * acc_re + acc_im * acc_im);
}

/* geolocate.hpp:41-75 for one pair and one snapshot over a lattice of points:
 * offsets per point (geometry.hpp:73-83) then the kernel. */
void orc_correlate_snapshot(const double* points, int64_t P, const double* st_i,
                            const double* st_j, const double* y1, const double* y2, int64_t n,
                            double fs, double fc, double* out) {
    const double wl = orc_wavelength(fc);
    for (int64_t p = 0; p < P; ++p) {
        int64_t d;
        double f;
        orc_predict_pair_offsets(points + 3 * p, st_i, st_j, fs, wl, &d, &f);
        out[p] = orc_correlate(y1, y2, n, d, f, fs);
    }
}

/* correlate.hpp:102-113 — acc = g0; acc += g_s in order */
void orc_accumulate(const double* grids, int64_t n_grids, int64_t P, double* out) {
    memcpy(out, grids, (size_t)P * sizeof(double));
    for (int64_t s = 1; s < n_grids; ++s)
        for (int64_t k = 0; k < P; ++k) out[k] += grids[s * P + k];
}

/* std::max_element: first maximum (tests/test_geolocate.cpp:30-33) */
int64_t orc_argmax(const double* v, int64_t P) {
    int64_t best = 0;
    for (int64_t k = 1; k < P; ++k)
        if (v[best] < v[k]) best = k;
    return best;
}

typedef struct {
    int64_t ilat, ilon;
    double score;
} orc_cand;

static int orc_cand_cmp(const void* pa, const void* pb) {
    const orc_cand* a = (const orc_cand*)pa;
    const orc_cand* b = (const orc_cand*)pb;
    if (a->score != b->score) return a->score > b->score ? -1 : 1;
    const int64_t ka = a->ilat * 1000000 + a->ilon, kb = b->ilat * 1000000 + b->ilon;
    return ka < kb ? -1 : (ka > kb ? 1 : 0);
}

/* correlate.hpp:127-201. Returns the number of detections (written up to cap)
 * or -1 for a negative radius. */
int64_t orc_detect_emitters(const double* v, int64_t n_lat, int64_t n_lon, double k_sigma,
                            int radius, int64_t cap, int64_t* out_index, double* out_score,
                            double* out_z) {
    if (radius < 0) return -1;
    const int64_t P = n_lat * n_lon;
    const double n = (double)P;
    double mean = 0.0;
    for (int64_t k = 0; k < P; ++k) mean += v[k];
    mean /= n;
    double var = 0.0;
    for (int64_t k = 0; k < P; ++k) var += (v[k] - mean) * (v[k] - mean);
    var /= n;
    const double sigma = sqrt(var);
    if (sigma == 0.0) return 0;
    const double thr = mean + k_sigma * sigma;
    int64_t n_peaks = 0, cap_peaks = 64;
    orc_cand* peaks = (orc_cand*)malloc((size_t)cap_peaks * sizeof(orc_cand));
    for (int64_t i = 0; i < n_lat; ++i)
        for (int64_t j = 0; j < n_lon; ++j) {
            const double x = v[i * n_lon + j];
            if (x <= thr) continue;
            int is_max = 1;
            for (int64_t di = -1; di <= 1 && is_max; ++di)
                for (int64_t dj = -1; dj <= 1 && is_max; ++dj) {
                    if (di == 0 && dj == 0) continue;
                    const int64_t ni = i + di, nj = j + dj;
                    if (ni < 0 || ni >= n_lat || nj < 0 || nj >= n_lon) continue;
                    if (v[ni * n_lon + nj] > x) is_max = 0;
                }
            if (!is_max) continue;
            if (n_peaks == cap_peaks) {
                cap_peaks *= 2;
                peaks = (orc_cand*)realloc(peaks, (size_t)cap_peaks * sizeof(orc_cand));
            }
            peaks[n_peaks].ilat = i;
            peaks[n_peaks].ilon = j;
            peaks[n_peaks].score = x;
            ++n_peaks;
        }
    qsort(peaks, (size_t)n_peaks, sizeof(orc_cand), orc_cand_cmp);
    int64_t n_acc = 0;
    orc_cand* acc = (orc_cand*)malloc((size_t)(n_peaks ? n_peaks : 1) * sizeof(orc_cand));
    for (int64_t c = 0; c < n_peaks; ++c) {
        int excluded = 0;
        for (int64_t a = 0; a < n_acc; ++a) {
            const int64_t dl = llabs(peaks[c].ilat - acc[a].ilat);
            const int64_t dn = llabs(peaks[c].ilon - acc[a].ilon);
            if ((dl > dn ? dl : dn) <= radius) {
                excluded = 1;
                break;
            }
        }
        if (excluded) continue;
        if (n_acc < cap) {
            out_index[n_acc] = peaks[c].ilat * n_lon + peaks[c].ilon;
            out_score[n_acc] = peaks[c].score;
            out_z[n_acc] = (peaks[c].score - mean) / sigma;
        }
        acc[n_acc++] = peaks[c];
    }
    free(peaks);
    free(acc);
    return n_acc;
}
