// C ABI of the surface / detection file formats (include/b200geo.h; reference
// io.hpp:169-280). Text and pixels are produced on the device (dg_writers.cu);
// this side writes the headers, then streams the device bytes to the file
// through the engine's pinned double buffer (the D2H copy of chunk i+1 overlaps
// the write of chunk i). Messages follow write_file_bytes / read_grid verbatim.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "b200geo.h"
#include "dg_host.hpp"
#include "dg_internal.cuh"

using namespace dg;

namespace {

constexpr size_t kChunk = 32ull << 20;
constexpr uint16_t kGridFormatVersion = 1;  // io.hpp:42

struct OutFile {  // write_file_bytes (io.hpp:114-119)
    std::FILE* f = nullptr;
    std::string path;
    explicit OutFile(const char* p) {
        if (!p) raise(DG_EINVAL, "null path");
        path = p;
        f = std::fopen(p, "wb");
        if (!f) raise(DG_ERUNTIME, "cannot open " + path + " for writing");
    }
    void write(const void* d, size_t n) {
        if (n && std::fwrite(d, 1, n, f) != n) raise(DG_ERUNTIME, "write failed: " + path);
    }
    void close() {
        std::FILE* t = f;
        f = nullptr;
        if (t && std::fclose(t) != 0) raise(DG_ERUNTIME, "write failed: " + path);
    }
    ~OutFile() {
        if (f) std::fclose(f);
    }
};

struct EventPair {
    cudaEvent_t e[2] = {nullptr, nullptr};
    EventPair() {
        for (auto& x : e) CK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    }
    ~EventPair() {
        for (auto x : e)
            if (x) cudaEventDestroy(x);
    }
};

void device_to_file(dg_engine* eng, cudaStream_t st, const void* dev, size_t bytes, OutFile& out) {
    if (!bytes) return;
    std::lock_guard<std::mutex> lk(eng->stage_mu);
    if (eng->stage_bytes < kChunk) {
        for (auto& p : eng->stage_host) {
            if (p) cudaFreeHost(p);
            p = nullptr;
        }
        eng->stage_bytes = 0;
        for (auto& p : eng->stage_host) CK(cudaHostAlloc(&p, kChunk, cudaHostAllocDefault));
        eng->stage_bytes = kChunk;
    }
    EventPair ev;
    const size_t n = (bytes + kChunk - 1) / kChunk;
    auto len = [&](size_t i) { return std::min(kChunk, bytes - i * kChunk); };
    auto issue = [&](size_t i) {
        CK(cudaMemcpyAsync(eng->stage_host[i & 1], static_cast<const char*>(dev) + i * kChunk,
                           len(i), cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(ev.e[i & 1], st));
    };
    issue(0);
    for (size_t i = 0; i < n; ++i) {
        if (i + 1 < n) issue(i + 1);  // its buffer was written out at step i - 1
        CK(cudaEventSynchronize(ev.e[i & 1]));
        out.write(eng->stage_host[i & 1], len(i));
    }
}

const double* device_values(const dg_grid* g, const double* values, int on_device, Scratch& sc) {
    if (on_device) return values;
    double* d = sc.alloc<double>(g->size());
    CK(cudaMemcpyAsync(d, values, g->size() * sizeof(double), cudaMemcpyHostToDevice, sc.st));
    return d;
}

// lattice axes of `g` (a slab's latitude axis starts at its first row)
double lat_value(const dg_grid* g, int64_t i) {
    return g->lat_start + static_cast<double>(g->row_offset + i) * g->lat_step;
}

void put_le(std::string& s, uint64_t v, int n) {  // detail::put_bytes (io.hpp:56-58)
    for (int i = 0; i < n; ++i) s.push_back(static_cast<char>((v >> (8 * i)) & 0xFF));
}
void put_f64(std::string& s, double v) {
    uint64_t b;
    std::memcpy(&b, &v, 8);
    put_le(s, b, 8);
}

void write_csv(dg_engine* eng, const dg_grid* g, const double* v, OutFile& out, Scratch& sc) {
    const int64_t n_lat = g->n_lat, n_lon = g->n_lon, P = g->size();
    char* lat_s = sc.alloc<char>((size_t)n_lat * kFmtSlot);
    char* lon_s = sc.alloc<char>((size_t)n_lon * kFmtSlot);
    char* val_s = sc.alloc<char>((size_t)P * kFmtSlot);
    uint8_t* lat_l = sc.alloc<uint8_t>(n_lat);
    uint8_t* lon_l = sc.alloc<uint8_t>(n_lon);
    uint8_t* val_l = sc.alloc<uint8_t>(P);
    launch_format_axis(g->lat_start, g->lat_step, g->row_offset, n_lat, lat_s, lat_l, sc.st);
    launch_format_axis(g->lon_start, g->lon_step, 0, n_lon, lon_s, lon_l, sc.st);
    launch_format_values(v, P, val_s, val_l, sc.st);
    int64_t* row_len = sc.alloc<int64_t>(P);
    int64_t* row_end = sc.alloc<int64_t>(P);
    const size_t tb = csv_scan_temp_bytes(P);
    void* temp = sc.alloc<char>(tb);
    launch_csv_offsets(lat_l, lon_l, val_l, n_lat, n_lon, row_len, row_end, temp, tb, sc.st);
    int64_t total = 0;
    CK(cudaMemcpyAsync(&total, row_end + P - 1, sizeof total, cudaMemcpyDeviceToHost, sc.st));
    CK(cudaStreamSynchronize(sc.st));
    char* body = sc.alloc<char>(total);
    launch_csv_emit(lat_s, lat_l, lon_s, lon_l, val_s, val_l, row_end, n_lat, n_lon, body, sc.st);
    CK(cudaGetLastError());
    static const char kHeader[] = "lat_deg,lon_deg,value\n";
    out.write(kHeader, sizeof kHeader - 1);
    device_to_file(eng, sc.st, body, (size_t)total, out);
}

}  // namespace

extern "C" {

int dg_write_grid(dg_engine* eng, const dg_grid* g, const double* values, int values_on_device,
                  const char* path, int format) {
    return guard([&] {
        if (!eng || !g || !values) raise(DG_EINVAL, "null argument");
        if (format != DG_GRID_CSV && format != DG_GRID_BINARY)
            raise(DG_EINVAL, "write_grid: unknown format");
        set_device(eng);
        StreamGuard sg(nullptr, eng->stream);
        Scratch sc(sg.st);
        const double* v = device_values(g, values, values_on_device, sc);
        OutFile out(path);
        if (format == DG_GRID_CSV) {
            write_csv(eng, g, v, out, sc);
        } else {  // io.hpp:187-202: 70-byte header, then the raw values
            std::string h;
            h.append("DGGR");
            put_le(h, kGridFormatVersion, 2);
            put_f64(h, lat_value(g, 0));
            put_f64(h, g->lat_step);
            put_le(h, (uint64_t)g->n_lat, 8);
            put_f64(h, g->lon_start);
            put_f64(h, g->lon_step);
            put_le(h, (uint64_t)g->n_lon, 8);
            put_f64(h, g->alt);
            put_le(h, (uint64_t)g->size(), 8);
            out.write(h.data(), h.size());
            device_to_file(eng, sg.st, v, g->size() * sizeof(double), out);
        }
        out.close();
    });
}

int dg_render_heatmap(dg_engine* eng, const dg_grid* g, const double* values, int values_on_device,
                      const char* path) {
    return guard([&] {
        if (!eng || !g || !values) raise(DG_EINVAL, "null argument");
        set_device(eng);
        StreamGuard sg(nullptr, eng->stream);
        Scratch sc(sg.st);
        const double* v = device_values(g, values, values_on_device, sc);
        const int64_t P = g->size();
        double2* part = sc.alloc<double2>(256);
        double2* mm = sc.alloc<double2>(1);
        launch_minmax(v, P, part, mm, sg.st);
        double2 h{};
        CK(cudaMemcpyAsync(&h, mm, sizeof h, cudaMemcpyDeviceToHost, sg.st));
        CK(cudaStreamSynchronize(sg.st));
        const double lo = h.x, hi = h.y;
        const double scale = (hi > lo) ? 65535.0 / (hi - lo) : 0.0;  // io.hpp:256
        uint8_t* px = sc.alloc<uint8_t>((size_t)P * 2);
        launch_heatmap(v, g->n_lat, g->n_lon, lo, scale, px, sg.st);
        CK(cudaGetLastError());
        const std::string head = "P5\n" + std::to_string(g->n_lon) + " " +
                                 std::to_string(g->n_lat) + "\n65535\n";
        OutFile out(path);
        out.write(head.data(), head.size());
        device_to_file(eng, sg.st, px, (size_t)P * 2, out);
        out.close();
    });
}

int dg_write_detections_csv(const dg_emitter_estimate* d, int64_t n, const char* path) {
    // io.hpp:270-280 (a handful of rows: the C library formats them, as there)
    return guard([&] {
        if (n < 0 || (n > 0 && !d)) raise(DG_EINVAL, "null argument");
        std::string s = "lat_deg,lon_deg,alt_m,grid_index,score,score_zsigma\n";
        char row[192];
        for (int64_t i = 0; i < n; ++i) {
            std::snprintf(row, sizeof row, "%.17g,%.17g,%.17g,%zu,%.17g,%.17g\n", d[i].lat_deg,
                          d[i].lon_deg, d[i].alt_m, static_cast<size_t>(d[i].grid_index),
                          d[i].score, d[i].score_zsigma);
            s += row;
        }
        OutFile out(path);
        out.write(s.data(), s.size());
        out.close();
    });
}

int dg_read_grid(const char* path, dg_grid_axes* axes, double* values, int64_t capacity) {
    // read_grid (io.hpp:205-240): the same checks in the same order
    return guard([&] {
        if (!path || !axes) raise(DG_EINVAL, "null argument");
        const std::string p(path);
        std::FILE* f = std::fopen(path, "rb");
        if (!f) raise(DG_ERUNTIME, "cannot open " + p);
        struct Closer {
            std::FILE* f;
            ~Closer() { std::fclose(f); }
        } closer{f};
        unsigned char hb[70];
        const size_t got = std::fread(hb, 1, sizeof hb, f);
        const std::string ctx = "read_grid(" + p + ")";
        if (got < 4) raise(DG_ERUNTIME, ctx + ": truncated file");
        if (std::memcmp(hb, "DGGR", 4) != 0) raise(DG_ERUNTIME, "read_grid: bad magic in " + p);
        if (got < 6) raise(DG_ERUNTIME, ctx + ": truncated file");
        const unsigned version = hb[4] | (hb[5] << 8);
        if (version != kGridFormatVersion)
            raise(DG_ERUNTIME, "read_grid: unsupported version " + std::to_string(version));
        if (got < 70) raise(DG_ERUNTIME, ctx + ": truncated file");
        uint64_t nlat = 0, nlon = 0, count = 0;
        std::memcpy(&axes->lat_start_deg, hb + 6, 8);  // little-endian host
        std::memcpy(&axes->lat_step_deg, hb + 14, 8);
        std::memcpy(&nlat, hb + 22, 8);
        std::memcpy(&axes->lon_start_deg, hb + 30, 8);
        std::memcpy(&axes->lon_step_deg, hb + 38, 8);
        std::memcpy(&nlon, hb + 46, 8);
        std::memcpy(&axes->altitude_m, hb + 54, 8);
        std::memcpy(&count, hb + 62, 8);
        axes->lat_count = (int64_t)nlat;
        axes->lon_count = (int64_t)nlon;
        if (count != nlat * nlon)
            raise(DG_ERUNTIME, "read_grid: value count does not match lattice in " + p);
        if (std::fseek(f, 0, SEEK_END) != 0) raise(DG_ERUNTIME, "cannot open " + p);
        const long end = std::ftell(f);
        if (end < 70 || (uint64_t)(end - 70) != count * 8)
            raise(DG_ERUNTIME, "read_grid: payload length mismatch in " + p);
        if (values && (int64_t)count <= capacity) {
            std::fseek(f, 70, SEEK_SET);
            if (std::fread(values, 8, count, f) != count) raise(DG_ERUNTIME, ctx + ": truncated file");
        }
    });
}

int dg_format_g17(dg_engine* eng, const double* values, int64_t n, char* slots, uint8_t* lengths) {
    return guard([&] {
        if (!eng || (n > 0 && (!values || !slots || !lengths))) raise(DG_EINVAL, "null argument");
        if (n <= 0) return;
        set_device(eng);
        StreamGuard sg(nullptr, eng->stream);
        Scratch sc(sg.st);
        double* v = sc.alloc<double>(n);
        char* s = sc.alloc<char>((size_t)n * kFmtSlot);
        uint8_t* l = sc.alloc<uint8_t>(n);
        CK(cudaMemcpyAsync(v, values, n * sizeof(double), cudaMemcpyHostToDevice, sg.st));
        launch_format_values(v, n, s, l, sg.st);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(slots, s, (size_t)n * kFmtSlot, cudaMemcpyDeviceToHost, sg.st));
        CK(cudaMemcpyAsync(lengths, l, n, cudaMemcpyDeviceToHost, sg.st));
        CK(cudaStreamSynchronize(sg.st));
    });
}

}  // extern "C"
