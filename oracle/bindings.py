"""ORACLE — TEST INFRASTRUCTURE ONLY (never imported by the product package).

ctypes bindings for the two CPU checkers built by ``oracle/Makefile``:

* ``RefLib``    — ``oracle/_ref/libdigeo_ref.so``: the unmodified reference
  headers (/root/reference/proj/include/digeo) behind ``oracle/ref_capi.cpp``.
* ``OracleLib`` — ``oracle/_build/liboracle.so``: the plain-C restatement
  ``oracle/digeo_oracle.c``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libdigeo_ref.so")
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int64)


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _i(a: np.ndarray):
    return a.ctypes.data_as(_ip)


class ReferenceError_(RuntimeError):
    """A std::exception thrown by the reference (code 1 = invalid_argument)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


PAIR_OFFSETS_DTYPE = np.dtype([("tdoa_samples", "<i8"), ("fdoa_hz", "<f8")])


@dataclass
class RefScene:
    n_snapshots: int
    n_rx: int
    n_samples: int
    fs: float
    fc: float
    bounds: tuple
    spacing: float
    alt: float
    k_sigma: float
    radius: int
    normalize: bool
    batch_size: int
    states: np.ndarray  # [S, R, 6]
    captures: np.ndarray  # [S, R, N] complex128


class RefLib:
    """The reference itself (compiled from /root/reference headers)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} missing: run `make -C oracle` (needs /root/reference) or "
                "__graft_entry__.build()")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_wavelength.restype = C.c_double
        L.ref_wavelength.argtypes = [C.c_double]
        for name in ("ref_scene_parse", "ref_scene_simulate", "ref_scene_capture",
                     "ref_scene_state", "ref_lla_to_ecef", "ref_build_grid",
                     "ref_predict_pair_offsets", "ref_correlate_point", "ref_correlate_batch",
                     "ref_plan_batches", "ref_geolocate", "ref_correlate_snapshot_timed",
                     "ref_detect_emitters", "ref_write_iq", "ref_read_iq"):
            getattr(L, name).restype = C.c_int
        L.ref_build_grid.argtypes = [_dp, C.c_double, C.c_double, C.c_uint64, _ip, _ip, _dp]
        L.ref_predict_pair_offsets.argtypes = [_dp, _dp, _dp, C.c_double, C.c_double, _ip, _dp]
        L.ref_correlate_point.argtypes = [_dp, _dp, C.c_int64, C.c_double, C.c_int64,
                                          C.c_double, _dp]
        L.ref_correlate_batch.argtypes = [C.c_char_p, C.c_uint, _dp, _dp, C.c_int64, C.c_double,
                                          C.c_void_p, C.c_int64, C.c_int64, _dp]
        L.ref_plan_batches.argtypes = [C.c_uint64] * 4 + [C.POINTER(C.c_uint64)]
        L.ref_lla_to_ecef.argtypes = [C.c_double, C.c_double, C.c_double, _dp]
        L.ref_scene_parse.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.ref_scene_free.argtypes = [C.c_void_p]
        L.ref_scene_simulate.argtypes = [C.c_void_p]
        L.ref_scene_info.argtypes = [C.c_void_p, _ip, _dp]
        L.ref_scene_capture.argtypes = [C.c_void_p, C.c_int64, C.c_int64, _dp]
        L.ref_scene_state.argtypes = [C.c_void_p, C.c_int64, C.c_int64, _dp]
        L.ref_geolocate.argtypes = [
            C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double, _dp, C.POINTER(_dp), _dp,
            C.c_double, C.c_double, C.c_char_p, C.c_uint, C.c_uint64, C.c_double, C.c_int,
            C.c_int, _dp, _dp, _ip, C.c_int64, _ip, _dp, _dp, _dp, _dp]
        L.ref_correlate_snapshot_timed.argtypes = [
            C.c_int64, C.c_double, C.c_double, _dp, _dp, _dp, _dp, _dp, C.c_double, C.c_double,
            C.c_char_p, C.c_uint, C.c_uint64, _dp, _dp]
        L.ref_detect_emitters.argtypes = [_dp, C.c_double, C.c_double, _dp, C.c_double, C.c_int,
                                          _ip, C.c_int64, _ip, _dp, _dp]
        L.ref_write_iq.argtypes = [C.c_char_p, _dp, C.c_int64, C.c_double, C.c_double,
                                   C.c_double]
        L.ref_read_iq.argtypes = [C.c_char_p, _dp, _dp, C.c_int64]
        L.ref_write_grid.argtypes = [C.c_char_p, _dp, C.c_double, _dp, C.c_int]
        L.ref_render_heatmap.argtypes = [C.c_char_p, _dp, C.c_double, _dp]
        L.ref_write_detections_csv.argtypes = [C.c_char_p, _dp, C.c_int64]
        L.ref_read_grid.argtypes = [C.c_char_p, _dp, _dp, _dp, C.c_int64]

    def _check(self, rc: int):
        if rc != 0:
            raise ReferenceError_(rc, self.lib.ref_last_error().decode())

    # -- DGIQ files (io.hpp:123-167) -----------------------------------------
    def write_iq(self, path, samples, fs, fc, t0=0.0):
        y = np.ascontiguousarray(samples, np.complex128)
        self._check(self.lib.ref_write_iq(str(path).encode(), y.ctypes.data_as(_dp), len(y), fs,
                                          fc, t0))

    def read_iq(self, path):
        """-> (samples complex128, sample_rate_hz, center_freq_hz, start_time_s)"""
        info = np.zeros(4)
        self._check(self.lib.ref_read_iq(str(path).encode(), _d(info), None, 0))
        n = int(info[3])
        out = np.zeros(n, np.complex128)
        self._check(self.lib.ref_read_iq(str(path).encode(), _d(info), out.ctypes.data_as(_dp),
                                         n))
        return out, info[0], info[1], info[2]

    # -- surface / detection writers (io.hpp:171-280) -------------------------
    @staticmethod
    def _axes(axes):
        """axes = (lat_start, lat_step, n_lat, lon_start, lon_step, n_lon)"""
        return np.asarray(axes, np.float64)

    def write_grid(self, path, axes, alt, values, csv: bool):
        a, v = self._axes(axes), np.ascontiguousarray(values, np.float64)
        self._check(self.lib.ref_write_grid(str(path).encode(), _d(a), alt, _d(v), int(csv)))

    def render_heatmap(self, path, axes, alt, values):
        a, v = self._axes(axes), np.ascontiguousarray(values, np.float64)
        self._check(self.lib.ref_render_heatmap(str(path).encode(), _d(a), alt, _d(v)))

    def write_detections_csv(self, path, rows):
        """rows: (lat, lon, alt, grid_index, score, zsigma) per detection"""
        d = np.ascontiguousarray(np.asarray(rows, np.float64).reshape(-1, 6))
        self._check(self.lib.ref_write_detections_csv(str(path).encode(), _d(d), len(d)))

    def read_grid(self, path):
        """-> (axes6, alt, values)"""
        a, alt = np.zeros(6), np.zeros(1)
        self._check(self.lib.ref_read_grid(str(path).encode(), _d(a), _d(alt), None, 0))
        v = np.zeros(int(a[2]) * int(a[5]))
        self._check(self.lib.ref_read_grid(str(path).encode(), _d(a), _d(alt), _d(v), len(v)))
        return a, float(alt[0]), v

    # -- scenes --------------------------------------------------------------
    def simulate(self, cfg_text: str) -> RefScene:
        h = C.c_void_p()
        self._check(self.lib.ref_scene_parse(cfg_text.encode(), C.byref(h)))
        try:
            self._check(self.lib.ref_scene_simulate(h))
            ints = np.zeros(3, np.int64)
            dbl = np.zeros(12, np.float64)
            self.lib.ref_scene_info(h, _i(ints), _d(dbl))
            S, R, N = (int(x) for x in ints)
            states = np.zeros((S, R, 6), np.float64)
            caps = np.zeros((S, R, N), np.complex128)
            for s in range(S):
                for r in range(R):
                    st = np.zeros(6, np.float64)
                    self._check(self.lib.ref_scene_state(h, s, r, _d(st)))
                    states[s, r] = st
                    buf = np.zeros(N, np.complex128)
                    self._check(self.lib.ref_scene_capture(h, s, r, buf.ctypes.data_as(_dp)))
                    caps[s, r] = buf
            return RefScene(S, R, N, dbl[0], dbl[1], tuple(dbl[2:6]), dbl[6], dbl[7], dbl[8],
                            int(dbl[9]), bool(dbl[10]), int(dbl[11]), states, caps)
        finally:
            self.lib.ref_scene_free(h)

    # -- geodesy / geometry --------------------------------------------------
    def wavelength(self, fc: float) -> float:
        return self.lib.ref_wavelength(fc)

    def lla_to_ecef(self, lat, lon, alt):
        out = np.zeros(3)
        self._check(self.lib.ref_lla_to_ecef(lat, lon, alt, _d(out)))
        return out

    def build_grid(self, bounds, spacing, alt=0.0, cap=20_000_000, points=True):
        b = np.asarray(bounds, np.float64)
        nl, nn = C.c_int64(), C.c_int64()
        self._check(self.lib.ref_build_grid(_d(b), spacing, alt, cap, C.byref(nl), C.byref(nn),
                                            None))
        pts = None
        if points:
            pts = np.zeros((nl.value * nn.value, 3))
            self._check(self.lib.ref_build_grid(_d(b), spacing, alt, cap, C.byref(nl),
                                                C.byref(nn), _d(pts)))
        return nl.value, nn.value, pts

    def predict_pair_offsets(self, cand, st_i, st_j, fs, wl):
        c = np.ascontiguousarray(cand, np.float64)
        a = np.ascontiguousarray(st_i, np.float64)
        b = np.ascontiguousarray(st_j, np.float64)
        d, f = C.c_int64(), C.c_double()
        self._check(self.lib.ref_predict_pair_offsets(_d(c), _d(a), _d(b), fs, wl, C.byref(d),
                                                      C.byref(f)))
        return d.value, f.value

    # -- correlation ---------------------------------------------------------
    def correlate_point(self, y1, y2, fs, tdoa, fdoa):
        y1 = np.ascontiguousarray(y1, np.complex128)
        y2 = np.ascontiguousarray(y2, np.complex128)
        out = C.c_double()
        self._check(self.lib.ref_correlate_point(y1.ctypes.data_as(_dp), y2.ctypes.data_as(_dp),
                                                 len(y1), fs, tdoa, fdoa, C.byref(out)))
        return out.value

    def correlate_batch(self, y1, y2, fs, offsets, backend="serial", workers=1, batch_size=None):
        y1 = np.ascontiguousarray(y1, np.complex128)
        y2 = np.ascontiguousarray(y2, np.complex128)
        off = np.ascontiguousarray(offsets, PAIR_OFFSETS_DTYPE)
        out = np.zeros(len(off))
        bs = batch_size or max(1, len(off))
        self._check(self.lib.ref_correlate_batch(
            backend.encode(), workers, y1.ctypes.data_as(_dp), y2.ctypes.data_as(_dp), len(y1),
            fs, off.ctypes.data, len(off), bs, _d(out)))
        return out

    def plan_batch_count(self, n_points, batch_size, budget=512 << 20, capture_bytes=0):
        out = C.c_uint64()
        self._check(self.lib.ref_plan_batches(n_points, batch_size, budget, capture_bytes,
                                              C.byref(out)))
        return out.value

    def geolocate(self, states, captures, fs, fc, bounds, spacing, alt=0.0, backend="serial",
                  workers=0, batch_size=8, k_sigma=5.0, radius=5, normalize=False,
                  per_snapshot=False, det_cap=4096):
        states = np.ascontiguousarray(states, np.float64)
        caps = np.ascontiguousarray(captures, np.complex128)
        S, R, N = caps.shape
        ptrs = (_dp * (S * R))(*[caps[s, r].ctypes.data_as(_dp) for s in range(S)
                                 for r in range(R)])
        n_lat, n_lon, _ = self.build_grid(bounds, spacing, alt, points=False)
        P = n_lat * n_lon
        acc = np.zeros(P)
        per = np.zeros((S, P)) if per_snapshot else None
        nd = C.c_int64()
        di = np.zeros(det_cap, np.int64)
        ds, dz, dla, dlo = (np.zeros(det_cap) for _ in range(4))
        b = np.asarray(bounds, np.float64)
        self._check(self.lib.ref_geolocate(
            S, R, N, fs, fc, _d(states), ptrs, _d(b), spacing, alt, backend.encode(), workers,
            batch_size, k_sigma, radius, int(normalize), _d(acc),
            _d(per) if per is not None else None, C.byref(nd), det_cap, _i(di), _d(ds), _d(dz),
            _d(dla), _d(dlo)))
        n = min(nd.value, det_cap)
        dets = [dict(grid_index=int(di[i]), score=float(ds[i]), zsigma=float(dz[i]),
                     lat_deg=float(dla[i]), lon_deg=float(dlo[i])) for i in range(n)]
        return dict(n_lat=n_lat, n_lon=n_lon, accumulated=acc, per_snapshot=per,
                    detections=dets)

    def correlate_snapshot_timed(self, st_i, st_j, y1, y2, fs, fc, bounds, spacing, alt=0.0,
                                 backend="parallel", workers=0, batch_size=4096,
                                 want_values=True):
        y1 = np.ascontiguousarray(y1, np.complex128)
        y2 = np.ascontiguousarray(y2, np.complex128)
        a = np.ascontiguousarray(st_i, np.float64)
        b_ = np.ascontiguousarray(st_j, np.float64)
        bb = np.asarray(bounds, np.float64)
        vals = None
        if want_values:
            n_lat, n_lon, _ = self.build_grid(bounds, spacing, alt, points=False)
            vals = np.zeros(n_lat * n_lon)
        sec = C.c_double()
        self._check(self.lib.ref_correlate_snapshot_timed(
            len(y1), fs, fc, _d(a), _d(b_), y1.ctypes.data_as(_dp), y2.ctypes.data_as(_dp),
            _d(bb), spacing, alt, backend.encode(), workers, batch_size,
            _d(vals) if vals is not None else None, C.byref(sec)))
        return sec.value, vals

    def build_workload(self, n_points, n_samples=4096, fs=5e6, seed=1):
        """bench.hpp:65-88 -> (y1, y2, offsets, workload_checksum)."""
        y1 = np.zeros(n_samples, np.complex128)
        y2 = np.zeros(n_samples, np.complex128)
        off = np.zeros(n_points, PAIR_OFFSETS_DTYPE)
        h = C.c_uint64()
        self._check(self.lib.ref_build_workload(
            C.c_uint64(n_points), C.c_uint64(n_samples), C.c_double(fs), C.c_uint64(seed),
            y1.ctypes.data_as(_dp), y2.ctypes.data_as(_dp), off.ctypes.data_as(C.c_void_p),
            C.byref(h)))
        return y1, y2, off, h.value

    def detect_emitters(self, bounds, spacing, alt, values, k_sigma=5.0, radius=5, cap=4096):
        v = np.ascontiguousarray(values, np.float64)
        b = np.asarray(bounds, np.float64)
        nd = C.c_int64()
        di = np.zeros(cap, np.int64)
        ds, dz = np.zeros(cap), np.zeros(cap)
        self._check(self.lib.ref_detect_emitters(_d(b), spacing, alt, _d(v), k_sigma, radius,
                                                 C.byref(nd), cap, _i(di), _d(ds), _d(dz)))
        n = min(nd.value, cap)
        return [(int(di[i]), float(ds[i]), float(dz[i])) for i in range(n)]


class OracleLib:
    """The plain-C restatement (oracle/digeo_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        L = self.lib = C.CDLL(path)
        L.orc_lla_to_ecef.argtypes = [C.c_double, C.c_double, C.c_double, _dp]
        L.orc_axis_count.restype = C.c_int64
        L.orc_axis_count.argtypes = [C.c_double, C.c_double]
        L.orc_build_grid.restype = C.c_int64
        L.orc_build_grid.argtypes = [_dp, C.c_double, C.c_double, C.c_uint64, _ip, _ip, _dp]
        L.orc_wavelength.restype = C.c_double
        L.orc_wavelength.argtypes = [C.c_double]
        L.orc_predict_pair_offsets.argtypes = [_dp, _dp, _dp, C.c_double, C.c_double, _ip, _dp]
        L.orc_correlate.restype = C.c_double
        L.orc_correlate.argtypes = [_dp, _dp, C.c_int64, C.c_int64, C.c_double, C.c_double]
        L.orc_correlate_snapshot.argtypes = [_dp, C.c_int64, _dp, _dp, _dp, _dp, C.c_int64,
                                             C.c_double, C.c_double, _dp]
        L.orc_accumulate.argtypes = [_dp, C.c_int64, C.c_int64, _dp]
        L.orc_argmax.restype = C.c_int64
        L.orc_argmax.argtypes = [_dp, C.c_int64]
        L.orc_detect_emitters.restype = C.c_int64
        L.orc_detect_emitters.argtypes = [_dp, C.c_int64, C.c_int64, C.c_double, C.c_int,
                                          C.c_int64, _ip, _dp, _dp]

    def lla_to_ecef(self, lat, lon, alt):
        out = np.zeros(3)
        self.lib.orc_lla_to_ecef(lat, lon, alt, _d(out))
        return out

    def build_grid(self, bounds, spacing, alt=0.0, cap=20_000_000):
        b = np.asarray(bounds, np.float64)
        nl, nn = C.c_int64(), C.c_int64()
        n = self.lib.orc_build_grid(_d(b), spacing, alt, cap, C.byref(nl), C.byref(nn), None)
        if n < 0:
            raise ValueError("invalid grid")
        pts = np.zeros((n, 3))
        self.lib.orc_build_grid(_d(b), spacing, alt, cap, C.byref(nl), C.byref(nn), _d(pts))
        return nl.value, nn.value, pts

    def wavelength(self, fc):
        return self.lib.orc_wavelength(fc)

    def predict_pair_offsets(self, cand, st_i, st_j, fs, wl):
        c = np.ascontiguousarray(cand, np.float64)
        a = np.ascontiguousarray(st_i, np.float64)
        b = np.ascontiguousarray(st_j, np.float64)
        d, f = C.c_int64(), C.c_double()
        self.lib.orc_predict_pair_offsets(_d(c), _d(a), _d(b), fs, wl, C.byref(d), C.byref(f))
        return d.value, f.value

    def correlate(self, y1, y2, tdoa, fdoa, fs):
        y1 = np.ascontiguousarray(y1, np.complex128)
        y2 = np.ascontiguousarray(y2, np.complex128)
        return self.lib.orc_correlate(y1.ctypes.data_as(_dp), y2.ctypes.data_as(_dp), len(y1),
                                      int(tdoa), float(fdoa), fs)

    def correlate_snapshot(self, points, st_i, st_j, y1, y2, fs, fc):
        pts = np.ascontiguousarray(points, np.float64)
        y1 = np.ascontiguousarray(y1, np.complex128)
        y2 = np.ascontiguousarray(y2, np.complex128)
        a = np.ascontiguousarray(st_i, np.float64)
        b = np.ascontiguousarray(st_j, np.float64)
        out = np.zeros(len(pts))
        self.lib.orc_correlate_snapshot(_d(pts), len(pts), _d(a), _d(b), y1.ctypes.data_as(_dp),
                                        y2.ctypes.data_as(_dp), len(y1), fs, fc, _d(out))
        return out

    def accumulate(self, grids):
        g = np.ascontiguousarray(grids, np.float64)
        out = np.zeros(g.shape[1])
        self.lib.orc_accumulate(_d(g), g.shape[0], g.shape[1], _d(out))
        return out

    def argmax(self, v):
        v = np.ascontiguousarray(v, np.float64)
        return int(self.lib.orc_argmax(_d(v), len(v)))

    def detect_emitters(self, values, n_lat, n_lon, k_sigma=5.0, radius=5, cap=4096):
        v = np.ascontiguousarray(values, np.float64)
        di = np.zeros(cap, np.int64)
        ds, dz = np.zeros(cap), np.zeros(cap)
        n = self.lib.orc_detect_emitters(_d(v), n_lat, n_lon, k_sigma, radius, cap, _i(di),
                                         _d(ds), _d(dz))
        if n < 0:
            raise ValueError("negative exclusion radius")
        n = min(n, cap)
        return [(int(di[i]), float(ds[i]), float(dz[i])) for i in range(n)]
