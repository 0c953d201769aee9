"""Algorithm-1 driver — host mirror of digeo geolocate.hpp:41-146 over the C ABI.

``geolocate_snapshots`` runs the whole path on the GPU in one call: per
snapshot and receiver pair, bit-exact TDOA/FDOA for every candidate, the FP32
correlator, FP64 re-evaluation of the elements the tolerance needs, pair sum,
optional median normalisation, non-coherent accumulation, the exact peak
(argmax) and ``detect_emitters``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import check, lib
from .backend import (DEFAULT_MEMORY_BUDGET_BYTES, B200Backend, BasebandCapture,
                      CorrelationSession, plan_batches)
from .engine import Engine, default_engine
from .geodesy import CandidateGrid, GeodeticCoord

SPEED_OF_LIGHT_M_S = 299792458.0  # geometry.hpp:32
GPS_L1_FREQ_HZ = 1575.42e6        # geometry.hpp:33


def wavelength_m(center_freq_hz: float) -> float:
    """geometry.hpp:36-39"""
    if not (center_freq_hz > 0.0):
        raise ValueError("wavelength_m: center_freq_hz <= 0")
    return SPEED_OF_LIGHT_M_S / center_freq_hz


@dataclass
class Snapshot:
    """scene.hpp:66-70. states: [R, 6] (ECEF position xyz, velocity xyz)."""
    epoch_s: float
    states: np.ndarray
    captures: list


@dataclass
class CorrelationGrid:
    """correlate.hpp:89-98"""
    grid: CandidateGrid
    values: np.ndarray


@dataclass
class EmitterEstimate:
    """correlate.hpp:117-122"""
    location: GeodeticCoord
    grid_index: int
    score: float
    score_zsigma: float


@dataclass
class GeolocateOptions:
    """geolocate.hpp:96-104 (backend_name selects this engine: "b200")."""
    backend_name: str = "b200"
    workers: int = 0
    batch_size: int = 8
    memory_budget_bytes: int = DEFAULT_MEMORY_BUDGET_BYTES
    k_sigma: float = 5.0
    exclusion_radius_cells: int = 5
    normalize_per_snapshot: bool = False
    keep_per_snapshot: bool = True   # the reference always keeps them (geolocate.hpp:108)
    detect: bool = True
    patch_peak: bool = True  # exact FP64 values at the re-ranked near-peak cells of host surfaces


@dataclass
class GeolocateResult:
    """geolocate.hpp:106-111 plus the exact peak and run statistics."""
    grid: CandidateGrid
    per_snapshot: list
    accumulated: CorrelationGrid
    detections: list
    argmax_index: int = 0
    argmax_value: float = 0.0
    stats: dict = field(default_factory=dict)


def _pair_states(a) -> _capi.dg_state:
    v = np.asarray(a, np.float64).reshape(6)
    return _capi.dg_state(_capi.dg_ecef(*v[:3]), _capi.dg_ecef(*v[3:]))


def correlate_snapshot(grid: CandidateGrid, snapshot: Snapshot, pair, backend: B200Backend,
                       batch_size: int = 8,
                       memory_budget_bytes: int = DEFAULT_MEMORY_BUDGET_BYTES) -> CorrelationGrid:
    """geolocate.hpp:41-75 — offsets and correlation for the whole grid on the GPU."""
    if grid is None or grid.size() == 0:
        raise ValueError("correlate_snapshot: empty grid")
    i, j = pair
    n_rx = len(snapshot.captures)
    if i >= n_rx or j >= n_rx or i == j:
        raise ValueError("correlate_snapshot: bad receiver pair")
    y1, y2 = snapshot.captures[i], snapshot.captures[j]
    wavelength_m(y1.center_freq_hz)
    cap_bytes = (len(y1.samples) + len(y2.samples)) * 16
    plan_batches(grid.size(), batch_size, memory_budget_bytes, cap_bytes)
    session = backend.stage(y1, y2)
    out = np.zeros(grid.size(), np.float64)
    si, sj = _pair_states(snapshot.states[i]), _pair_states(snapshot.states[j])
    check(lib.dg_correlate_snapshot(session.handle, grid.handle, C.byref(si), C.byref(sj),
                                    float(y1.center_freq_hz),
                                    out.ctypes.data_as(C.POINTER(C.c_double))))
    return CorrelationGrid(grid, out)


def predict_offsets(grid: CandidateGrid, state_i, state_j, sample_rate_hz: float,
                    wavelength: float) -> np.ndarray:
    """predict_pair_offsets (geometry.hpp:73-83) for every grid point, on the GPU."""
    from .backend import PAIR_OFFSETS_DTYPE
    out = np.zeros(grid.size(), PAIR_OFFSETS_DTYPE)
    si, sj = _pair_states(state_i), _pair_states(state_j)
    check(lib.dg_predict_offsets(grid.engine.handle, grid.handle, C.byref(si), C.byref(sj),
                                 float(sample_rate_hz), float(wavelength),
                                 out.ctypes.data_as(C.POINTER(_capi.dg_pair_offsets))))
    return out


class StagedSnapshots:
    """A run's captures and states resident in HBM (float2 + double2 copies)."""

    def __init__(self, states: np.ndarray, captures: np.ndarray, sample_rate_hz: float,
                 center_freq_hz: float, engine: Engine | None = None):
        self.engine = engine or default_engine()
        snaps, self._keep = _snapshots_struct(states, captures, sample_rate_hz, center_freq_hz)
        h = C.c_void_p()
        check(lib.dg_stage_snapshots(self.engine.handle, C.byref(snaps), C.byref(h)))
        self._h = h
        self._keep = None  # host buffers no longer needed
        self.shape = captures.shape

    @property
    def handle(self):
        return self._h

    @classmethod
    def from_iq_files(cls, paths, states, engine: Engine | None = None) -> "StagedSnapshots":
        """load_snapshots (tools/digeo_cli.cpp:64-85) from DGIQ files: paths[s][r],
        states [S, R, 6]; payloads go disk -> pinned -> HBM as float32 I/Q."""
        self = cls.__new__(cls)
        self.engine = engine or default_engine()
        S, R = len(paths), len(paths[0])
        if any(len(row) != R for row in paths):
            raise ValueError("geolocate_snapshots: receiver count differs between snapshots")
        st = np.ascontiguousarray(states, np.float64).reshape(S * R, 6)
        st_arr = (_capi.dg_state * (S * R))(*[_pair_states(st[k]) for k in range(S * R)])
        cpaths = (C.c_char_p * (S * R))(*[str(p).encode() for row in paths for p in row])
        h = C.c_void_p()
        check(lib.dg_stage_snapshots_iq(self.engine.handle, cpaths, S, R, st_arr, C.byref(h)))
        self._h = h
        self._keep = None
        hdr = read_iq_header(paths[0][0])
        self.shape = (S, R, hdr.sample_count)
        return self

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.dg_staged_destroy(h)
            self._h = None


def read_iq_header(path) -> "_capi.dg_iq_header":
    """The DGIQ header (io.hpp:45-52), validated like read_iq (io.hpp:140-167)."""
    h = _capi.dg_iq_header()
    check(lib.dg_read_iq_header(str(path).encode(), C.byref(h)))
    return h


def read_iq(path) -> BasebandCapture:
    """read_iq (io.hpp:140-167): a DGIQ file as a BasebandCapture with complex64
    samples (the file's float32 I/Q, exact)."""
    h = _capi.dg_iq_header()
    check(lib.dg_read_iq_header(str(path).encode(), C.byref(h)))
    buf = np.empty(h.sample_count, np.complex64)
    check(lib.dg_read_iq(str(path).encode(), C.byref(h),
                         buf.ctypes.data_as(C.POINTER(C.c_float)), h.sample_count))
    return BasebandCapture(buf, h.sample_rate_hz, h.start_time_s, h.center_freq_hz)


def _snapshots_struct(states, captures, fs, fc):
    """captures: [S, R, N] complex128 (reference layout) or complex64 (DGIQ)."""
    caps = np.asarray(captures)
    if caps.ndim != 3:
        raise ValueError("captures must be [n_snapshots, n_receivers, n_samples]")
    S, R, N = caps.shape
    # dg_state is 6 packed doubles (position, velocity): view the states array
    st = np.array(states, np.float64, order="C", copy=True).reshape(S * R, 6)
    st_arr = (_capi.dg_state * (S * R)).from_buffer(st)
    keep = [st, st_arr]
    snaps = _capi.dg_snapshots()
    snaps.n_snapshots, snaps.n_receivers, snaps.n_samples = S, R, N
    snaps.sample_rate_hz, snaps.center_freq_hz = float(fs), float(fc)
    snaps.states = st_arr
    if caps.dtype == np.complex64:
        caps = np.ascontiguousarray(caps)
        fp = C.POINTER(C.c_float)
    else:
        caps = np.ascontiguousarray(caps, np.complex128)
        fp = C.POINTER(C.c_double)
    # one pointer per (snapshot, receiver) row, computed as addresses
    addr = np.asarray(caps.ctypes.data + np.arange(S * R, dtype=np.uint64) * (N * caps.itemsize),
                      dtype=np.uintp)
    ptrs = (fp * (S * R)).from_buffer(addr)
    keep.append(addr)
    if caps.dtype == np.complex64:
        snaps.captures_f32 = ptrs
    else:
        snaps.captures_iq = ptrs
    keep += [caps, ptrs]
    return snaps, keep


def _options(options: GeolocateOptions, stream=None, profile=False, peak_stage=0,
             peak_max=0.0) -> _capi.dg_options:
    o = _capi.dg_options()
    lib.dg_options_default(C.byref(o))
    o.k_sigma = float(options.k_sigma)
    o.exclusion_radius_cells = int(options.exclusion_radius_cells)
    o.normalize_per_snapshot = int(bool(options.normalize_per_snapshot))
    o.detect = int(bool(options.detect))
    o.stream = stream
    o.profile = int(bool(profile))
    o.patch_peak = int(bool(options.patch_peak))
    o.peak_stage = int(peak_stage)
    o.peak_max = float(peak_max)
    return o


def _run(grid: CandidateGrid, options: GeolocateOptions, n_snap: int, call, *, want_surface=True,
         want_per_snapshot=False, accumulated_device=None, stream=None, profile=False,
         det_cap=4096, out=None, peak_stage=0, peak_max=0.0):
    P = grid.size()
    res = _capi.dg_result()
    acc = None
    if want_surface:  # `out`: a caller-owned (e.g. pinned) float64 [P] host buffer
        if out is not None and (out.dtype != np.float64 or out.size != P or
                                not out.flags["C_CONTIGUOUS"]):
            raise ValueError("out: need a contiguous float64 array of grid.size() values")
        acc = out if out is not None else np.empty(P, np.float64)
    per = np.empty((n_snap, P), np.float64) if want_per_snapshot else None
    dets = (_capi.dg_emitter_estimate * det_cap)()
    if acc is not None:
        res.accumulated = acc.ctypes.data_as(C.POINTER(C.c_double))
    if per is not None:
        res.per_snapshot = per.ctypes.data_as(C.POINTER(C.c_double))
    if accumulated_device is not None:
        res.accumulated_device = int(accumulated_device)
    res.detections = dets
    res.detections_capacity = det_cap
    opt = _options(options, stream, profile, peak_stage, peak_max)
    check(call(C.byref(opt), C.byref(res)))
    if options.detect and res.n_detections > det_cap:
        # the engine never truncates: the whole list from the returned surface
        surf, on_dev = (acc.ctypes.data, 0) if acc is not None else (accumulated_device, 1)
        if surf is None:
            raise RuntimeError(f"{res.n_detections} detections exceed the {det_cap}-entry buffer "
                               "and no surface was returned to re-run detect_emitters on")
        det_cap = int(res.n_detections)
        dets = (_capi.dg_emitter_estimate * det_cap)()
        n = C.c_int64()
        check(lib.dg_detect_emitters(grid.engine.handle, grid.handle, C.c_void_p(int(surf)), on_dev,
                                     float(options.k_sigma), int(options.exclusion_radius_cells),
                                     dets, det_cap, C.byref(n)))
        res.n_detections = n.value
    detections = [EmitterEstimate(GeodeticCoord(d.lat_deg, d.lon_deg, d.alt_m), int(d.grid_index),
                                  d.score, d.score_zsigma)
                  for d in dets[:min(res.n_detections, det_cap)]]
    stats = dict(n_refined=res.n_refined, n_reranked=res.n_reranked,
                 sum_overlap_samples=res.sum_overlap_samples, correlate_ms=res.correlate_ms,
                 correlate_launches=res.correlate_launches, total_ms=res.total_ms,
                 kernel_launches=res.kernel_launches, n_detections=res.n_detections,
                 moments_ms=res.moments_ms, evaluate_ms=res.evaluate_ms,
                 moment_ffma2=res.moment_ffma2, evaluate_ffma2=res.evaluate_ffma2,
                 direct_steps=res.direct_steps, evaluate_tc_flop=res.evaluate_tc_flop,
                 moment_fft_flop=res.moment_fft_flop)
    per_list = [CorrelationGrid(grid, per[s]) for s in range(n_snap)] if per is not None else []
    return GeolocateResult(grid, per_list, CorrelationGrid(grid, acc), detections,
                           int(res.argmax_index), float(res.argmax_value), stats)


def detect_emitters(grid: CorrelationGrid, k_sigma: float = 5.0,
                    exclusion_radius_cells: int = 5, values_device: int | None = None) -> list:
    """detect_emitters (correlate.hpp:127-201) on the GPU: every detection, in the
    reference's order. `grid.values` (host float64) or, if given, a device
    pointer to the surface (values_device) over grid.grid."""
    g = grid.grid
    if values_device is None:
        v = np.ascontiguousarray(grid.values, np.float64)
        if v.size != g.size():
            raise ValueError("CorrelationGrid: value count != grid size")
        surf, on_dev = v.ctypes.data, 0
    else:
        surf, on_dev = int(values_device), 1
    cap = 256
    while True:
        out = (_capi.dg_emitter_estimate * cap)()
        n = C.c_int64()
        check(lib.dg_detect_emitters(g.engine.handle, g.handle, C.c_void_p(surf), on_dev,
                                     float(k_sigma), int(exclusion_radius_cells), out, cap,
                                     C.byref(n)))
        if n.value <= cap:
            return [EmitterEstimate(GeodeticCoord(d.lat_deg, d.lon_deg, d.alt_m),
                                    int(d.grid_index), d.score, d.score_zsigma)
                    for d in out[:n.value]]
        cap = int(n.value)


def geolocate_arrays(grid: CandidateGrid, states: np.ndarray, captures: np.ndarray,
                     sample_rate_hz: float, center_freq_hz: float,
                     options: GeolocateOptions | None = None, **kw) -> GeolocateResult:
    """Host arrays in ([S,R,6] states, [S,R,N] captures), host results out."""
    options = options or GeolocateOptions()
    snaps, keep = _snapshots_struct(states, captures, sample_rate_hz, center_freq_hz)
    kw.setdefault("want_per_snapshot", options.keep_per_snapshot)
    return _run(grid, options, captures.shape[0],
                lambda o, r: lib.dg_geolocate_snapshots(grid.engine.handle, grid.handle,
                                                        C.byref(snaps), o, r), **kw)


def geolocate_staged(grid: CandidateGrid, staged: StagedSnapshots,
                     options: GeolocateOptions | None = None, **kw) -> GeolocateResult:
    """Inputs already resident in HBM (the bench's device-only `value`)."""
    options = options or GeolocateOptions()
    kw.setdefault("want_per_snapshot", False)
    return _run(grid, options, staged.shape[0],
                lambda o, r: lib.dg_geolocate_staged(grid.engine.handle, grid.handle,
                                                     staged.handle, o, r), **kw)


def correlate_steps(grid: CandidateGrid, staged: StagedSnapshots, s_begin: int, s_end: int,
                    grids_device: int, medians_device: int | None = None,
                    options: GeolocateOptions | None = None, stream=None,
                    profile: bool = False) -> dict:
    """Per-snapshot surfaces of snapshots [s_begin, s_end) over the whole grid
    into a device buffer [(s_end - s_begin)][P] (float64, e.g. a torch tensor's
    data_ptr()): correlate_snapshot_all_pairs (+ normalize_by_median) of
    geolocate.hpp:79-122 — the snapshot-sharded half of geolocate_snapshots."""
    options = options or GeolocateOptions()
    res = _capi.dg_result()
    opt = _options(options, stream, profile)
    check(lib.dg_correlate_steps(grid.engine.handle, grid.handle, staged.handle, int(s_begin),
                                 int(s_end), C.byref(opt), C.c_void_p(int(grids_device)),
                                 C.c_void_p(int(medians_device)) if medians_device else None,
                                 C.byref(res)))
    return dict(n_refined=res.n_refined, sum_overlap_samples=res.sum_overlap_samples,
                correlate_ms=res.correlate_ms, moments_ms=res.moments_ms,
                evaluate_ms=res.evaluate_ms, moment_ffma2=res.moment_ffma2,
                evaluate_ffma2=res.evaluate_ffma2, direct_steps=res.direct_steps,
                evaluate_tc_flop=res.evaluate_tc_flop, moment_fft_flop=res.moment_fft_flop,
                kernel_launches=res.kernel_launches, correlate_launches=res.correlate_launches)


def correlate_units(grid: CandidateGrid, staged: StagedSnapshots, units, raw_device: int,
                    options: GeolocateOptions | None = None, stream=None,
                    profile: bool = False) -> dict:
    """Raw surfaces [len(units)][P] (device pointer) of work units (step, part,
    parts) — dg_correlate_units, the unit-sharded half of geolocate_snapshots."""
    options = options or GeolocateOptions()
    res = _capi.dg_result()
    opt = _options(options, stream, profile)
    arr = (_capi.dg_work_unit * max(len(units), 1))(
        *[_capi.dg_work_unit(int(s), int(p), int(n), 0, 0) for s, p, n in units])
    check(lib.dg_correlate_units(grid.engine.handle, grid.handle, staged.handle, arr, len(units),
                                 C.byref(opt), C.c_void_p(int(raw_device)), C.byref(res)))
    return dict(n_refined=res.n_refined, sum_overlap_samples=res.sum_overlap_samples,
                correlate_ms=res.correlate_ms, moments_ms=res.moments_ms,
                evaluate_ms=res.evaluate_ms, moment_ffma2=res.moment_ffma2,
                evaluate_ffma2=res.evaluate_ffma2, direct_steps=res.direct_steps,
                evaluate_tc_flop=res.evaluate_tc_flop, moment_fft_flop=res.moment_fft_flop,
                kernel_launches=res.kernel_launches, correlate_launches=res.correlate_launches)


def accumulate_peak(grid: CandidateGrid, staged: StagedSnapshots, grids_device: int,
                    medians_device: int | None = None, options: GeolocateOptions | None = None,
                    **kw) -> GeolocateResult:
    """accumulate_grids + exact argmax (+ detect_emitters) of per-snapshot
    surfaces [S][P_grid] already on the device, for a grid or a slab of one."""
    options = options or GeolocateOptions()
    kw.setdefault("want_per_snapshot", False)
    med = C.c_void_p(int(medians_device)) if medians_device else None
    return _run(grid, options, staged.shape[0],
                lambda o, r: lib.dg_accumulate_peak(grid.engine.handle, grid.handle,
                                                    staged.handle, C.c_void_p(int(grids_device)),
                                                    med, o, r), **kw)


def geolocate_snapshots(snapshots: list, grid: CandidateGrid,
                        options: GeolocateOptions | None = None) -> GeolocateResult:
    """geolocate.hpp:127-146 — same inputs/outputs as the reference driver."""
    options = options or GeolocateOptions()
    if not snapshots:
        raise ValueError("geolocate_snapshots: no snapshots")
    if options.backend_name != "b200":
        raise ValueError(f"make_backend: unknown backend '{options.backend_name}' "
                         "(expected b200)")
    R = len(snapshots[0].captures)
    if R < 2:
        raise ValueError("correlate_snapshot_all_pairs: need >= 2 receivers")
    c0 = snapshots[0].captures[0]
    for snap in snapshots:
        if len(snap.captures) != R:
            raise ValueError("geolocate_snapshots: receiver count differs between snapshots")
        for c in snap.captures:
            c.validate()
            if c.sample_rate_hz != c0.sample_rate_hz:
                raise ValueError("backend stage: sample rates differ")
            if len(c.samples) != len(c0.samples):
                raise ValueError("backend stage: sample counts differ")
            # the reference takes each pair's wavelength from its first capture
            # (geolocate.hpp:55); the engine runs one carrier per run
            if c.center_freq_hz != c0.center_freq_hz:
                raise ValueError("geolocate_snapshots: center frequencies differ")
    f32 = all(np.asarray(c.samples).dtype == np.complex64 for s in snapshots for c in s.captures)
    caps = np.stack([np.stack([np.asarray(c.samples) for c in s.captures]) for s in snapshots])
    caps = caps.astype(np.complex64 if f32 else np.complex128, copy=False)
    states = np.stack([np.asarray(s.states, np.float64).reshape(R, 6) for s in snapshots])
    plan_batches(grid.size(), options.batch_size, options.memory_budget_bytes,
                 2 * len(c0.samples) * 16)
    return geolocate_arrays(grid, states, caps, c0.sample_rate_hz, c0.center_freq_hz, options)
