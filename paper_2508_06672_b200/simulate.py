"""Scenario synthesis on the GPU (reference scene.hpp:200-310).

Mirrors the reference's scenario types and ``simulate_scenario``:

* ``EmitterDef`` (scene.hpp:46-60) with a waveform spec — ``SpooferSpec``,
  ``ToneSpec``, ``ChirpSpec``, ``SawtoothSpec`` (waveform.hpp:58-97);
* receivers as ``CircularOrbit`` (orbit.hpp:30-35) or an explicit [S, 6] state
  table;
* ``Scenario`` (scene.hpp:72-114).

``simulate_scenario(scenario)`` returns the reference's ``list[Snapshot]``
(complex128 captures on the host); ``simulate_staged(scenario)`` leaves the
captures in HBM as a ``StagedSnapshots`` run that ``geolocate_staged`` solves
without any host round trip. Waveforms, the FFT fractional delay, the Doppler
channel and the MT19937-64 / Box-Muller noise all run on the device.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import check, lib
from .backend import BasebandCapture
from .engine import Engine, default_engine
from .geodesy import GeodeticCoord
from .geolocate import Snapshot, StagedSnapshots


@dataclass
class SpooferSpec:
    prn: int = 1
    data_seed: int = 0


@dataclass
class ToneSpec:
    offset_hz: float = 0.0


@dataclass
class ChirpSpec:
    bandwidth_hz: float = 0.0
    period_s: float = 0.0


@dataclass
class SawtoothSpec:
    bandwidth_hz: float = 0.0
    chirp_period_s: float = 0.0


@dataclass
class EmitterDef:
    location: GeodeticCoord
    waveform: object
    ref_snr_db: float = 0.0
    ref_range_m: float = 1.0


@dataclass
class CircularOrbit:
    alt_m: float = 550e3
    inclination_deg: float = 53.0
    raan_deg: float = 0.0
    phase_deg: float = 0.0


@dataclass
class Scenario:
    receivers: list = field(default_factory=list)   # CircularOrbit | ndarray [S, 6]
    emitters: list = field(default_factory=list)
    snapshot_count: int = 1
    snapshot_spacing_s: float = 1.0
    capture_duration_s: float = 0.05
    sample_rate_hz: float = 5e6
    center_freq_hz: float = 1575.42e6
    start_time_s: float = 0.0
    noise_seed: int = 0
    noise_power: float = 1.0


def _emitter(e: EmitterDef) -> _capi.dg_emitter_def:
    d = _capi.dg_emitter_def()
    d.lat_deg, d.lon_deg, d.alt_m = e.location.lat_deg, e.location.lon_deg, e.location.alt_m
    d.ref_snr_db, d.ref_range_m = e.ref_snr_db, e.ref_range_m
    w = e.waveform
    if isinstance(w, SpooferSpec):
        d.waveform, d.prn, d.data_seed = 0, int(w.prn), int(w.data_seed)
    elif isinstance(w, ToneSpec):
        d.waveform, d.tone_offset_hz = 1, float(w.offset_hz)
    elif isinstance(w, ChirpSpec):
        d.waveform, d.bandwidth_hz, d.period_s = 2, float(w.bandwidth_hz), float(w.period_s)
    elif isinstance(w, SawtoothSpec):
        d.waveform, d.bandwidth_hz, d.period_s = 3, float(w.bandwidth_hz), float(w.chirp_period_s)
    else:
        raise ValueError(f"unknown waveform spec {w!r}")
    return d


def _scenario(sc: Scenario):
    keep = []
    rx = (_capi.dg_receiver_def * max(len(sc.receivers), 1))()
    for i, r in enumerate(sc.receivers):
        if isinstance(r, CircularOrbit):
            rx[i] = _capi.dg_receiver_def(r.alt_m, r.inclination_deg, r.raan_deg, r.phase_deg, None)
        else:
            st = np.ascontiguousarray(r, np.float64).reshape(-1, 6)
            if len(st) != sc.snapshot_count:
                raise ValueError("Scenario: state table length != snapshot_count")
            keep.append(st)
            rx[i] = _capi.dg_receiver_def(0, 0, 0, 0, st.ctypes.data_as(C.POINTER(_capi.dg_state)))
    em = (_capi.dg_emitter_def * max(len(sc.emitters), 1))(*[_emitter(e) for e in sc.emitters])
    d = _capi.dg_scenario(rx, len(sc.receivers), em, len(sc.emitters), int(sc.snapshot_count),
                          float(sc.snapshot_spacing_s), float(sc.capture_duration_s),
                          float(sc.sample_rate_hz), float(sc.center_freq_hz),
                          float(sc.start_time_s), int(sc.noise_seed) & (2 ** 64 - 1),
                          float(sc.noise_power))
    return d, (rx, em, keep)


def samples_per_capture(sc: Scenario) -> int:
    d, _keep = _scenario(sc)
    n = C.c_int64()
    check(lib.dg_scenario_samples(C.byref(d), C.byref(n)))
    return n.value


def simulate_arrays(sc: Scenario, engine: Engine | None = None, staged: bool = False):
    """-> (states [S, R, 6], captures [S, R, N] complex128, epochs [S], staged or None)."""
    eng = engine or default_engine()
    d, _keep = _scenario(sc)
    S, R = int(sc.snapshot_count), len(sc.receivers)
    N = samples_per_capture(sc)
    caps = np.empty((S, R, max(N, 0)), np.complex128)
    states = np.empty((S, R, 6), np.float64)
    epochs = np.empty(S, np.float64)
    h = C.c_void_p()
    check(lib.dg_simulate_scenario(eng.handle, C.byref(d), C.byref(h) if staged else None,
                                   caps.ctypes.data_as(C.POINTER(C.c_double)),
                                   states.ctypes.data_as(C.POINTER(_capi.dg_state)),
                                   epochs.ctypes.data_as(C.POINTER(C.c_double))))
    st = None
    if staged:
        st = StagedSnapshots.__new__(StagedSnapshots)
        st.engine, st._h, st._keep, st.shape = eng, h, None, (S, R, N)
    return states, caps, epochs, st


def simulate_scenario(sc: Scenario, engine: Engine | None = None) -> list:
    """scene.hpp:253-310: one Snapshot per epoch, captures synthesised on the GPU."""
    states, caps, epochs, _ = simulate_arrays(sc, engine)
    out = []
    for s in range(caps.shape[0]):
        out.append(Snapshot(float(epochs[s]), states[s],
                            [BasebandCapture(caps[s, r], sc.sample_rate_hz, float(epochs[s]),
                                             sc.center_freq_hz) for r in range(caps.shape[1])]))
    return out


def simulate_staged(sc: Scenario, engine: Engine | None = None) -> StagedSnapshots:
    """The run's captures synthesised straight into HBM (no host copy of the samples)."""
    eng = engine or default_engine()
    d, _keep = _scenario(sc)
    h = C.c_void_p()
    check(lib.dg_simulate_scenario(eng.handle, C.byref(d), C.byref(h), None, None, None))
    st = StagedSnapshots.__new__(StagedSnapshots)
    st.engine, st._h, st._keep = eng, h, None
    st.shape = (int(sc.snapshot_count), len(sc.receivers), samples_per_capture(sc))
    return st
