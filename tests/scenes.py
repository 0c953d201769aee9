"""Scenario parameter sets for parity tests and the bench, rendered into the
reference's `key = value` scenario format (config.hpp:269-324) so the
reference simulator (oracle/_ref) can synthesise identical captures.

DESK_FOURJAM / DESK_SAWTOOTH restate the parameters of the reference's
desk-scale scenes (proj/configs/desk_fourjam.cfg, desk_sawtooth.cfg), whose
known answers are in tests/golden/. C1..C5 are BASELINE.json's workloads
(SURVEY.md §8d).
"""
from __future__ import annotations

KM_DEG = 0.0089932161  # 1 km of arc on a 6371 km sphere, in degrees


def render(scene: dict) -> str:
    lines = []
    for k, v in scene.items():
        if k in ("receivers", "emitters"):
            continue
        lines.append(f"{k} = {v}")
    for rx in scene.get("receivers", []):
        lines.append("[receiver]")
        lines += [f"{k} = {v}" for k, v in rx.items()]
    for em in scene.get("emitters", []):
        lines.append("[emitter]")
        lines += [f"{k} = {v}" for k, v in em.items()]
    return "\n".join(lines) + "\n"


def _orbit(alt, inc, raan, phase):
    return dict(orbit_alt_m=alt, orbit_inclination_deg=inc, orbit_raan_deg=raan,
                orbit_phase_deg=phase)


def _spoofer(lat, lon, snr, prn=7, seed=7):
    return dict(lat_deg=lat, lon_deg=lon, waveform="spoofer", prn=prn, data_seed=seed,
                ref_snr_db=snr, ref_range_m=650e3)


def _tone(lat, lon, snr, off=0):
    return dict(lat_deg=lat, lon_deg=lon, waveform="tone", tone_offset_hz=off, ref_snr_db=snr,
                ref_range_m=650e3)


def _chirp(lat, lon, snr, bw=2e6, per=20e-6):
    return dict(lat_deg=lat, lon_deg=lon, waveform="chirp", chirp_bandwidth_hz=bw,
                chirp_period_s=per, ref_snr_db=snr, ref_range_m=650e3)


def _saw(lat, lon, snr, bw=200e3, per=2.5e-3):
    return dict(lat_deg=lat, lon_deg=lon, waveform="sawtooth", sawtooth_bandwidth_hz=bw,
                sawtooth_chirp_period_s=per, ref_snr_db=snr, ref_range_m=650e3)


def _grid(lat0, lat1, lon0, lon1, spacing):
    return dict(grid_lat_min_deg=lat0, grid_lat_max_deg=lat1, grid_lon_min_deg=lon0,
                grid_lon_max_deg=lon1, grid_spacing_deg=spacing, grid_alt_m=0)


def _base(snapshots, spacing_s, dur, fs, seed, **extra):
    d = dict(snapshots=snapshots, snapshot_spacing_s=spacing_s, capture_duration_s=dur,
             sample_rate_hz=fs, center_freq_hz=1575.42e6, noise_seed=seed)
    d.update(extra)
    return d


DESK_FOURJAM = {
    **_base(10, 1.0, 5e-3, 2.048e6, 2026),
    **_grid(-0.8, 0.8, -0.8, 0.8, 0.02),
    "backend": "serial", "batch_size": 8, "k_sigma": 5, "exclusion_radius_cells": 30,
    "receivers": [_orbit(550e3, 90, 0.4, -0.65), _orbit(550e3, 90, 179.2, 179.2)],
    "emitters": [_spoofer(-0.4, -0.4, -5), _tone(-0.4, 0.4, -5), _chirp(0.4, -0.4, -5),
                 _saw(0.4, 0.4, -5)],
}

DESK_SAWTOOTH = {
    **_base(10, 20.0, 5e-3, 2.048e6, 404),
    **_grid(-0.6, 0.6, -0.6, 0.6, 0.02),
    "backend": "serial", "batch_size": 8, "k_sigma": 5, "exclusion_radius_cells": 5,
    "receivers": [_orbit(550e3, 53, -1.0, -0.65), _orbit(550e3, 53, 1.0, -0.05)],
    "emitters": [_saw(0.0, 0.0, -3)],
}

# three receivers: exercises the all-pairs sum (geolocate.hpp:79-94)
TRIPLE_RX = {
    **_base(3, 5.0, 2e-3, 2.048e6, 99),
    **_grid(-0.3, 0.3, -0.3, 0.3, 0.02),
    "backend": "serial", "batch_size": 8, "k_sigma": 5, "exclusion_radius_cells": 5,
    "receivers": [_orbit(550e3, 53, -0.9, -0.7), _orbit(550e3, 53, 0.9, 0.5),
                  _orbit(600e3, 80, 0.2, -1.5)],
    "emitters": [_chirp(0.1, -0.12, -3, 1e6, 50e-6)],
}

# four receivers: six pairs per snapshot (the all-pairs sum and the shared
# per-receiver geometry pass, geolocate.hpp:79-94)
QUAD_RX = {
    **_base(3, 5.0, 4e-3, 2.048e6, 123),
    **_grid(-0.4, 0.4, -0.4, 0.4, 0.02),
    "backend": "serial", "batch_size": 8, "k_sigma": 5, "exclusion_radius_cells": 5,
    "receivers": [_orbit(550e3, 53, -0.9, -0.7), _orbit(550e3, 53, 0.9, 0.5),
                  _orbit(600e3, 80, 0.2, -1.5), _orbit(520e3, 97, -0.4, 0.9)],
    "emitters": [_chirp(0.1, -0.12, -6, 1e6, 50e-6), _tone(-0.2, 0.2, -8, 1500)],
}

# BASELINE.json configs; receivers as paper_scenario.cfg
_PAPER_RX = [_orbit(550e3, 53, -1.2, -1.1), _orbit(550e3, 53, 1.2, -0.7)]
_FOUR = [_spoofer(0.5, -1.5, -20), _tone(0.5, 1.5, -20), _chirp(-0.5, -1.5, -20),
         _saw(-0.5, 1.5, -20)]


def config(name: str, spacing_km: float = 1.0) -> dict:
    sp = KM_DEG * spacing_km
    if name == "C1":
        half = 50 * KM_DEG
        return {**_base(1, 1.0, 0.05, 5e6, 1, noise_power=1.0), **_grid(-half, half, -half, half, sp),
                "receivers": _PAPER_RX, "emitters": [_tone(0.0, 0.0, -5)]}
    if name == "C2":
        half = 250 * KM_DEG
        return {**_base(10, 1.0, 0.01, 5e6, 2), **_grid(-half, half, -half, half, sp),
                "receivers": _PAPER_RX, "emitters": [_chirp(0.0, 0.0, -10)]}
    if name == "C4":  # coarse global lattice at 10 km (the fine 100 m grids are built
        # around the coarse detections by the test)
        return {**_base(10, 1.0, 0.01, 5e6, 4), **_grid(-90.0, 90.0, -180.0, 179.9, 10 * sp),
                "receivers": _PAPER_RX,
                "emitters": [{**e, "ref_snr_db": -15} for e in _FOUR]}
    if name in ("C3", "C5"):
        half = (1000 if name == "C3" else 2000) * KM_DEG
        steps = 50 if name == "C3" else 100
        return {**_base(steps, 1.0, 0.01, 5e6, 3 if name == "C3" else 5),
                **_grid(-half, half, -half, half, sp), "receivers": _PAPER_RX, "emitters": _FOUR}
    raise KeyError(name)


def to_scenario(sim, scene: dict):
    """The same scene as a paper_2508_06672_b200.simulate.Scenario (the
    reference's Scenario fields, config.hpp:269-324 defaults)."""
    rx = [sim.CircularOrbit(r["orbit_alt_m"], r["orbit_inclination_deg"],
                            r.get("orbit_raan_deg", 0.0), r.get("orbit_phase_deg", 0.0))
          for r in scene["receivers"]]
    em = []
    for e in scene["emitters"]:
        kind = e["waveform"]
        if kind == "spoofer":
            w = sim.SpooferSpec(int(e["prn"]), int(e.get("data_seed", 0)))
        elif kind == "tone":
            w = sim.ToneSpec(float(e.get("tone_offset_hz", 0.0)))
        elif kind == "chirp":
            w = sim.ChirpSpec(float(e["chirp_bandwidth_hz"]), float(e["chirp_period_s"]))
        else:
            w = sim.SawtoothSpec(float(e["sawtooth_bandwidth_hz"]),
                                 float(e["sawtooth_chirp_period_s"]))
        from paper_2508_06672_b200.geodesy import GeodeticCoord
        em.append(sim.EmitterDef(GeodeticCoord(float(e["lat_deg"]), float(e["lon_deg"]),
                                               float(e.get("alt_m", 0.0))), w,
                                 float(e["ref_snr_db"]), float(e["ref_range_m"])))
    return sim.Scenario(rx, em, int(scene["snapshots"]), float(scene["snapshot_spacing_s"]),
                        float(scene["capture_duration_s"]), float(scene["sample_rate_hz"]),
                        float(scene["center_freq_hz"]), float(scene.get("start_time_s", 0.0)),
                        int(scene["noise_seed"]), float(scene.get("noise_power", 1.0)))
