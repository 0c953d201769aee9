"""Synthetic scene generator for bench inputs (off the hot path).

Produces receiver states and complex-baseband captures of the shape the
reference simulator emits (scene.hpp:253-310) for BASELINE.json's workloads.
It is NOT the reference simulator: waveforms are evaluated analytically at
the delayed time (no FFT fractional-delay filter) and the spoofer is a seeded
BPSK chip stream rather than a Gold code. The bench measures throughput on
these inputs; parity tests use the reference's own simulator (oracle/_ref).
"""
from __future__ import annotations

import numpy as np

C = 299792458.0
A = 6378137.0
F = 1.0 / 298.257223563
E2 = F * (2.0 - F)
MU = 3.986004418e14
KM_DEG = 0.0089932161


def lla_to_ecef(lat_deg, lon_deg, alt_m):
    lat, lon = np.deg2rad(lat_deg), np.deg2rad(lon_deg)
    slat, clat = np.sin(lat), np.cos(lat)
    n = A / np.sqrt(1.0 - E2 * slat * slat)
    return np.stack([(n + alt_m) * clat * np.cos(lon), (n + alt_m) * clat * np.sin(lon),
                     (n * (1.0 - E2) + alt_m) * slat], axis=-1)


def circular_orbit(alt_m, inc_deg, raan_deg, phase_deg, epochs):
    """Two-body circular orbit treated as ECEF (the reference's orbit.hpp model)."""
    r = A + alt_m
    nmot = np.sqrt(MU / r ** 3)
    v = r * nmot
    inc, raan = np.deg2rad(inc_deg), np.deg2rad(raan_deg)
    u = np.deg2rad(phase_deg) + nmot * np.asarray(epochs, np.float64)
    ci, si, co, so = np.cos(inc), np.sin(inc), np.cos(raan), np.sin(raan)

    def rot(px, py):
        x1, y1, z1 = px, ci * py, si * py
        return np.stack([co * x1 - so * y1, so * x1 + co * y1, z1], axis=-1)

    return np.concatenate([rot(r * np.cos(u), r * np.sin(u)),
                           rot(-v * np.sin(u), v * np.cos(u))], axis=-1)


def _waveform(kind: str, t: np.ndarray, p: dict, rng_seed: int) -> np.ndarray:
    if kind == "tone":
        return np.exp(2j * np.pi * p.get("offset", 0.0) * t)
    if kind == "chirp":
        bw, per = p.get("bw", 2e6), p.get("period", 20e-6)
        u = np.mod(t, per)
        return np.exp(2j * np.pi * (bw / (2 * per) * u * u - 0.5 * bw * u))
    if kind == "sawtooth":
        bw, per = p.get("bw", 200e3), p.get("period", 2.5e-3)
        v = np.mod(t, 2 * per)
        u = np.mod(t, per)
        ph = 2 * np.pi * (bw / (2 * per) * u * u - 0.5 * bw * u)
        return np.exp(1j * np.where(v < per, ph, -ph))
    if kind == "spoofer":
        chips = np.floor(t * 1.023e6 + 1e-6).astype(np.int64)
        h = (chips.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)) ^ np.uint64(rng_seed)
        h ^= h >> np.uint64(31)
        return np.where((h & np.uint64(1)) == 0, 1.0, -1.0).astype(np.complex128)
    raise ValueError(kind)


PAPER_RECEIVERS = [(550e3, 53.0, -1.2, -1.1), (550e3, 53.0, 1.2, -0.7)]
FOUR_EMITTERS = [("spoofer", 0.5, -1.5, {}), ("tone", 0.5, 1.5, {}), ("chirp", -0.5, -1.5, {}),
                 ("sawtooth", -0.5, 1.5, {})]


def synthesize(n_snapshots: int, n_samples: int, fs: float, emitters, snr_db: float,
               receivers=PAPER_RECEIVERS, fc: float = 1575.42e6, spacing_s: float = 1.0,
               seed: int = 3, noise_power: float = 1.0, dtype=np.complex128):
    """Return (states [S,R,6], captures [S,R,N]) for point emitters at lattice nodes."""
    rng = np.random.default_rng(seed)
    S, R, N = n_snapshots, len(receivers), n_samples
    epochs = np.arange(S) * spacing_s
    states = np.stack([circular_orbit(*rx, epochs) for rx in receivers], axis=1)  # [S,R,6]
    wl = C / fc
    t = np.arange(N) / fs
    caps = np.zeros((S, R, N), np.complex128)
    amp0 = 10 ** (snr_db / 20.0)
    for ei, (kind, lat, lon, p) in enumerate(emitters):
        pos = lla_to_ecef(lat, lon, 0.0)
        for s in range(S):
            for r in range(R):
                rv = states[s, r, :3] - pos
                rho = np.linalg.norm(rv)
                dop = -np.dot(rv / rho, states[s, r, 3:]) / wl
                tau = rho / C
                x = _waveform(kind, epochs[s] + t - tau, p, seed * 1000 + ei)
                caps[s, r] += amp0 * 650e3 / rho * x * np.exp(2j * np.pi * dop * t)
    if noise_power > 0:
        sig = np.sqrt(noise_power / 2)
        caps += sig * (rng.standard_normal((S, R, N)) + 1j * rng.standard_normal((S, R, N)))
    return states, caps.astype(dtype, copy=False)


def grid_bounds_km(half_km: float):
    h = half_km * KM_DEG
    return (-h, h, -h, h)
