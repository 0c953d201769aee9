"""Capture synthesis on the GPU against the reference's
simulate_scenario (oracle/_ref, scene.hpp:253-310).

Scenario arithmetic (epochs, orbit states) is bit-identical; samples agree to
FP64 rounding: the device's cos/sin/log and FFT rounding differ from glibc's and
the reference's radix-2 FFT by ulps, everything else (MT19937-64 stream, C/A
chips, nav bits, Doppler phasor recurrence, delays, amplitudes) is exact. The
tolerance is 1e-12 absolute (measured: 1e-15 at C3) on unit-variance noise + emitter amplitudes <= ~2.
"""
import numpy as np
import pytest

import scenes
from oracle.bindings import ReferenceError_

TOL = 1e-12


@pytest.fixture(scope="module")
def sim():
    import paper_2508_06672_b200.simulate as sim
    return sim


def _compare(sim, ref, scene, tol=TOL):
    want = ref.simulate(scenes.render(scene))
    states, caps, epochs, _ = sim.simulate_arrays(scenes.to_scenario(sim, scene))
    assert caps.shape == want.captures.shape
    assert np.array_equal(states, want.states)  # orbit propagation, bit for bit
    err = np.abs(caps - want.captures).max()
    assert err <= tol, err
    return caps, want


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["DESK_FOURJAM", "DESK_SAWTOOTH", "TRIPLE_RX"])
def test_desk_scenes_match_reference(sim, ref, name):
    """All four waveforms (spoofer / tone / chirp / sawtooth), 2 and 3 receivers."""
    _compare(sim, ref, getattr(scenes, name))


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_baseline_configs_match_reference(sim, ref, cfg):
    """C1: one 250k-sample tone snapshot; C2: ten chirp snapshots."""
    _compare(sim, ref, scenes.config(cfg))


@pytest.mark.gpu
def test_noise_only_and_noise_free(sim, ref):
    base = dict(scenes.DESK_SAWTOOTH)
    _compare(sim, ref, {**base, "emitters": []}, tol=1e-12)       # MT19937-64 + Box-Muller
    caps, want = _compare(sim, ref, {**base, "noise_power": 0})   # channel only
    assert np.abs(caps).max() > 0


@pytest.mark.gpu
def test_simulated_run_solves_like_reference_captures(sim, ref, b2):
    """simulate_staged -> geolocate_staged (no host round trip) finds the same
    peak and detections as solving the reference's own captures."""
    scene = scenes.DESK_FOURJAM
    want = ref.simulate(scenes.render(scene))
    grid = b2.build_candidate_grid(b2.LatLonBounds(*want.bounds), want.spacing)
    opts = b2.GeolocateOptions(k_sigma=want.k_sigma, exclusion_radius_cells=want.radius)
    a = b2.geolocate_arrays(grid, want.states, want.captures, want.fs, want.fc, opts)
    staged = sim.simulate_staged(scenes.to_scenario(sim, scene))
    b = b2.geolocate_staged(grid, staged, opts)
    assert a.argmax_index == b.argmax_index
    assert [d.grid_index for d in a.detections] == [d.grid_index for d in b.detections]
    rel = np.abs(a.accumulated.values - b.accumulated.values) / a.accumulated.values.max()
    assert rel.max() < 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("edit", [
    {"capture_duration_s": 0.06},
    {"noise_power": -1},
    {"receivers": [scenes._orbit(150e3, 53, 0, 0), scenes._orbit(550e3, 53, 1, 0)]},
    {"emitters": [scenes._tone(95.0, 0.0, -5)]},
    {"emitters": [scenes._tone(0.0, 0.0, -5, off=2e6)]},
    {"emitters": [scenes._chirp(0.0, 0.0, -5, bw=3e6)]},
])
def test_errors_match_reference(sim, ref, edit):
    scene = {**scenes.DESK_SAWTOOTH, **edit}
    with pytest.raises(ReferenceError_) as want:
        ref.simulate(scenes.render(scene))
    with pytest.raises(ValueError) as got:
        sim.simulate_arrays(scenes.to_scenario(sim, scene))
    assert str(got.value) == str(want.value)
