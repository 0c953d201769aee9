"""CPU: the oracle restatement (oracle/digeo_oracle.c) pinned against the
reference itself (oracle/_ref) and the committed golden vectors.

Mirrors the reference's own tests: test_correlate.cpp, test_geometry.cpp,
test_geodesy.cpp, test_geolocate.cpp (paths under /root/reference/proj/tests).
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle.bindings import PAIR_OFFSETS_DTYPE

KAT = json.load(open(os.path.join(GOLDEN, "kat.json")))


def test_known_answers(orc):
    ones = np.ones(1000, np.complex128)
    assert orc.correlate(ones, ones, 0, 0.0, 1e6) == KAT["all_ones_n1000"] == 1000.0
    ones100 = np.ones(100, np.complex128)
    for d, want in KAT["truncation_n100"].items():
        assert orc.correlate(ones100, ones100, int(d), 0.0, 1e6) == want
    assert KAT["truncation_n100"]["40"] == pytest.approx(60.0)
    assert KAT["truncation_n100"]["-30"] == pytest.approx(70.0)
    assert orc.wavelength(1575.42e6) == float.fromhex(KAT["wavelength_l1"])
    assert orc.wavelength(1575.42e6) == pytest.approx(0.190293672798365, rel=1e-12)
    e = orc.lla_to_ecef(0.0, 0.0, 0.0)
    assert [float.fromhex(h) for h in KAT["ecef_equator"]] == list(e)
    pole = orc.lla_to_ecef(90.0, 0.0, 0.0)
    assert [float.fromhex(h) for h in KAT["ecef_pole"]] == list(pole)
    assert pole[2] == pytest.approx(6356752.314, abs=1e-3)
    near, far = orc.lla_to_ecef(0.0, 0.0, 500e3), orc.lla_to_ecef(0.0, 0.0, 800e3)
    z = np.zeros(3)
    d, f = orc.predict_pair_offsets(e, np.r_[near, z], np.r_[far, z], 5e6, 0.19)
    assert d == KAT["tdoa_300km_5mhz"] == 5003


def test_grid_counts(orc):
    for key, bounds, sp in (("10x10_at_0.01", (0.0, 10.0, 0.0, 10.0), 0.01),
                            ("zero_span", (5.0, 5.0, 7.0, 7.0), 0.5),
                            ("1x2_at_0.5", (0.0, 1.0, 0.0, 2.0), 0.5)):
        assert [orc.lib.orc_axis_count(bounds[1] - bounds[0], sp),
                orc.lib.orc_axis_count(bounds[3] - bounds[2], sp)] == KAT["grid_counts"][key]


def test_correlate_matches_reference_bit_exact(orc, ref):
    rng = np.random.default_rng(4242)
    for trial in range(60):
        n = int(rng.integers(1000, 4000))
        y1 = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        y2 = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        d = int(rng.integers(-n - 5, n + 5))
        f = float(rng.uniform(-1.25e6, 1.25e6))
        assert orc.correlate(y1, y2, d, f, 5e6) == ref.correlate_point(y1, y2, 5e6, d, f)


def test_correlate_golden(orc):
    g = np.load(os.path.join(GOLDEN, "correlate_small.npz"))
    got = np.array([orc.correlate(g["y1"], g["y2"], o["tdoa_samples"], o["fdoa_hz"], float(g["fs"]))
                    for o in g["offsets"]])
    assert np.array_equal(got, g["want"])


def test_offsets_golden_bit_exact(orc):
    g = np.load(os.path.join(GOLDEN, "offsets_small.npz"))
    nl, nn, pts = orc.build_grid(tuple(g["bounds"]), float(g["spacing"]))
    assert np.array_equal(pts, g["points"])
    for s in range(g["states"].shape[0]):
        got = np.zeros(len(pts), PAIR_OFFSETS_DTYPE)
        for i, p in enumerate(pts):
            got[i] = orc.predict_pair_offsets(p, g["states"][s, 0], g["states"][s, 1],
                                              float(g["fs"]), float(g["wavelength"]))
        assert np.array_equal(got, g["offsets"][s])


def test_geometry_pair_swap_antisymmetry(orc, ref):
    """test_geometry.cpp:96-108 / acceptance.cpp criterion 6."""
    rng = np.random.default_rng(0xD16E0)
    wl = orc.wavelength(1575.42e6)
    for _ in range(300):
        c = orc.lla_to_ecef(rng.uniform(-45, 45), rng.uniform(-90, 90), 0.0)
        a = np.r_[orc.lla_to_ecef(rng.uniform(-60, 60), rng.uniform(-180, 179),
                                  rng.uniform(400e3, 1200e3)), rng.uniform(-7600, 7600, 3)]
        b = np.r_[orc.lla_to_ecef(rng.uniform(-60, 60), rng.uniform(-180, 179),
                                  rng.uniform(400e3, 1200e3)), rng.uniform(-7600, 7600, 3)]
        ab = orc.predict_pair_offsets(c, a, b, 5e6, wl)
        ba = orc.predict_pair_offsets(c, b, a, 5e6, wl)
        assert ab[0] == -ba[0]
        assert abs(ab[1] + ba[1]) <= 1e-9
        assert ab == ref.predict_pair_offsets(c, a, b, 5e6, wl)


def test_grid_points_match_reference(orc, ref):
    for bounds, sp, alt in (((-1.0, 1.0, 10.0, 11.0), 0.25, 120.0),
                            ((-0.8, 0.8, -0.8, 0.8), 0.02, 0.0),
                            ((59.0, 61.5, 170.0, 179.9), 0.1, -30.0)):
        assert np.array_equal(orc.build_grid(bounds, sp, alt)[2], ref.build_grid(bounds, sp, alt)[2])


def test_scene_small_golden(orc):
    """Restated driver reproduces the reference's per-snapshot grids bit for bit."""
    g = np.load(os.path.join(GOLDEN, "scene_small.npz"))
    nl, nn, pts = orc.build_grid(tuple(g["bounds"]), float(g["spacing"]), float(g["alt"]))
    per = np.stack([orc.correlate_snapshot(pts, g["states"][s, 0], g["states"][s, 1],
                                           g["captures"][s, 0], g["captures"][s, 1],
                                           float(g["fs"]), float(g["fc"]))
                    for s in range(g["states"].shape[0])])
    assert np.array_equal(per, g["per_snapshot"])
    acc = orc.accumulate(per)
    assert np.array_equal(acc, g["accumulated"])
    det = orc.detect_emitters(acc, nl, nn, float(g["k_sigma"]), int(g["radius"]))
    assert [d[0] for d in det] == list(g["detections"]["grid_index"])
    assert [d[1] for d in det] == list(g["detections"]["score"])


def test_detect_emitters_matches_reference(orc, ref):
    """test_correlate.cpp:160-192 cases plus random surfaces."""
    bounds, sp = (0.0, 1.0, 0.0, 1.0), 0.1  # 11x11
    flat = np.full(121, 3.0)
    assert orc.detect_emitters(flat, 11, 11) == [] == ref.detect_emitters(bounds, sp, 0.0, flat)
    rng = np.random.default_rng(77)
    v = 1.0 + 0.01 * rng.random(121)
    v[7 * 11 + 4] = 2.0
    d = orc.detect_emitters(v, 11, 11, 5.0, 2)
    assert [x[0] for x in d] == [7 * 11 + 4]
    assert d == ref.detect_emitters(bounds, sp, 0.0, v, 5.0, 2)
    v = np.zeros(121)
    v[5 * 11 + 5], v[5 * 11 + 7], v[5 * 11 + 6] = 10.0, 9.0, 8.0
    assert [x[0] for x in orc.detect_emitters(v, 11, 11, 1.0, 5)] == [5 * 11 + 5]
    for seed in range(5):
        v = np.random.default_rng(seed).gamma(2.0, 1.0, 121)
        for k, r in ((1.0, 1), (2.0, 0), (0.5, 3)):
            assert orc.detect_emitters(v, 11, 11, k, r) == ref.detect_emitters(bounds, sp, 0.0, v,
                                                                               k, r)


def test_argmax_first_maximum(orc):
    v = np.array([1.0, 3.0, 2.0, 3.0])
    assert orc.argmax(v) == 1 == int(np.argmax(v))


@pytest.mark.parametrize("name", ["DESK_FOURJAM", "DESK_SAWTOOTH"])
def test_desk_scene_golden(orc, ref, name):
    """The restated driver reproduces the reference's desk-scene answers (scenes.json)."""
    import scenes
    want = json.load(open(os.path.join(GOLDEN, "scenes.json")))[name]
    sc = ref.simulate(scenes.render(getattr(scenes, name)))
    nl, nn, pts = orc.build_grid(sc.bounds, sc.spacing, sc.alt)
    per = np.stack([orc.correlate_snapshot(pts, sc.states[s, 0], sc.states[s, 1],
                                           sc.captures[s, 0], sc.captures[s, 1], sc.fs, sc.fc)
                    for s in range(sc.n_snapshots)])
    acc = orc.accumulate(per)
    import hashlib
    assert hashlib.sha256(acc.tobytes()).hexdigest() == want["accumulated_sha256"]
    assert orc.argmax(acc) == want["argmax"]
    assert acc[want["argmax"]] == float.fromhex(want["argmax_value"])
    det = orc.detect_emitters(acc, nl, nn, sc.k_sigma, sc.radius)
    assert [d[0] for d in det] == want["detections"]
