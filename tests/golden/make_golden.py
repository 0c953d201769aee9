"""Regenerate the golden fixtures in tests/golden/ from the reference itself.

    python tests/golden/make_golden.py      (needs oracle/_ref, i.e. /root/reference here)

Every value below is produced by the unmodified reference headers compiled into
oracle/_ref/libdigeo_ref.so (reference paths relative to /root/reference/proj):

* kat.json          known answers from the reference's own tests:
                    test_correlate.cpp:62-104, test_geometry.cpp:31-79,
                    test_geodesy.cpp:9-23,73-91, test_backend.cpp:35-42
* correlate_small.npz   two Gaussian captures (test_backend.cpp random_capture
                    style) + 256 offsets and the reference correlate_batch output
* offsets_small.npz grid points, receiver states and reference PairOffsets
* scene_small.npz   a 2-snapshot, 2-receiver scene (reference simulator) with the
                    reference's per-snapshot grids, accumulated grid and detections
* scenes.json       desk-scale scenes (tests/scenes.py): reference argmax (index
                    and exact value), detections and a sha256 of the accumulated grid
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle.bindings import PAIR_OFFSETS_DTYPE, RefLib  # noqa: E402
import scenes  # noqa: E402

SMALL_SCENE = {
    **scenes._base(2, 10.0, 2e-3, 1.024e6, 17),
    **scenes._grid(-0.2, 0.2, -0.2, 0.2, 0.02),
    "backend": "serial", "batch_size": 8, "k_sigma": 4, "exclusion_radius_cells": 3,
    "receivers": [scenes._orbit(550e3, 53, -0.9, -0.7), scenes._orbit(550e3, 53, 0.9, 0.5)],
    "emitters": [scenes._chirp(0.06, -0.08, 0, 1e6, 50e-6)],
}


def hexf(x: float) -> str:
    return float(x).hex()


def main():
    ref = RefLib()
    out = {}

    # -- known answers ---------------------------------------------------------
    ones = np.ones(1000, np.complex128)
    kat = {"all_ones_n1000": ref.correlate_point(ones, ones, 1e6, 0, 0.0)}
    ones100 = np.ones(100, np.complex128)
    kat["truncation_n100"] = {str(d): ref.correlate_point(ones100, ones100, 1e6, d, 0.0)
                              for d in (100, -250, 40, -30, 0)}
    kat["wavelength_l1"] = hexf(ref.wavelength(1575.42e6))
    e = ref.lla_to_ecef(0.0, 0.0, 0.0)
    near = ref.lla_to_ecef(0.0, 0.0, 500e3)
    far = ref.lla_to_ecef(0.0, 0.0, 800e3)
    st = lambda p: np.concatenate([p, np.zeros(3)])  # noqa: E731
    d, f = ref.predict_pair_offsets(e, st(near), st(far), 5e6, 0.19)
    kat["tdoa_300km_5mhz"] = d
    kat["ecef_equator"] = [hexf(v) for v in e]
    kat["ecef_pole"] = [hexf(v) for v in ref.lla_to_ecef(90.0, 0.0, 0.0)]
    kat["grid_counts"] = {
        "10x10_at_0.01": list(ref.build_grid((0.0, 10.0, 0.0, 10.0), 0.01, points=False)[:2]),
        "zero_span": list(ref.build_grid((5.0, 5.0, 7.0, 7.0), 0.5, points=False)[:2]),
        "1x2_at_0.5": list(ref.build_grid((0.0, 1.0, 0.0, 2.0), 0.5, points=False)[:2]),
    }
    kat["plan_batches_1e6_8"] = ref.plan_batch_count(1_000_000, 8)
    out["kat.json"] = kat

    # -- correlate_batch ---------------------------------------------------------
    rng = np.random.default_rng(20261017)
    n = 2048
    y1 = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    y2 = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    off = np.zeros(256, PAIR_OFFSETS_DTYPE)
    off["tdoa_samples"] = rng.integers(-n, n, 256)
    off["tdoa_samples"][:8] = [0, 1, -1, n - 1, -(n - 1), n, -n, 3 * n]
    off["fdoa_hz"] = rng.uniform(-1.25e6, 1.25e6, 256)
    off["fdoa_hz"][:4] = 0.0
    want = ref.correlate_batch(y1, y2, 5e6, off, "serial")
    np.savez_compressed(os.path.join(HERE, "correlate_small.npz"), y1=y1, y2=y2, offsets=off,
                        fs=5e6, want=want)

    # -- offsets -----------------------------------------------------------------
    sc = ref.simulate(scenes.render(scenes.DESK_FOURJAM))
    nl, nn, pts = ref.build_grid(sc.bounds, sc.spacing, sc.alt)
    wl = ref.wavelength(sc.fc)
    offs = np.zeros((2, len(pts)), PAIR_OFFSETS_DTYPE)
    for s in range(2):
        for i, p in enumerate(pts):
            offs[s, i] = ref.predict_pair_offsets(p, sc.states[s, 0], sc.states[s, 1], sc.fs, wl)
    np.savez_compressed(os.path.join(HERE, "offsets_small.npz"), bounds=np.array(sc.bounds),
                        spacing=sc.spacing, points=pts, states=sc.states[:2], fs=sc.fs,
                        wavelength=wl, offsets=offs)

    # -- small scene ------------------------------------------------------------
    sc = ref.simulate(scenes.render(SMALL_SCENE))
    res = ref.geolocate(sc.states, sc.captures, sc.fs, sc.fc, sc.bounds, sc.spacing, sc.alt,
                        k_sigma=sc.k_sigma, radius=sc.radius, per_snapshot=True)
    det = np.array([(d["grid_index"], d["score"], d["zsigma"]) for d in res["detections"]],
                   dtype=[("grid_index", "<i8"), ("score", "<f8"), ("zsigma", "<f8")])
    np.savez_compressed(os.path.join(HERE, "scene_small.npz"), states=sc.states,
                        captures=sc.captures, fs=sc.fs, fc=sc.fc, bounds=np.array(sc.bounds),
                        spacing=sc.spacing, alt=sc.alt, k_sigma=sc.k_sigma, radius=sc.radius,
                        per_snapshot=res["per_snapshot"], accumulated=res["accumulated"],
                        detections=det)

    # -- desk scenes ----------------------------------------------------------------
    summary = {}
    for name in ("DESK_FOURJAM", "DESK_SAWTOOTH", "TRIPLE_RX"):
        sc = ref.simulate(scenes.render(getattr(scenes, name)))
        res = ref.geolocate(sc.states, sc.captures, sc.fs, sc.fc, sc.bounds, sc.spacing,
                            sc.alt, backend="parallel", batch_size=4096, k_sigma=sc.k_sigma,
                            radius=sc.radius)
        acc = res["accumulated"]
        am = int(np.argmax(acc))
        summary[name] = {
            "n_lat": res["n_lat"], "n_lon": res["n_lon"], "argmax": am,
            "argmax_value": hexf(acc[am]),
            "top2_gap_rel": float((acc[am] - np.sort(acc)[-2]) / acc[am]),
            "detections": [d["grid_index"] for d in res["detections"]],
            "scores": [hexf(d["score"]) for d in res["detections"]],
            "accumulated_sha256": hashlib.sha256(acc.tobytes()).hexdigest(),
        }
    out["scenes.json"] = summary

    for fname, obj in out.items():
        with open(os.path.join(HERE, fname), "w") as fh:
            json.dump(obj, fh, indent=1, sort_keys=True)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
