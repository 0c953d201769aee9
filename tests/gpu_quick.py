"""Ad-hoc GPU diagnostics (not collected by pytest): parity + timing summary."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2508_06672_b200 as b2  # noqa: E402
from oracle.bindings import PAIR_OFFSETS_DTYPE, OracleLib, RefLib  # noqa: E402

ref = RefLib()
orc = OracleLib()


def rel_err(a, b):
    return np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-300)


def batch_case(n_samples, n_points, fs, seed, fdoa_span):
    rng = np.random.default_rng(seed)
    y1 = rng.standard_normal(n_samples) + 1j * rng.standard_normal(n_samples)
    y2 = rng.standard_normal(n_samples) + 1j * rng.standard_normal(n_samples)
    off = np.zeros(n_points, PAIR_OFFSETS_DTYPE)
    off["tdoa_samples"] = rng.integers(-n_samples, n_samples, n_points)
    off["fdoa_hz"] = rng.uniform(-fdoa_span, fdoa_span, n_points)
    t = time.time()
    want = ref.correlate_batch(y1, y2, fs, off, "parallel", 0, 4096)
    t_ref = time.time() - t
    be = b2.make_backend("b200")
    t = time.time()
    sess = be.stage(b2.BasebandCapture(y1, fs), b2.BasebandCapture(y2, fs))
    got = sess.correlate_batch(off)
    t_gpu = time.time() - t
    got2 = sess.correlate_batch(off)
    e = rel_err(got, want)
    print(f"batch N={n_samples} P={n_points}: max rel {e.max():.3e}  n>1e-4: {(e > 1e-4).sum()}  "
          f"rerun identical: {np.array_equal(got, got2)}  ref {t_ref:.2f}s gpu {t_gpu:.3f}s")
    return e.max()


def scene_case(name):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import scenes
    sc = ref.simulate(scenes.render(getattr(scenes, name)))
    t = time.time()
    want = ref.geolocate(sc.states, sc.captures, sc.fs, sc.fc, sc.bounds, sc.spacing, sc.alt,
                         backend="parallel", batch_size=4096, k_sigma=sc.k_sigma, radius=sc.radius,
                         per_snapshot=True)
    t_ref = time.time() - t
    grid = b2.build_candidate_grid(b2.LatLonBounds(*sc.bounds), sc.spacing, sc.alt)
    opts = b2.GeolocateOptions(k_sigma=sc.k_sigma, exclusion_radius_cells=sc.radius)
    t = time.time()
    res = b2.geolocate_arrays(grid, sc.states, sc.captures, sc.fs, sc.fc, opts)
    t_gpu = time.time() - t
    e = rel_err(res.accumulated.values, want["accumulated"])
    ep = rel_err(np.stack([g.values for g in res.per_snapshot]), want["per_snapshot"])
    print(f"{name}: P={grid.size()} S={sc.n_snapshots} acc max rel {e.max():.3e} per-snap max rel "
          f"{ep.max():.3e} (n>1e-4 {(ep > 1e-4).sum()})  argmax gpu {res.argmax_index} ref "
          f"{int(np.argmax(want['accumulated']))}  val {res.argmax_value!r} vs "
          f"{want['accumulated'][np.argmax(want['accumulated'])]!r}")
    print("   detections gpu", [d.grid_index for d in res.detections], "ref",
          [d["grid_index"] for d in want["detections"]], " stats", res.stats,
          f" ref {t_ref:.2f}s gpu {t_gpu:.3f}s")


if __name__ == "__main__":
    print(b2.default_engine().descriptor())
    import ctypes as C
    from paper_2508_06672_b200._capi import lib
    v = C.c_double()
    lib.dg_fp32_peak_tflops(0, C.byref(v)); print("FFMA peak TFLOP/s", v.value)
    lib.dg_fp32x2_peak_tflops(0, C.byref(v)); print("FFMA2 peak TFLOP/s", v.value)
    # grid + offsets bit-exact
    grid = b2.build_candidate_grid(b2.LatLonBounds(-1.0, 1.0, 10.0, 11.0), 0.25, 120.0)
    nl, nn, pts = ref.build_grid((-1.0, 1.0, 10.0, 11.0), 0.25, 120.0)
    print("grid points bit-exact:", np.array_equal(pts, grid.points))
    batch_case(2048, 10000, 2.048e6, 1, 5e5)
    batch_case(2000, 10000, 5e6, 2, 1.25e6)
    batch_case(50000, 4000, 5e6, 3, 15e3)
    for name in ("DESK_FOURJAM", "DESK_SAWTOOTH", "TRIPLE_RX"):
        scene_case(name)
